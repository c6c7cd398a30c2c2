#!/bin/bash
cd $(dirname $0)/../..
O=gpurun_out/r02d; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "fwd or shard or host or sparse or partial" > $O/pytest_gpu.txt 2>&1
python bench.py --sweep sweep1024,sweep2048,sweep8192,gsweep2048,cfg5 --no-cpu-baseline --no-torch-baseline > $O/bench.json 2> $O/bench.err
bash tools/trace_fwd.sh build > $O/trace_build.log 2>&1
for a in "1024" "8192"; do bash tools/trace_fwd.sh $a >> $O/trace.txt 2>&1; done
