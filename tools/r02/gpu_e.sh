#!/bin/bash
cd $(dirname $0)/../..
O=gpurun_out/r02e; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "fwd_causal or cfg1 or cfg2 or flat or delta or host or shard or short_filter or edge" > $O/pytest_gpu.txt 2>&1
python bench.py --sweep sweep256,sweep512,sweep1024,gsweep512 --no-cpu-baseline --no-torch-baseline > $O/bench.json 2> $O/bench.err
bash tools/trace_fwd.sh build > $O/trace_build.log 2>&1
for a in "1024"; do bash tools/trace_fwd.sh $a >> $O/trace.txt 2>&1; done
