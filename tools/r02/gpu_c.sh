#!/bin/bash
cd $(dirname $0)/../..
O=gpurun_out/r02c; mkdir -p $O
( time python bench.py ) > $O/bench_default.json 2> $O/bench_default.err
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1
python bench.py --shard cfg4 --steps 10 --warmup 3 > $O/shard_cfg4.json 2> $O/shard_cfg4.err
bash tools/trace_fwd.sh build > $O/trace_build.log 2>&1
for a in "1024" "8192"; do bash tools/trace_fwd.sh $a >> $O/trace.txt 2>&1; done
