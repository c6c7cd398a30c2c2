#!/bin/bash
# session-2 baseline: GPU tests, default bench, ncu launch lists + full captures
cd $(dirname $0)/../..
O=gpurun_out/r02j; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
( time python bench.py ) > $O/bench_default.json 2> $O/bench_default.err
bash tools/r02/prof_a.sh > $O/prof.log 2>&1
