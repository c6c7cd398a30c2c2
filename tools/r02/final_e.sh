#!/bin/bash
# last check of the round: full GPU tests, smoke, default bench (+ sweep)
cd $(dirname $0)/../..
O=gpurun_out/final_f; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
( time python bench.py ) > $O/bench_default.json 2> $O/bench_default.err
nvidia-smi > $O/smi.txt
tail -3 $O/pytest_gpu.log; tail -1 $O/smoke.log
