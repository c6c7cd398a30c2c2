#!/bin/bash
cd $(dirname $0)/../..
python tools/microbench.py > gpurun_out/microbench2.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_partial.py tests/test_gpu_sparse.py -x -q > gpurun_out/pytest_m.log 2>&1; echo "rc $?" >> gpurun_out/pytest_m.log
bash tools/ab.sh "old new" "cfg2 gsweep2048 sweep2048 sweep1024 gsweep4096 sweep8192 circ1024" 2
