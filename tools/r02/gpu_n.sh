#!/bin/bash
cd $(dirname $0)/../..
timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_partial.py tests/test_gpu_sparse.py tests/test_gpu_bidir.py -x -q > gpurun_out/pytest_n.log 2>&1; echo "rc $?" >> gpurun_out/pytest_n.log
bash tools/ab.sh "nots ts" "cfg2 gsweep2048 sweep2048 sweep1024 gsweep4096 sweep8192 circ1024 circ16384 cfg4" 2
