#!/bin/bash
cd $(dirname $0)/../..
timeout 1200 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_partial.py tests/test_gpu_host.py tests/test_gpu_sparse.py -x -q > gpurun_out/pytest_s.log 2>&1; echo "rc $?" >> gpurun_out/pytest_s.log
bash tools/ab.sh "skp pdl" "cfg2 sweep1024 sweep256 gsweep2048 sweep8192 cfg4" 2
