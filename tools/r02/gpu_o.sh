#!/bin/bash
cd $(dirname $0)/../..
timeout 1200 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_sparse.py tests/test_gpu_partial.py tests/test_gpu_bidir.py tests/test_gpu_shard.py -x -q > gpurun_out/pytest_o.log 2>&1; echo "rc $?" >> gpurun_out/pytest_o.log
bash tools/ab.sh "nopipe0 pipe0" "cfg2 gsweep2048 sweep2048 sweep1024 gsweep4096 sweep8192 circ1024 cfg5" 2
