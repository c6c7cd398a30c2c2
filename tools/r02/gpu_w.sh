#!/bin/bash
cd $(dirname $0)/../..
timeout 1200 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_bidir.py tests/test_gpu_host.py tests/test_gpu_shard.py tests/test_gpu_sparse.py -x -q > gpurun_out/pytest_w.log 2>&1; echo "rc $?" >> gpurun_out/pytest_w.log
bash tools/ab.sh "allwait direct" "cfg2 sweep1024 sweep256 gsweep512 gsweep2048 gsweep4096 sweep2048 sweep4096" 2
