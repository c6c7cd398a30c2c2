#!/bin/bash
cd $(dirname $0)/../..
timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_bidir.py tests/test_gpu_host.py tests/test_gpu_shard.py -x -q > gpurun_out/pytest_ab3.log 2>&1; echo "rc $?" >> gpurun_out/pytest_ab3.log
bash tools/ab.sh "cur3 cur4" "gsweep2048 gsweep4096 cfg2" 1
python tools/kf_timing.py > gpurun_out/kf_timing.txt 2>&1
