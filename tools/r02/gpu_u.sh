#!/bin/bash
cd $(dirname $0)/../..
timeout 900 python -m pytest tests/test_gpu_fwd.py -q -k "multipass or dit or order3 or 2048 or 4096" > gpurun_out/pytest_u.log 2>&1; echo "rc $?" >> gpurun_out/pytest_u.log
bash tools/ab.sh "skp ditslot" "sweep2048 sweep4096 gsweep2048 gsweep4096 cfg2" 2
