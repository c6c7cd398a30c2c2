#!/bin/bash
cd $(dirname $0)/../..
FFTCONV_LIB=$PWD/paper_2311_05908_b200/variants/libfftconv_ditu1d.so timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_bidir.py tests/test_gpu_host.py -x -q > gpurun_out/pytest_ab2.log 2>&1; echo "rc $?" >> gpurun_out/pytest_ab2.log
bash tools/ab.sh "cur3 ditu1 ditu1d" "gsweep2048 gsweep4096 sweep2048 sweep4096" 2
