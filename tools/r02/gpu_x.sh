#!/bin/bash
cd $(dirname $0)/../..
FFTCONV_LIB=$PWD/paper_2311_05908_b200/variants/libfftconv_aits.so timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_bidir.py -x -q -k "causal or fused or bidir" > gpurun_out/pytest_x.log 2>&1; echo "rc $?" >> gpurun_out/pytest_x.log
bash tools/ab.sh "cur2 aits pipe2 split2" "cfg2 sweep1024 sweep256 gsweep512 sweep8192 circ1024" 2
