#!/bin/bash
cd $(dirname $0)/../..
FFTCONV_LIB=$PWD/paper_2311_05908_b200/variants/libfftconv_bwdpf.so timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_partial.py tests/test_gpu_bidir.py -x -q -k "bwd or partial" > gpurun_out/pytest_aa.log 2>&1; echo "rc $?" >> gpurun_out/pytest_aa.log
bash tools/ab.sh "cur3 bwdpf" "cfg3 cfg4bwd long1m" 2
