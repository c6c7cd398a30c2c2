#!/bin/bash
cd $(dirname $0)/../..
O=gpurun_out/r02k; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_bidir.py -x -q > $O/pytest_bidir.log 2>&1; echo "rc $?" >> $O/pytest_bidir.log
for a in "1024" "1024 causal-plain" "2048 circular-plain"; do
  FFTCONV_LIB=$PWD/paper_2311_05908_b200/ablate/libfftconv_trace.so timeout 300 python tools/trace_fwd.py $a >> $O/trace.txt 2>&1
done
