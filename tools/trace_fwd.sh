#!/bin/bash
# Experiment: build a -DFC_TRACE library and print per-phase cycle stamps.
set -e
cd $(dirname $0)/..
C=paper_2311_05908_b200/csrc
mkdir -p paper_2311_05908_b200/ablate
[ "$1" = build ] && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -I include -I $C \
  --expt-relaxed-constexpr -DFC_TRACE $EXTRA -o paper_2311_05908_b200/ablate/libfftconv_trace.so \
  $C/plan.cpp $C/api.cu $C/kernels_fwd.cu $C/kernels_kf.cu $C/kernels_mp.cu $C/kernels_bwd.cu $C/kernels_f32.cu
[ "$1" = build ] && exit 0
FFTCONV_LIB=$PWD/paper_2311_05908_b200/ablate/libfftconv_trace.so python tools/trace_fwd.py ${1:-1024} $2
