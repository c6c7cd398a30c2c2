#!/bin/bash
# Build experiment variants of libfftconv.so: tools/variants.sh NAME "-DFLAG=.. -DFLAG2=.."
set -e
cd $(dirname $0)/..
C=paper_2311_05908_b200/csrc
mkdir -p paper_2311_05908_b200/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -I include -I $C \
  --expt-relaxed-constexpr $2 -o paper_2311_05908_b200/variants/libfftconv_$1.so \
  $C/plan.cpp $C/api.cu $C/kernels_fwd.cu $C/kernels_kf.cu $C/kernels_mp.cu $C/kernels_bwd.cu $C/kernels_f32.cu
