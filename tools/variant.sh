#!/bin/bash
# Experiment helper: build a variant library with extra -D flags
#   tools/variant.sh build NAME "-DFLAG ..."   -> paper_2311_05908_b200/ablate/libfftconv_NAME.so
#   tools/variant.sh run "NAME1 NAME2 ..." [workload]  -> conv kernel ms of each
set -e
cd $(dirname $0)/..
C=paper_2311_05908_b200/csrc
if [ "$1" = build ]; then
  mkdir -p paper_2311_05908_b200/ablate
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -I include -I $C \
    --expt-relaxed-constexpr $3 -o paper_2311_05908_b200/ablate/libfftconv_$2.so \
    $C/plan.cpp $C/api.cu $C/kernels_fwd.cu $C/kernels_kf.cu $C/kernels_mp.cu $C/kernels_bwd.cu $C/kernels_f32.cu
else
  for v in $2; do
    if [ "$v" = main ]; then lib=$PWD/paper_2311_05908_b200/libfftconv.so; else lib=$PWD/paper_2311_05908_b200/ablate/libfftconv_$v.so; fi
    echo -n "$v ${3:-cfg2} "
    FFTCONV_LIB=$lib python bench.py --workload ${3:-cfg2} --steps ${STEPS:-300} --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('conv_ms %.4f frac %.3f' % (d['roofline']['kernel_ms'], d['roofline']['frac']))"
  done
fi
