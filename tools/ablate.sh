#!/bin/bash
# Build ablation variants of libfftconv.so (experiments only; not the product)
# and time a workload's conv with each: tools/ablate.sh build | run [workload]
set -e
cd $(dirname $0)/..
if [ "$1" = build ]; then
  C=paper_2311_05908_b200/csrc
  for a in 0 1 2 4 3 6; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -I include -I $C \
      --expt-relaxed-constexpr -DFC_ABLATE=$a -o paper_2311_05908_b200/ablate/libfftconv_a$a.so \
      $C/plan.cpp $C/api.cu $C/kernels_fwd.cu $C/kernels_kf.cu $C/kernels_mp.cu $C/kernels_bwd.cu &
  done
  wait
else
  for a in 0 1 2 4 3 6; do
    echo -n "ablate=$a "
    FFTCONV_LIB=$PWD/paper_2311_05908_b200/ablate/libfftconv_a$a.so python bench.py --workload ${2:-cfg2} --steps 200 --no-cpu-baseline --e2e-steps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('conv_ms %.4f' % d['roofline']['kernel_ms'])"
  done
fi
