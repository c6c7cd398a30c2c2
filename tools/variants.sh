#!/bin/bash
# Build experiment variants of libfftconv.so: tools/variants.sh NAME "-DFLAG=.. -DFLAG2=.." [sources to rebuild]
# Objects of the other sources are compiled once (build_obj/base) and reused.
set -e
cd $(dirname $0)/..
C=paper_2311_05908_b200/csrc
V=paper_2311_05908_b200/variants
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I include -I $C --expt-relaxed-constexpr"
mkdir -p $V build_obj/base build_obj/$1
ALL="plan.cpp api.cu kernels_fwd.cu kernels_kf.cu kernels_mp.cu kernels_bwd.cu kernels_f32.cu"
REB=${3:-kernels_fwd.cu}
objs=""
pids=""
for s in $ALL; do
  if [[ " $REB " == *" $s "* ]]; then
    nvcc $F $2 -c $C/$s -o build_obj/$1/$s.o & pids="$pids $!"
    objs="$objs build_obj/$1/$s.o"
  else
    newer=$(find $C include -newer build_obj/base/$s.o \( -name '*.h' -o -name '*.cuh' -o -name $s \) 2>/dev/null | head -1)
    if [ ! -f build_obj/base/$s.o ] || [ -n "$newer" ]; then
      nvcc $F -c $C/$s -o build_obj/base/$s.o & pids="$pids $!"
    fi
    objs="$objs build_obj/base/$s.o"
  fi
done
for p in $pids; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o $V/libfftconv_$1.so $objs
echo built $V/libfftconv_$1.so
