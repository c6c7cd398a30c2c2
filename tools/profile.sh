#!/bin/bash
# ncu evidence for the bench workloads (run under gpurun; 1 GPU).
# Usage: tools/profile.sh <tag>   -> gpurun_out/prof_<tag>/...
tag=${1:-r01}
d=gpurun_out/prof_$tag
mkdir -p $d
K='regex:fftconv|precompute|mp_|dk_|kf_'
# 1. launch lists (cold-cache, serialised: compare shares, not absolutes)
for w in ${WORKLOADS:-cfg2 cfg3 cfg4 cfg5 sweep2048 sweep8192}; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 40 --csv \
      --log-file $d/launches_$w.csv python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
done
# 2. full sections of the dominant kernels
if [ -z "$NOFULL" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fftconv_fwd_o2 -s 3 -c 1 -o $d/fwd_cfg2 \
    python bench.py --workload cfg2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fftconv_bwd_o2 -s 1 -c 1 -o $d/bwd_cfg3 \
    python bench.py --workload cfg3 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"mp_pass|fftconv_fwd_o2" -s 3 -c 3 -o $d/mp_sweep8192 \
    python bench.py --workload sweep8192 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
fi
# 3. text summaries
for r in $d/*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>/dev/null
done
ls -la $d
