#!/bin/bash
# ncu evidence for the bench workloads (run under gpurun; 1 GPU).
# Usage: tools/profile.sh <tag>   -> gpurun_out/prof_<tag>/...
tag=${1:-r01}
d=gpurun_out/prof_$tag
mkdir -p $d
K='regex:fftconv|precompute|mp_|dk_|kf_'
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed
# 1. launch lists of one warm step (cold-cache, serialised: compare shares, not absolutes)
for w in ${WORKLOADS:-cfg2 cfg3 cfg4 cfg4bwd cfg5 sweep1024 sweep8192 long1m}; do
  timeout 900 ncu --metrics $M --clock-control none -k "$K" -c 60 --csv \
      --log-file $d/launches_$w.csv python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done
# 2. full sections of the dominant kernels
if [ -z "$NOFULL" ]; then
full() {  # name workload kernel-regex skip count
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$3" -s $4 -c $5 -o $d/$1 \
      python bench.py --workload $2 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
}
full fwd_cfg2 cfg2 fftconv_fwd_o2 3 1
full kf_cfg2 cfg2 precompute_kf 3 1
full bwd_cfg3 cfg3 fftconv_bwd_o2 2 1
full mp_sweep8192 sweep8192 "mp_pass|fftconv_fwd_o2" 3 3
fi
# 3. text summaries
for r in $d/*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>/dev/null
done
ls -la $d
