#!/bin/bash
# ncu of the last build's order-3 kernels (launch lists + full captures)
cd $(dirname $0)/../..
d=gpurun_out/prof_g; mkdir -p $d
K='regex:fftconv|precompute|mp_|dk_|kf_'
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.per_cycle_active
for w in cfg2 sweep2048 sweep4096 sweep8192 gsweep8192; do
  timeout 600 ncu --metrics $M --clock-control none -k "$K" -c 60 --csv \
      --log-file $d/launches_$w.csv python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --no-torch-baseline --no-sweep --e2e-steps 0 > /dev/null 2>&1
done
full() {
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$3" -s $4 -c $5 -o $d/$1 \
      python bench.py --workload $2 --steps 1 --warmup 3 --no-cpu-baseline --no-torch-baseline --no-sweep --e2e-steps 0 > /dev/null 2>&1
}
full o3_sweep4096 sweep4096 fftconv_fwd_o2 3 1
full o3_sweep8192 sweep8192 fftconv_fwd_o2 3 1
full o3g_gsweep8192 gsweep8192 fftconv_fwd_o2 3 1
full kf_sweep8192 sweep8192 precompute_kf 3 1
for r in $d/*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>/dev/null
  ncu -i $r --page source --csv > ${r%.ncu-rep}_source.csv 2>/dev/null
done
rm -f $d/*.ncu-rep
ls $d
