#!/bin/bash
# round-2 session-3 closing evidence on one B200: GPU tests, default bench
# (+ sweep), extra workloads, ncu launch lists + full captures
cd $(dirname $0)/../..
O=gpurun_out/final_d; mkdir -p $O
[ -z "$SKIP_TESTS" ] && { timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log; }
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
( time python bench.py ) > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --workload cfg2 --steps 50 --warmup 5 --no-cpu-baseline --no-torch-baseline --e2e-steps 0 \
  --sweep cfg1,cfg5b,long1m,circ512,circ4096,circ65536,circ262144,circ1048576,circ4194304,sp1m91,gsweep16384,sweep16384 \
  > $O/bench_extra.json 2> $O/bench_extra.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/reference.json 2> $O/reference.err
d=$O/prof; mkdir -p $d
K='regex:fftconv|precompute|mp_|dk_|kf_'
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.per_cycle_active
for w in cfg2 sweep1024 sweep2048 sweep4096 sweep8192 gsweep8192 cfg3 cfg4; do
  timeout 600 ncu --metrics $M --clock-control none -k "$K" -c 60 --csv \
      --log-file $d/launches_$w.csv python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --no-torch-baseline --no-sweep --e2e-steps 0 > /dev/null 2>&1
done
full() {
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$3" -s $4 -c $5 -o $d/$1 \
      python bench.py --workload $2 --steps 1 --warmup 3 --no-cpu-baseline --no-torch-baseline --no-sweep --e2e-steps 0 > /dev/null 2>&1
}
full fwd_cfg2 cfg2 fftconv_fwd_o2 3 1
full kf_cfg2 cfg2 precompute_kf 3 1
full o3_sweep2048 sweep2048 fftconv_fwd_o2 3 1
full o3_sweep8192 sweep8192 fftconv_fwd_o2 3 1
full o3g_gsweep8192 gsweep8192 fftconv_fwd_o2 3 1
for r in $d/*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>/dev/null
  ncu -i $r --page source --csv > ${r%.ncu-rep}_source.csv 2>/dev/null
done
rm -f $d/*.ncu-rep  # (gpurun copies back <= 64 MiB)
nvidia-smi > $O/smi.txt
cat $O/smoke.log | tail -1; tail -c 400 $O/bench_default.json; tail -c 300 $O/reference.json
