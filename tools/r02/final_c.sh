#!/bin/bash
# round-2 session-3 evidence on one B200: GPU tests, PDL probe, default bench
# (+ sweep), extra workloads, sanitizer slice over the order-3 kernels, ncu
cd $(dirname $0)/../..
O=gpurun_out/final_c; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log
for p in 1 0; do for n in 1024 8192; do FFTCONV_PDL=$p timeout 300 python tools/pdl_probe.py $n gated; done; done > $O/pdl_probe.txt 2>&1
( time python bench.py ) > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --workload cfg2 --steps 50 --warmup 5 --no-cpu-baseline --no-torch-baseline --e2e-steps 0 \
  --sweep cfg1,cfg5b,long1m,circ512,circ4096,circ65536,circ262144,circ1048576,circ4194304,sp1m91,gsweep16384,sweep16384 \
  > $O/bench_extra.json 2> $O/bench_extra.err
K="test_fwd_order3_single_pass and f16 or test_fwd_causal_parity and 1024 and f16 and True"
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 \
  python -m pytest tests -m gpu -q -x -k "$K" > $O/memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 \
  python -m pytest tests -m gpu -q -x -k "test_fwd_order3_single_pass and f16" > $O/racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/racecheck.log
timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 9 \
  python -m pytest tests -m gpu -q -x -k "test_fwd_order3_single_pass and f16 and False" > $O/synccheck.log 2>&1; echo "synccheck rc=$?" >> $O/synccheck.log
d=$O/prof; mkdir -p $d
K='regex:fftconv|precompute|mp_|dk_|kf_'
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.per_cycle_active
for w in cfg2 sweep2048 sweep4096 sweep8192 gsweep8192 cfg3; do
  timeout 600 ncu --metrics $M --clock-control none -k "$K" -c 60 --csv \
      --log-file $d/launches_$w.csv python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --no-torch-baseline --no-sweep --e2e-steps 0 > /dev/null 2>&1
done
full() {
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$3" -s $4 -c $5 -o $d/$1 \
      python bench.py --workload $2 --steps 1 --warmup 3 --no-cpu-baseline --no-torch-baseline --no-sweep --e2e-steps 0 > /dev/null 2>&1
}
full fwd_cfg2 cfg2 fftconv_fwd_o2 3 1
full o3_sweep4096 sweep4096 fftconv_fwd_o2 3 1
full o3_sweep8192 sweep8192 fftconv_fwd_o2 3 1
for r in $d/*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>/dev/null
  ncu -i $r --page source --csv > ${r%.ncu-rep}_source.csv 2>/dev/null
done
nvidia-smi > $O/smi.txt
cat $O/pytest_gpu.log | tail -3; cat $O/pdl_probe.txt; tail -1 $O/memcheck.log; tail -1 $O/racecheck.log; tail -1 $O/synccheck.log
