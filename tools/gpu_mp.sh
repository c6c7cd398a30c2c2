timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
: > gpurun_out/bench_mp.jsonl
for w in ${WL:-sweep2048 sweep4096 sweep8192 sweep16384 cfg3 cfg4 cfg5}; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --e2e-steps 3 2>&1 | tail -1 >> gpurun_out/bench_mp.jsonl
done
d=gpurun_out/prof_mp; mkdir -p $d
for w in ${PW:-sweep8192}; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k 'regex:fftconv|precompute|mp_|dk_|kf_' -c 12 --csv \
      --log-file $d/launches_$w.csv python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
done
cat gpurun_out/pytest_gpu.log
