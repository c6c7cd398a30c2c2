timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
python tools/f32_report.py > gpurun_out/f32_report.txt 2>&1
: > gpurun_out/bench_big.jsonl
for w in cfg2 sweep1048576 cfg5b cfg3; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline --e2e-steps 3 2>&1 | tail -1 >> gpurun_out/bench_big.jsonl
done
timeout 600 ncu --metrics gpu__time_duration.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum --clock-control none -k 'regex:kf_|mp_cols|precompute' -c 6 --csv --log-file gpurun_out/launches_kf1m.csv python bench.py --workload sweep1048576 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
cat gpurun_out/pytest_gpu.log
