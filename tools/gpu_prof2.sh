d=gpurun_out/prof_r01c; mkdir -p $d
K='regex:fftconv|precompute|mp_|dk_|kf_'
for w in sweep2048 sweep8192 cfg4; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k "$K" -c 12 --csv \
      --log-file $d/launches_$w.csv python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > /dev/null 2>&1
done
FFTCONV_LIB=$PWD/paper_2311_05908_b200/trace/libfftconv_trace.so python tools/trace_fwd.py 2048 circular_plain > $d/trace_circ_plain.txt 2>&1
ls $d
