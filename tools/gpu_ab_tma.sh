timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
: > gpurun_out/ab.txt
for r in 1 2; do for w in sweep2048 sweep8192 sweep16384 cfg4 cfg5 cfg3; do for t in 0 1; do
 echo -n "$w tma=$t " >> gpurun_out/ab.txt
 FFTCONV_TMA_Y=$t timeout 300 python bench.py --workload $w --steps 200 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('conv_ms %.4f step_ms %.4f' % (d['roofline']['kernel_ms'], d['ms_per_step']))" >> gpurun_out/ab.txt 2>&1
done; done; done
sort gpurun_out/ab.txt
