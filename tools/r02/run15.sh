timeout 1200 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_bwd.py tests/test_gpu_bidir.py tests/test_gpu_shard.py -q -x 2>&1 | tail -3
for w in sweep2048 sweep4096 gsweep2048 gsweep4096 sweep8192; do
echo -n "$w "; timeout 300 python bench.py --workload $w --steps 100 --no-cpu-baseline --e2e-steps 2 --no-sweep 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step_ms %.4f conv_ms %.4f frac %.3f' % (d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac']))"
done
