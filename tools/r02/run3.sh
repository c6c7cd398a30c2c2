timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_bwd.py tests/test_gpu_bidir.py tests/test_gpu_shard.py -q -x 2>&1 | tail -3
for w in sweep2048 sweep4096 gsweep2048 gsweep4096; do
echo -n "$w "; timeout 300 python bench.py --workload $w --steps 200 --no-cpu-baseline --e2e-steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step_ms %.4f conv_ms %.4f frac %.3f' % (d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac']))"
done
for n in "4096 causal-plain" "2048 causal-plain" "4096 causal-gated"; do bash tools/trace_fwd.sh $n 2>&1 | tail -22; done
