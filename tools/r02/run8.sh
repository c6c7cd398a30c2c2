timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for w in sweep8192 gsweep8192 cfg3 sweep4096 gsweep4096 sweep2048 cfg2; do
echo -n "$w "; timeout 300 python bench.py --workload $w --steps 100 --no-cpu-baseline --e2e-steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step_ms %.4f conv_ms %.4f frac %.3f' % (d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac']))"
done
bash tools/trace_fwd.sh 8192 causal-plain 2>&1 | tail -22
