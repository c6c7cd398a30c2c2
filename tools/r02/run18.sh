timeout 200 python -u tools/r02/cpl_check.py 8192 2>&1 | grep rel
for w in sweep8192 gsweep8192; do
echo -n "$w "; timeout 300 python bench.py --workload $w --steps 100 --no-cpu-baseline --e2e-steps 2 --no-sweep 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step_ms %.4f conv_ms %.4f frac %.3f' % (d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac']))"
done
