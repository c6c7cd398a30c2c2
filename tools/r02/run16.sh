timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_bidir.py -q -x -k "causal or circular or bidir or host" 2>&1 | tail -2
for p in 0; do for n in 1024; do FFTCONV_PDL=$p timeout 300 python tools/pdl_probe.py $n gated; done; done
for w in cfg2 sweep256 sweep1024; do
echo -n "$w "; timeout 300 python bench.py --workload $w --steps 300 --no-cpu-baseline --e2e-steps 2 --no-sweep 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step_ms %.4f conv_ms %.4f frac %.3f' % (d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac']))"
done
