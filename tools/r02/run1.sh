set -x
timeout 600 python -m pytest tests/test_gpu_fwd.py -q -x 2>&1 | tail -3
for r in 1 2; do for p in 0 1; do for w in cfg2 sweep2048 sweep1024; do
echo -n "pdl=$p $w "; FFTCONV_PDL=$p timeout 300 python bench.py --workload $w --steps 300 --no-cpu-baseline --e2e-steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step_ms %.4f conv_ms %.4f' % (d['ms_per_step'], d['roofline']['kernel_ms']))"
done; done; done
for n in "1024 causal-plain" "2048 causal-plain" "4096 causal-plain" "4096 causal-gated"; do bash tools/trace_fwd.sh $n 2>&1 | tail -25; done
