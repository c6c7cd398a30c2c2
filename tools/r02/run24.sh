timeout 1200 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_bidir.py tests/test_gpu_shard.py -q -x 2>&1 | tail -2
for w in sweep2048 gsweep2048 sweep4096 gsweep4096 sweep8192 gsweep8192; do
STEPS=200 bash tools/variant.sh run "main" $w 2>&1
done
