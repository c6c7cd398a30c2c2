timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
: > gpurun_out/chunk.jsonl
for mb in 0 16 32 48 96; do
 for w in sweep2048 sweep8192 sweep16384 cfg4 cfg5; do
  echo "chunk $mb $w" >> gpurun_out/chunk.jsonl
  FFTCONV_CHUNK_MB=$mb timeout 300 python bench.py --workload $w --no-cpu-baseline --e2e-steps 3 --steps 100 2>&1 | tail -1 >> gpurun_out/chunk.jsonl
 done
done
cat gpurun_out/pytest_gpu.log
