set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench_default.log 2>&1
bash tools/bench_all.sh gpurun_out/bench_all.jsonl
tail -3 gpurun_out/pytest_gpu.log
tail -2 gpurun_out/bench_default.log
