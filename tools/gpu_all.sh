timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
python tools/f32_report.py > gpurun_out/f32_report.txt 2>&1
bash tools/bench_all.sh gpurun_out/bench_all.jsonl
cat gpurun_out/pytest_gpu.log
