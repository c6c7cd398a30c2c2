# round-end evidence: GPU tests, bench over every workload, ncu launch lists + full captures
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
python tools/f32_report.py > gpurun_out/f32_report.txt 2>&1
bash tools/bench_all.sh gpurun_out/bench_all.jsonl
bash tools/profile.sh final > /dev/null 2>&1
cat gpurun_out/pytest_gpu.log
