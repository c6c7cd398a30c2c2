timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest10.log
timeout 900 python bench.py > gpurun_out/bench10.json 2> gpurun_out/bench10.err
cat gpurun_out/pytest10.log
