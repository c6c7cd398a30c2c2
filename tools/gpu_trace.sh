timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
export FFTCONV_LIB=$PWD/paper_2311_05908_b200/trace/libfftconv_trace.so
( python tools/trace_fwd.py 1024; python tools/trace_fwd.py 1024 plain; python tools/trace_fwd.py 2048 circular ) > gpurun_out/trace.txt 2>&1
unset FFTCONV_LIB
python tools/microbench.py > gpurun_out/microbench.txt 2>&1
timeout 300 python bench.py --workload sweep32768 --no-cpu-baseline --e2e-steps 3 2>&1 | tail -1 > gpurun_out/b32k.json
cat gpurun_out/pytest_gpu.log
