#!/bin/bash
cd $(dirname $0)/../..
timeout 1500 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_sparse.py tests/test_gpu_bidir.py tests/test_gpu_host.py tests/test_gpu_shard.py tests/test_gpu_partial.py -x -q > gpurun_out/pytest_y.log 2>&1; echo "rc $?" >> gpurun_out/pytest_y.log
python bench.py > gpurun_out/bench_y.json 2> gpurun_out/bench_y.err
