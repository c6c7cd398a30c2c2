#!/bin/bash
cd $(dirname $0)/../..
timeout 1500 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_fwd.py tests/test_gpu_partial.py tests/test_gpu_sparse.py tests/test_gpu_f32.py tests/test_gpu_bidir.py tests/test_gpu_shard.py tests/test_gpu_host.py -q > gpurun_out/pytest_q.log 2>&1; echo "rc $?" >> gpurun_out/pytest_q.log
bash tools/ab.sh "main circ cur" "cfg3 sweep8192 circ1024 circ16384 cfg4 cfg4bwd sweep65536" 1
