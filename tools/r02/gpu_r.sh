#!/bin/bash
cd $(dirname $0)/../..
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_fwd.py -q > gpurun_out/pytest_r.log 2>&1; echo "rc $?" >> gpurun_out/pytest_r.log
for w in cfg5a cfg5dense sp1m_lp sp1m91 cfg5; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-torch-baseline --no-sweep --e2e-steps 0 > gpurun_out/sp_$w.json 2> gpurun_out/sp_$w.err
done
bash tools/r02/prof_b.sh > gpurun_out/prof_b.log 2>&1
