#!/bin/bash
cd $(dirname $0)/../..
timeout 1200 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_sparse.py tests/test_gpu_bidir.py -x -q > gpurun_out/pytest_p.log 2>&1; echo "rc $?" >> gpurun_out/pytest_p.log
bash tools/ab.sh "old main e1p" "cfg2 sweep1024 sweep2048 gsweep4096 sweep8192 circ1024" 2
for w in cfg5 cfg5a cfg5dense sp1m_lp sp1m91; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-torch-baseline --no-sweep --e2e-steps 0 > gpurun_out/sp_$w.json 2> gpurun_out/sp_$w.err
done
