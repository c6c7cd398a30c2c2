#!/bin/bash
# A/B: fused forward after a change -- fwd parity tests + key workloads
cd $(dirname $0)/../..
O=gpurun_out/${1:-r02l}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_bidir.py tests/test_gpu_host.py tests/test_gpu_shard.py -x -q > $O/pytest.log 2>&1; echo "rc $?" >> $O/pytest.log
for w in cfg2 sweep1024 sweep256 sweep2048 gsweep2048 sweep4096 circ1024 sweep8192; do
  timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline --no-torch-baseline --no-sweep --e2e-steps 0 > $O/bench_$w.json 2>$O/bench_$w.err
done
python tools/show.py $O/bench_*.json > $O/summary.txt 2>&1
