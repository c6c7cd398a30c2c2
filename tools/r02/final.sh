#!/bin/bash
# round-2 final evidence on one B200: GPU tests, default bench (+ sweep),
# extra workloads, cost-model constants, sanitizer slice, ncu of cfg2
cd $(dirname $0)/../..
O=gpurun_out/final; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log
( time python bench.py ) > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --workload cfg2 --steps 50 --warmup 5 --no-cpu-baseline --no-torch-baseline --e2e-steps 0 \
  --sweep cfg1,cfg5b,long1m,circ512,circ4096,circ65536,circ262144,circ1048576,circ4194304,sp1m91,gsweep16384,sweep16384 \
  > $O/bench_extra.json 2> $O/bench_extra.err
timeout 600 python tools/cost_model.py measure $O/cost_constants.json > $O/cost.log 2>&1
K="test_fwd_causal_parity and 1024 and f16 or test_fwd_multipass_parity and 8192 and f16 or test_bwd_parity and 1024 or test_bwd_parity and 8192 or test_partial_parity and 700 or test_sparse_lowpass_slow_digit_skip and 8192 or test_bidir_fwd and 2048 or test_fwd_host_matches_device"
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 \
  python -m pytest tests -m gpu -q -x -k "$K" > $O/memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/memcheck.log
K2="test_fwd_causal_parity and 1024 and f16 or test_fwd_multipass_parity and 8192 and f16 and False or test_bwd_parity and 1024 and f16"
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 \
  python -m pytest tests -m gpu -q -x -k "$K2" > $O/racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/racecheck.log
WL="cfg2 sweep8192 cfg3" bash tools/r02/prof_b.sh > $O/prof.log 2>&1
nvidia-smi > $O/smi.txt
