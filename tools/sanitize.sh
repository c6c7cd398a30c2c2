#!/bin/bash
# compute-sanitizer memcheck over a small representative slice of the GPU tests
mkdir -p gpurun_out
K="test_fwd_causal_parity and 1024 and f16 or test_fwd_multipass_parity and 8192 and f16 or test_bwd_parity and 1024 or test_partial_parity and 700 or test_f32_fused_causal or test_fwd_host_matches_device or test_fwd_stream or test_bwd_multilevel_parity and 32768 and f16 or test_sparse_rows_skipped"
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 \
  python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/memcheck.log
tail -5 gpurun_out/memcheck.log
