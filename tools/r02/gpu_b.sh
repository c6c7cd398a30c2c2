#!/bin/bash
cd $(dirname $0)/../..
mkdir -p gpurun_out/r02b
bash tools/trace_fwd.sh build > gpurun_out/r02b/trace_build.log 2>&1
for a in "1024" "1024 causal-plain" "2048 circular-plain"; do
  bash tools/trace_fwd.sh $a >> gpurun_out/r02b/trace.txt 2>&1
done
timeout 1500 python -m pytest tests -m gpu -x -q -k "range_stress or whole_rows or short_filter or sparse_partial or cfg2_full or cfg3 or cfg4 or cfg5 or f32 or bwd_parity" > gpurun_out/r02b/pytest_new.txt 2>&1
