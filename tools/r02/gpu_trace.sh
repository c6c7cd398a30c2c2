#!/bin/bash
# round-2 baseline: per-phase stamps of the fused kernel + conv ms of key workloads
cd $(dirname $0)/../..
mkdir -p gpurun_out/r02a
bash tools/trace_fwd.sh build > gpurun_out/r02a/trace_build.log 2>&1
for a in "1024" "1024 causal-plain" "2048 circular-plain"; do
  bash tools/trace_fwd.sh $a >> gpurun_out/r02a/trace.txt 2>&1
done
for w in cfg2 sweep1024 sweep2048 sweep8192 cfg3 cfg5; do
  python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r02a/bench_$w.json 2>gpurun_out/r02a/bench_$w.err
done
nvidia-smi > gpurun_out/r02a/smi.txt
