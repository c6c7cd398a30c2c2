#!/bin/bash
# Runs the bench on every workload (one JSON line each) into gpurun_out/bench_all.jsonl
out=${1:-gpurun_out/bench_all.jsonl}
mkdir -p gpurun_out
: > $out
for w in cfg1 cfg2 cfg3 cfg4 cfg4bwd long1m circ512 circ1024 circ4096 circ16384 circ65536 circ262144 circ1048576 circ4194304 cfg5 cfg5dense cfg5b sweep256 sweep512 sweep1024 sweep2048 sweep4096 sweep8192 sweep16384 sweep32768 sweep65536 sweep262144 sweep1048576 sweep4194304; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --e2e-steps 3 2>&1 | tail -1 >> $out
done
