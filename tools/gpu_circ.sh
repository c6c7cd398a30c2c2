: > gpurun_out/bench_circ.jsonl
for w in circ512 circ1024 circ4096 circ16384 circ65536 circ262144 circ1048576 circ4194304; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --e2e-steps 3 2>&1 | tail -1 >> gpurun_out/bench_circ.jsonl
done
