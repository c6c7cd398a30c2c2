#!/bin/bash
cd $(dirname $0)/../..
O=gpurun_out/r02i; mkdir -p $O
python tools/cost_model.py measure $O/cost_constants.json > $O/cost_measure.log 2>&1
( time python bench.py ) > $O/bench_default.json 2> $O/bench_default.err
python bench.py --workload cfg2 --steps 50 --warmup 5 --no-cpu-baseline --no-torch-baseline --e2e-steps 0 --sweep sweep4096,gsweep4096,cfg5b,long1m,circ4096,circ65536,circ1048576 > $O/bench_extra.json 2> $O/bench_extra.err
