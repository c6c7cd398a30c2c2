#!/bin/bash
cd $(dirname $0)/../..
O=gpurun_out/r02f; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q -k "order3 or short_filter or bwd_parity or multipass_parity or host or shard" > $O/pytest_gpu.txt 2>&1
python bench.py --sweep sweep2048,sweep4096,gsweep2048,gsweep4096 --no-cpu-baseline --no-torch-baseline --e2e-steps 0 > $O/bench.json 2> $O/bench.err
FFTCONV_DIT=0 python bench.py --sweep sweep2048,sweep4096,gsweep2048,gsweep4096 --no-cpu-baseline --no-torch-baseline --e2e-steps 0 > $O/bench_nodit.json 2> $O/bench_nodit.err
