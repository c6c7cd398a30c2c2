#!/bin/bash
cd $(dirname $0)/../..
O=gpurun_out/r02h; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q -k "order3 or short_filter or bwd_parity" > $O/pytest_gpu.txt 2>&1
python bench.py --sweep sweep2048,sweep4096,gsweep2048,gsweep4096,sweep8192,sweep65536,sweep1048576,sweep4194304 --no-cpu-baseline --no-torch-baseline --e2e-steps 0 > $O/bench.json 2> $O/bench.err
