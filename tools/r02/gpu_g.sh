#!/bin/bash
cd $(dirname $0)/../..
O=gpurun_out/r02g; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
