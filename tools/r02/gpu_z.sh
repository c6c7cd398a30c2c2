#!/bin/bash
cd $(dirname $0)/../..
O=gpurun_out/shard; mkdir -p $O
for w in cfg4 cfg5b; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 1 --steps 10 --warmup 3 --shard $w > $O/shard_$w.json 2> $O/shard_$w.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus 1 --steps 20 --warmup 5 > $O/torchrun_default.json 2> $O/torchrun_default.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/reference.json 2> $O/reference.err
