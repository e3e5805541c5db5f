#!/bin/bash
# the N>1 launch path (torchrun, per-rank user shards, max/sum reductions) on a one-GPU box:
# two ranks share GPU 0 with gloo reductions (functional check, not a scaling number)
MTKV_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --steps 6 --warmup 3 --users 256 > gpurun_out/torchrun2.log 2>&1
