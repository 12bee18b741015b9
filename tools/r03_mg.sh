#!/bin/bash
# N = 2 bench path on one GPU with the gloo backend and the collective gather (no device-side
# waits between the two processes' kernels): checks the sharded step and the W=1 vs W=N gather check
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --dist-backend gloo --gather nccl --steps 3 --warmup 3 --no-e2e --no-cpu --no-latency > gpurun_out/r03_mg_nccl.json 2> gpurun_out/r03_mg_nccl.err
