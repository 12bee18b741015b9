for g in fused nccl; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2952$([ $g = fused ] && echo 1 || echo 2) bench.py --gpus 2 --dist-backend gloo --gather $g --steps 3 --warmup 3 --no-e2e --no-cpu --no-latency > gpurun_out/r02_mg_$g.json 2> gpurun_out/r02_mg_$g.err
done
