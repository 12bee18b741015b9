set -x
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --dist-backend gloo --gather fused --steps 3 --warmup 3 --no-e2e --no-cpu --no-latency > gpurun_out/r02_mg_fused.json 2> gpurun_out/r02_mg_fused.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --dist-backend gloo --gather nccl --steps 3 --warmup 3 --no-e2e --no-cpu --no-latency > gpurun_out/r02_mg_nccl.json 2> gpurun_out/r02_mg_nccl.err
start=$(date +%s); timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/r02_gpu_tests.txt 2>&1; echo "elapsed $(( $(date +%s) - start )) s" >> gpurun_out/r02_gpu_tests.txt
