MODE=cast bash tools/sweep.sh 'run cur' 'run cur2' > gpurun_out/r02_s4_sweep.txt 2>&1
BENCH_ARGS="--config C5 --poses 256" MODE=cast bash tools/sweep.sh 'run c5cur' >> gpurun_out/r02_s4_sweep.txt 2>&1
BENCH_ARGS="--config C4" MODE=cast bash tools/sweep.sh 'run c4cur' >> gpurun_out/r02_s4_sweep.txt 2>&1
bash tools/ncu_cast.sh cur > gpurun_out/r02_ncu_cur.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_cast.py tests/test_gpu_wide.py tests/test_gpu_refit.py tests/test_gpu_build.py tests/test_gpu_graph_replay.py tests/test_gpu_peer_gather.py -x -q > gpurun_out/r02_s4_tests.txt 2>&1
