timeout 900 python -m pytest tests/test_gpu_wide.py -x -q > gpurun_out/r02_w8_tests.txt 2>&1
MODE=cast bash tools/sweep.sh 'run w2' > gpurun_out/r02_w8_sweep.txt 2>&1
BENCH_ARGS="--width 8" MODE=cast bash tools/sweep.sh 'run w8' >> gpurun_out/r02_w8_sweep.txt 2>&1
BENCH_ARGS="--width 8" MODE=full bash tools/sweep.sh 'run w8full' >> gpurun_out/r02_w8_sweep.txt 2>&1
BENCH_ARGS="--config C5 --poses 256 --width 8" MODE=cast bash tools/sweep.sh 'run c5w8' >> gpurun_out/r02_w8_sweep.txt 2>&1
bash tools/ncu_cast.sh w8 --width 8 > gpurun_out/r02_ncu_w8.txt 2>&1
