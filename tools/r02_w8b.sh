timeout 900 python -m pytest tests/test_gpu_wide.py -x -q > gpurun_out/r02_w8b_tests.txt 2>&1
BENCH_ARGS="--width 8" MODE=cast bash tools/sweep.sh 'run w8mb8' 'run w8mb6 FGL_LIB=build_ab/libfgl_w8mb6.so' 'run w8mb10 FGL_LIB=build_ab/libfgl_w8mb10.so' > gpurun_out/r02_w8b_sweep.txt 2>&1
BENCH_ARGS="--leaf-size 1" MODE=cast bash tools/sweep.sh 'run leaf1' >> gpurun_out/r02_w8b_sweep.txt 2>&1
BENCH_ARGS="--leaf-size 3" MODE=cast bash tools/sweep.sh 'run leaf3' >> gpurun_out/r02_w8b_sweep.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02_launches_w8.csv python bench.py --width 8 --steps 1 --warmup 1 --no-e2e --no-cpu --no-latency > /dev/null 2>&1
python tools/launches.py gpurun_out/r02_launches_w8.csv > gpurun_out/r02_launches_w8.txt 2>&1
