for k in -2 -4 -6 -8; do BENCH_ARGS="--restructure $k" MODE=full bash tools/sweep.sh "run t4_$k"; done > gpurun_out/r02_s14_sweep.txt 2>&1
BENCH_ARGS="--restructure -6" MODE=full bash tools/sweep.sh "run t8_-6 FGL_LIB=build_ab/libfgl_t8.so" >> gpurun_out/r02_s14_sweep.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_t4.csv python bench.py --restructure -4 --steps 1 --warmup 1 --no-e2e --no-cpu --no-latency > /dev/null 2>&1
python tools/launches.py gpurun_out/r02_launches_t4.csv > gpurun_out/r02_launches_t4.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_refit.py -x -q > gpurun_out/r02_s14_tests.txt 2>&1
