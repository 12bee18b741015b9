for k in -2 -4 -6; do BENCH_ARGS="--restructure $k" MODE=full bash tools/sweep.sh "run t4_$k"; done > gpurun_out/r02_s17_sweep.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_t4b.csv python bench.py --restructure -4 --steps 1 --warmup 1 --no-e2e --no-cpu --no-latency > /dev/null 2>&1
python tools/launches.py gpurun_out/r02_launches_t4b.csv > gpurun_out/r02_launches_t4b.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_refit.py tests/test_gpu_build.py tests/test_gpu_wide.py -x -q > gpurun_out/r02_s17_tests.txt 2>&1
