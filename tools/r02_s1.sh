python tools/raygen_err.py > gpurun_out/r02_raygen_err.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_cast.py tests/test_gpu_wide.py tests/test_gpu_refit.py -x -q > gpurun_out/r02_s1_tests.txt 2>&1
MODE=cast bash tools/sweep.sh 'run noexp' 'run noexp2' > gpurun_out/r02_s1_sweep.txt 2>&1
BENCH_ARGS="--config C5 --poses 256" MODE=cast bash tools/sweep.sh 'run c5noexp' >> gpurun_out/r02_s1_sweep.txt 2>&1
bash tools/ncu_cast.sh noexp > gpurun_out/r02_ncu_noexp.txt 2>&1
