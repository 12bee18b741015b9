set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err
timeout 3000 python -m pytest tests -m gpu -q -x --durations=30 > gpurun_out/r02_gpu_tests.txt 2>&1
bash tools/r02_profile.sh
