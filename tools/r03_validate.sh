#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_cast.py -m gpu -q -k "error or valid or upload or async or matches_oracle or rooms" > gpurun_out/r03_validate_tests.txt 2>&1; echo "rc $?" >> gpurun_out/r03_validate_tests.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r03_validate_launches_C2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-latency > /dev/null 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu --no-latency > gpurun_out/r03_validate_bench.json 2>/dev/null
