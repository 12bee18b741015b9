#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_graph_replay.py -m gpu -x -q > gpurun_out/r03_prep_tests.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r03_prep_tests.txt
SCENE=terrain timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so > gpurun_out/r03_prep_build_ms.txt 2>&1
timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so >> gpurun_out/r03_prep_build_ms.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r03_prep_launches_C2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-latency > /dev/null 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu --no-latency > gpurun_out/r03_prep_bench.json 2>/dev/null
