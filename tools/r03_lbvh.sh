#!/bin/bash
# k_lbvh (fused width-2 build) check: build tests, graph replay, refit, cast parity; build timing C2/C3; bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_graph_replay.py tests/test_gpu_refit.py tests/test_gpu_cast.py -m gpu -x -q > gpurun_out/r03_lbvh_tests.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r03_lbvh_tests.txt
SCENE=terrain timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so > gpurun_out/r03_lbvh_build_ms.txt 2>&1
timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so >> gpurun_out/r03_lbvh_build_ms.txt 2>&1
timeout 300 python bench.py --no-cpu --no-latency > gpurun_out/r03_lbvh_bench.json 2> gpurun_out/r03_lbvh_bench.err
timeout 300 python bench.py --config C3 --no-cpu --no-e2e --no-latency > gpurun_out/r03_lbvh_bench_C3.json 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' --csv python bench.py --config C3 --steps 1 --warmup 0 --no-cpu --no-e2e --no-latency > gpurun_out/r03_lbvh_launches_C3.csv 2>/dev/null
