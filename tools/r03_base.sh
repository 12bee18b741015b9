#!/bin/bash
# Session-3 baseline on the current HEAD: GPU tests, default bench, C3 bench line, build timing.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r03_gputest.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r03_gputest.txt
timeout 300 python bench.py > gpurun_out/r03_bench.json 2> gpurun_out/r03_bench.err
timeout 300 python bench.py --config C3 --no-cpu --no-e2e > gpurun_out/r03_bench_C3.json 2>/dev/null
SCENE=terrain timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so > gpurun_out/r03_build_ms.txt 2>&1
