#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_graph_replay.py tests/test_gpu_refit.py -m gpu -x -q > gpurun_out/r03_lbvh12_tests.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r03_lbvh12_tests.txt
SCENE=terrain timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so > gpurun_out/r03_lbvh12_build_ms.txt 2>&1
timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so >> gpurun_out/r03_lbvh12_build_ms.txt 2>&1
timeout 600 bash tools/ncu_build.sh lbvh12
