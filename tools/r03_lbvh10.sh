#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_graph_replay.py tests/test_gpu_refit.py -m gpu -x -q > gpurun_out/r03_lbvh10_tests.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r03_lbvh10_tests.txt
L="paper_2509_17390_b200/libfgl.so build_ab/libfgl_win16.so build_ab/libfgl_win32.so"
SCENE=terrain timeout 300 bash tools/build_ms.sh $L > gpurun_out/r03_lbvh10_build_ms.txt 2>&1
timeout 300 bash tools/build_ms.sh $L >> gpurun_out/r03_lbvh10_build_ms.txt 2>&1
timeout 600 bash tools/ncu_build.sh lbvh10
