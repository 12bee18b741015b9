#!/bin/bash
mkdir -p gpurun_out
L="paper_2509_17390_b200/libfgl.so build_ab/libfgl_c256.so build_ab/libfgl_unfused.so"
SCENE=terrain timeout 300 bash tools/build_ms.sh $L > gpurun_out/r03_ab1_build_ms.txt 2>&1
timeout 300 bash tools/build_ms.sh $L >> gpurun_out/r03_ab1_build_ms.txt 2>&1
FGL_LIB=build_ab/libfgl_c256.so timeout 600 python -m pytest tests/test_gpu_build.py -m gpu -x -q -k "fused or rooms or matches_oracle" > gpurun_out/r03_ab1_c256_tests.txt 2>&1; echo "rc $?" >> gpurun_out/r03_ab1_c256_tests.txt
