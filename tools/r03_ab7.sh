#!/bin/bash
mkdir -p gpurun_out
FGL_LIB=build_ab/libfgl_ord.so timeout 900 python -m pytest tests/test_gpu_build.py -m gpu -x -q > gpurun_out/r03_ab7_tests.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r03_ab7_tests.txt
L="paper_2509_17390_b200/libfgl.so build_ab/libfgl_ord.so"
SCENE=terrain timeout 300 bash tools/build_ms.sh $L > gpurun_out/r03_ab7.txt 2>&1
timeout 300 bash tools/build_ms.sh $L >> gpurun_out/r03_ab7.txt 2>&1
FGL_LIB=build_ab/libfgl_ord.so timeout 600 bash tools/ncu_build.sh ord
