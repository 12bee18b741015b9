#!/bin/bash
mkdir -p gpurun_out
L="paper_2509_17390_b200/libfgl.so build_ab/libfgl_c128.so build_ab/libfgl_m8.so"
SCENE=terrain timeout 300 bash tools/build_ms.sh $L > gpurun_out/r03_ab2_build_ms.txt 2>&1
timeout 300 bash tools/build_ms.sh $L >> gpurun_out/r03_ab2_build_ms.txt 2>&1
FGL_LIB=build_ab/libfgl_m8.so timeout 600 bash tools/ncu_build.sh m8
