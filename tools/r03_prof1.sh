#!/bin/bash
mkdir -p gpurun_out
SCENE=terrain timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so build_ab/libfgl_c256.so > gpurun_out/r03_prof1_build_ms.txt 2>&1
timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so build_ab/libfgl_c256.so >> gpurun_out/r03_prof1_build_ms.txt 2>&1
timeout 600 bash tools/ncu_build.sh lbvh
