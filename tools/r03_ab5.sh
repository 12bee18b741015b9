#!/bin/bash
mkdir -p gpurun_out
L="paper_2509_17390_b200/libfgl.so build_ab/libfgl_g4.so build_ab/libfgl_g16.so"
SCENE=terrain timeout 300 bash tools/build_ms.sh $L > gpurun_out/r03_ab5.txt 2>&1
timeout 300 bash tools/build_ms.sh $L >> gpurun_out/r03_ab5.txt 2>&1
