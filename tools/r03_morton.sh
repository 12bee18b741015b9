#!/bin/bash
mkdir -p gpurun_out
L="paper_2509_17390_b200/libfgl.so build_ab/libfgl_mo2.so build_ab/libfgl_mo1.so"
timeout 300 bash tools/build_ms.sh $L > gpurun_out/r03_morton.txt 2>&1
SCENE=terrain timeout 300 bash tools/build_ms.sh $L >> gpurun_out/r03_morton.txt 2>&1
