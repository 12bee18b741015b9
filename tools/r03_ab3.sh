#!/bin/bash
mkdir -p gpurun_out
L="paper_2509_17390_b200/libfgl.so build_ab/libfgl_it16.so"
SCENE=terrain timeout 300 bash tools/build_ms.sh $L > gpurun_out/r03_ab3_build_ms.txt 2>&1
timeout 300 bash tools/build_ms.sh $L >> gpurun_out/r03_ab3_build_ms.txt 2>&1
for i in 1 2; do
MODE=full bash tools/sweep.sh 'run plain' 'run t_leaf1 -- --treelets 1 --leaf-size 1' 'run t_leaf2 -- --treelets 1' >> gpurun_out/r03_ab3_sweep.txt 2>&1
done
