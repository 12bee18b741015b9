#!/bin/bash
mkdir -p gpurun_out
MODE=full bash tools/sweep.sh 'run plain' 'run t1 -- --treelets 1 --leaf-size 1' 'run t1_tm8 FGL_LIB=build_ab/libfgl_tm8.so -- --treelets 1 --leaf-size 1' 'run t1_tm32 FGL_LIB=build_ab/libfgl_tm32.so -- --treelets 1 --leaf-size 1' 'run t2_tm8 FGL_LIB=build_ab/libfgl_tm8.so -- --treelets 1' 'run t2_tm32 FGL_LIB=build_ab/libfgl_tm32.so -- --treelets 1' > gpurun_out/r03_ab6.txt 2>&1
