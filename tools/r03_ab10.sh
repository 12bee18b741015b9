#!/bin/bash
mkdir -p gpurun_out
MODE=full bash tools/sweep.sh 'run plain' 'run t1 -- --treelets 1 --leaf-size 1' 'run t1_tl5 FGL_LIB=build_ab/libfgl_tl5.so -- --treelets 1 --leaf-size 1' 'run t2 -- --treelets 1' > gpurun_out/r03_ab10.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_refit.py -m gpu -x -q -k treelets >> gpurun_out/r03_ab10.txt 2>&1
