#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_graph_replay.py tests/test_gpu_refit.py -m gpu -x -q > gpurun_out/r03_lbvh9_tests.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r03_lbvh9_tests.txt
SCENE=terrain timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so > gpurun_out/r03_lbvh9_build_ms.txt 2>&1
timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so >> gpurun_out/r03_lbvh9_build_ms.txt 2>&1
MODE=full bash tools/sweep.sh 'run plain' 'run treelets -- --treelets 1' 'run t_leaf1 -- --treelets 1 --leaf-size 1' > gpurun_out/r03_lbvh9_sweep.txt 2>&1
timeout 600 bash tools/ncu_build.sh lbvh9
