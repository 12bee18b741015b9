#!/bin/bash
# k_lbvh + k_lbvh_top (fused width-2 build), optional in-build treelets: tests, timing, bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_graph_replay.py tests/test_gpu_refit.py -m gpu -x -q > gpurun_out/r03_lbvh2_tests.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r03_lbvh2_tests.txt
SCENE=terrain timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so > gpurun_out/r03_lbvh2_build_ms.txt 2>&1
timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so >> gpurun_out/r03_lbvh2_build_ms.txt 2>&1
MODE=full bash tools/sweep.sh 'run plain' 'run treelets -- --treelets 1' > gpurun_out/r03_lbvh2_sweep.txt 2>&1
BENCH_ARGS="--config C3" MODE=full bash tools/sweep.sh 'run c3plain' 'run c3treelets -- --treelets 1' >> gpurun_out/r03_lbvh2_sweep.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' --csv python bench.py --config C3 --steps 1 --warmup 0 --no-cpu --no-e2e --no-latency > gpurun_out/r03_lbvh2_launches_C3.csv 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' --csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-latency --treelets 1 > gpurun_out/r03_lbvh2_launches_C2T.csv 2>/dev/null
