#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lbvh -c 2 -f -o gpurun_out/r03_lbvh_tl python bench.py --treelets 1 --leaf-size 1 --steps 1 --warmup 0 --no-cpu --no-e2e --no-latency > gpurun_out/r03_prof_tl.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lbvh -c 2 -f -o gpurun_out/r03_lbvh_plain python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-latency >> gpurun_out/r03_prof_tl.log 2>&1
