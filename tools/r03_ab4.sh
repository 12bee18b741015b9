#!/bin/bash
mkdir -p gpurun_out
timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so > gpurun_out/r03_ab4.txt 2>&1
FGL_SORT_RTS_MIN=0 timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so >> gpurun_out/r03_ab4.txt 2>&1
SCENE=terrain FGL_SORT_RTS_MIN=0 timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so >> gpurun_out/r03_ab4.txt 2>&1
FGL_SORT_RTS_MIN=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' --csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-latency > gpurun_out/r03_ab4_launches_rts.csv 2>/dev/null
