#!/bin/bash
mkdir -p gpurun_out
MODE=cast bash tools/sweep.sh 'run ffma2' 'run fma FGL_LIB=build_ab/libfgl_noffma2.so' 'run ffma2_b' 'run fma_b FGL_LIB=build_ab/libfgl_noffma2.so' > gpurun_out/r03_ffma2.txt 2>&1
BENCH_ARGS="--config C5 --poses 256" MODE=cast bash tools/sweep.sh 'run c5ffma2' 'run c5fma FGL_LIB=build_ab/libfgl_noffma2.so' >> gpurun_out/r03_ffma2.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_cast.py tests/test_gpu_parity_coverage.py -m gpu -x -q >> gpurun_out/r03_ffma2.txt 2>&1
