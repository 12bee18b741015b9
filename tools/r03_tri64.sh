#!/bin/bash
mkdir -p gpurun_out
MODE=cast bash tools/sweep.sh 'run base' 'run tri64 FGL_LIB=build_ab/libfgl_tri64.so' 'run base_b' 'run tri64_b FGL_LIB=build_ab/libfgl_tri64.so' > gpurun_out/r03_tri64.txt 2>&1
BENCH_ARGS="--config C5 --poses 256" MODE=cast bash tools/sweep.sh 'run c5base' 'run c5tri64 FGL_LIB=build_ab/libfgl_tri64.so' >> gpurun_out/r03_tri64.txt 2>&1
MODE=full bash tools/sweep.sh 'run fullbase' 'run fulltri64 FGL_LIB=build_ab/libfgl_tri64.so' >> gpurun_out/r03_tri64.txt 2>&1
FGL_LIB=build_ab/libfgl_tri64.so timeout 900 python -m pytest tests/test_gpu_cast.py tests/test_gpu_build.py tests/test_gpu_metrics.py -m gpu -x -q >> gpurun_out/r03_tri64.txt 2>&1
