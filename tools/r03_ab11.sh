#!/bin/bash
mkdir -p gpurun_out
MODE=cast bash tools/sweep.sh 'run base' 'run unroll3 FGL_LIB=build_ab/libfgl_unroll3.so' 'run mb12 FGL_LIB=build_ab/libfgl_mb12.so' 'run mb8 FGL_LIB=build_ab/libfgl_mb8.so' 'run t256 FGL_LIB=build_ab/libfgl_t256.so' 'run base_b' > gpurun_out/r03_ab11.txt 2>&1
