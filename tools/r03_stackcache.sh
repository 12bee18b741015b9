#!/bin/bash
mkdir -p gpurun_out
MODE=cast bash tools/sweep.sh 'run base' 'run c1 FGL_LIB=build_ab/libfgl_c1.so' 'run c2 FGL_LIB=build_ab/libfgl_c2.so' 'run c1m9 FGL_LIB=build_ab/libfgl_c1m9.so' 'run c2m9 FGL_LIB=build_ab/libfgl_c2m9.so' 'run base_b' > gpurun_out/r03_stackcache.txt 2>&1
