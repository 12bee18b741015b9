#!/bin/bash
mkdir -p gpurun_out
MODE=cast bash tools/sweep.sh 'run base' 'run pairleaf FGL_LIB=build_ab/libfgl_pairleaf.so' 'run base_b' 'run pairleaf_b FGL_LIB=build_ab/libfgl_pairleaf.so' > gpurun_out/r03_pairleaf.txt 2>&1
