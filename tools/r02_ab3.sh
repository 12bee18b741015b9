MODE=cast bash tools/sweep.sh 'run pf0 FGL_LIB=build_ab/libfgl_pf0.so' 'run pf1' 'run pf2 FGL_LIB=build_ab/libfgl_pf2.so' 'run pf0b FGL_LIB=build_ab/libfgl_pf0.so' 'run pf1b' > gpurun_out/r02_ab3.txt 2>&1
BENCH_ARGS="--config C5 --poses 256" MODE=cast bash tools/sweep.sh 'run c5pf0 FGL_LIB=build_ab/libfgl_pf0.so' 'run c5pf1' 'run c5pf2 FGL_LIB=build_ab/libfgl_pf2.so' >> gpurun_out/r02_ab3.txt 2>&1
bash tools/ncu_cast.sh pf1 > gpurun_out/r02_ncu_pf1.txt 2>&1
