MODE=cast bash tools/sweep.sh 'run base' 'run flat FGL_LIB=build_ab/libfgl_flat.so' 'run base2' 'run flat2 FGL_LIB=build_ab/libfgl_flat.so' > gpurun_out/r02_s19_sweep.txt 2>&1
BENCH_ARGS="--config C5 --poses 256" MODE=cast bash tools/sweep.sh 'run c5base' 'run c5flat FGL_LIB=build_ab/libfgl_flat.so' >> gpurun_out/r02_s19_sweep.txt 2>&1
FGL_LIB=build_ab/libfgl_flat.so bash tools/ncu_cast.sh flat > gpurun_out/r02_ncu_flat.txt 2>&1
