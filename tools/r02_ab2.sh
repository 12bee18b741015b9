MODE=cast bash tools/sweep.sh 'run ss0 FGL_LIB=build_ab/libfgl_ss0.so' 'run ss4 FGL_LIB=build_ab/libfgl_ss4.so' 'run ss6' 'run ss8 FGL_LIB=build_ab/libfgl_ss8.so' 'run ss12 FGL_LIB=build_ab/libfgl_ss12.so' 'run ss16 FGL_LIB=build_ab/libfgl_ss16.so' > gpurun_out/r02_ab2.txt 2>&1
BENCH_ARGS="--config C5 --poses 256" MODE=cast bash tools/sweep.sh 'run c5ss0 FGL_LIB=build_ab/libfgl_ss0.so' 'run c5ss6' 'run c5ss8 FGL_LIB=build_ab/libfgl_ss8.so' >> gpurun_out/r02_ab2.txt 2>&1
bash tools/ncu_cast.sh ss6 > gpurun_out/r02_ncu_ss6.txt 2>&1
