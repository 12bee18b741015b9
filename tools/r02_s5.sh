MODE=cast bash tools/sweep.sh 'run top' 'run notop FGL_LIB=build_ab/libfgl_notop.so' 'run top2' 'run notop2 FGL_LIB=build_ab/libfgl_notop.so' > gpurun_out/r02_s5_sweep.txt 2>&1
BENCH_ARGS="--config C5 --poses 256" MODE=cast bash tools/sweep.sh 'run c5top' 'run c5notop FGL_LIB=build_ab/libfgl_notop.so' >> gpurun_out/r02_s5_sweep.txt 2>&1
bash tools/ncu_cast.sh top > gpurun_out/r02_ncu_top.txt 2>&1
