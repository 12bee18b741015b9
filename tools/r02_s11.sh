FGL_LIB=build_ab/libfgl_FGL_APPROX_NORM_1.so python tools/raygen_err.py > gpurun_out/r02_s11_raygen.txt 2>&1
MODE=cast bash tools/sweep.sh 'run base' 'run norm FGL_LIB=build_ab/libfgl_FGL_APPROX_NORM_1.so' 'run normunroll FGL_LIB=build_ab/libfgl_norm_unroll.so' 'run base2' 'run norm2 FGL_LIB=build_ab/libfgl_FGL_APPROX_NORM_1.so' 'run normunroll2 FGL_LIB=build_ab/libfgl_norm_unroll.so' > gpurun_out/r02_s11_sweep.txt 2>&1
BENCH_ARGS="--config C4" MODE=cast bash tools/sweep.sh 'run c4base' 'run c4norm FGL_LIB=build_ab/libfgl_FGL_APPROX_NORM_1.so' 'run c4normunroll FGL_LIB=build_ab/libfgl_norm_unroll.so' >> gpurun_out/r02_s11_sweep.txt 2>&1
BENCH_ARGS="--restructure 3" MODE=cast bash tools/sweep.sh 'run restr3' 'run restr3norm FGL_LIB=build_ab/libfgl_FGL_APPROX_NORM_1.so' >> gpurun_out/r02_s11_sweep.txt 2>&1
BENCH_ARGS="--restructure 1" MODE=cast bash tools/sweep.sh 'run restr1' >> gpurun_out/r02_s11_sweep.txt 2>&1
