MODE=cast bash tools/sweep.sh 'run hand' 'run nohand FGL_LIB=build_ab/libfgl_nohand.so' 'run hand2' > gpurun_out/r02_s2_sweep.txt 2>&1
MODE=full bash tools/sweep.sh 'run fused' 'run nofuse FGL_LIB=build_ab/libfgl_nofuse.so' >> gpurun_out/r02_s2_sweep.txt 2>&1
BENCH_ARGS="--config C3" MODE=full bash tools/sweep.sh 'run c3fused' 'run c3nofuse FGL_LIB=build_ab/libfgl_nofuse.so' >> gpurun_out/r02_s2_sweep.txt 2>&1
BENCH_ARGS="--config C5 --poses 256" MODE=cast bash tools/sweep.sh 'run c5hand' 'run c5nohand FGL_LIB=build_ab/libfgl_nohand.so' >> gpurun_out/r02_s2_sweep.txt 2>&1
bash tools/ncu_cast.sh hand > gpurun_out/r02_ncu_hand.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_cast.py -x -q > gpurun_out/r02_s2_tests.txt 2>&1
