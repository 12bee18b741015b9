MODE=cast bash tools/sweep.sh 'run hand' 'run nohand FGL_LIB=build_ab/libfgl_nohand.so' 'run hand2' 'run nohand2 FGL_LIB=build_ab/libfgl_nohand.so' > gpurun_out/r02_s3_sweep.txt 2>&1
bash tools/ncu_cast.sh hand > gpurun_out/r02_ncu_hand.txt 2>&1
FGL_LIB=build_ab/libfgl_nohand.so bash tools/ncu_cast.sh nohand > gpurun_out/r02_ncu_nohand.txt 2>&1
