bash tools/build_ms.sh build_ab/libfgl_r01.so build_ab/libfgl_head.so build_ab/libfgl_nofusecode.so > gpurun_out/r02_s8_build.txt 2>&1
SCENE=terrain bash tools/build_ms.sh build_ab/libfgl_r01.so build_ab/libfgl_head.so build_ab/libfgl_nofusecode.so >> gpurun_out/r02_s8_build.txt 2>&1
