bash tools/build_ms.sh build_ab/libfgl_rbstatic.so build_ab/libfgl_rbdyn.so build_ab/libfgl_rbdyn_fused.so > gpurun_out/r02_s7_build.txt 2>&1
SCENE=terrain bash tools/build_ms.sh build_ab/libfgl_rbstatic.so build_ab/libfgl_rbdyn.so build_ab/libfgl_rbdyn_fused.so >> gpurun_out/r02_s7_build.txt 2>&1
FGL_LIB=build_ab/libfgl_rbdyn_fused.so timeout 600 python -m pytest tests/test_gpu_build.py -x -q > gpurun_out/r02_s7_tests.txt 2>&1
