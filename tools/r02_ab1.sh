set -x
MODE=cast bash tools/sweep.sh 'run new' 'run div FGL_LIB=build_ab/libfgl_div.so' 'run new2' > gpurun_out/r02_ab1.txt 2>&1
python -m pytest tests/test_gpu_graph_replay.py tests/test_gpu_cast.py -x -q > gpurun_out/r02_ab1_tests.txt 2>&1
bash tools/ncu_cast.sh new > gpurun_out/r02_ncu_new.txt 2>&1
