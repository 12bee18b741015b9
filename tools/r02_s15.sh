L="paper_2509_17390_b200/libfgl.so build_ab/libfgl_FGL_SORT_MINB_2.so build_ab/libfgl_FGL_SORT_MINB_3.so build_ab/libfgl_FGL_SORT_WIN_4.so build_ab/libfgl_FGL_SORT_BACKOFF_100.so"
bash tools/build_ms.sh $L > gpurun_out/r02_s15_build.txt 2>&1
SCENE=terrain bash tools/build_ms.sh $L >> gpurun_out/r02_s15_build.txt 2>&1
