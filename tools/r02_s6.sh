bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so build_ab/libfgl_FGL_SORT_WIN_16.so build_ab/libfgl_FGL_SORT_ITEMS_K_6.so > gpurun_out/r02_s6_build.txt 2>&1
SCENE=terrain bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so build_ab/libfgl_FGL_SORT_WIN_16.so build_ab/libfgl_FGL_SORT_ITEMS_K_6.so >> gpurun_out/r02_s6_build.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_C2.csv python bench.py --config C2 --steps 1 --warmup 1 --no-e2e --no-cpu --no-latency > /dev/null 2>&1
python tools/launches.py gpurun_out/r02_launches_C2.csv > gpurun_out/r02_launches_C2.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_C3.csv python bench.py --config C3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-latency > /dev/null 2>&1
python tools/launches.py gpurun_out/r02_launches_C3.csv > gpurun_out/r02_launches_C3.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_w8.csv python bench.py --width 8 --steps 1 --warmup 1 --no-e2e --no-cpu --no-latency > /dev/null 2>&1
python tools/launches.py gpurun_out/r02_launches_w8.csv > gpurun_out/r02_launches_w8.txt 2>&1
bash tools/ncu_build.sh r02c3
