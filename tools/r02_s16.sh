SCENE=terrain bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so build_ab/libfgl_nort.so > gpurun_out/r02_s16_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_cast.py -x -q -k "sort or c3 or c5 or build" > gpurun_out/r02_s16_tests.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_C3rts.csv python bench.py --config C3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-latency > /dev/null 2>&1
python tools/launches.py gpurun_out/r02_launches_C3rts.csv > gpurun_out/r02_launches_C3rts.txt 2>&1
