python tools/simt_tail.py > gpurun_out/r02_simt_tail.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_cast_dyn -s 3 -c 1 -o gpurun_out/r02_cast_full python bench.py --mode cast --steps 1 --warmup 2 --no-e2e --no-cpu --no-latency > gpurun_out/r02_cast_full.log 2>&1
