set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_base_default.json 2> gpurun_out/r02_base_default.err
MODE=cast bash tools/sweep.sh 'run bvh2' 'run bvh4 -- ' > gpurun_out/r02_base_sweep.txt 2>&1
BENCH_ARGS="--width 4" MODE=cast bash tools/sweep.sh 'run w4' >> gpurun_out/r02_base_sweep.txt 2>&1
BENCH_ARGS="--width 4 --quantized 1" MODE=cast bash tools/sweep.sh 'run w4q' >> gpurun_out/r02_base_sweep.txt 2>&1
BENCH_ARGS="--restructure 3" MODE=cast bash tools/sweep.sh 'run restr3' >> gpurun_out/r02_base_sweep.txt 2>&1
bash tools/ncu_cast.sh base > gpurun_out/r02_ncu_base.txt 2>&1
