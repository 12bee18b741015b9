#!/bin/bash
# Round-3 measurement session (run under gpurun): ncu --set full of the cast kernel per config
# (after the FFMA2 slab test), launch lists, the C3 build kernels, bench lines per config.
mkdir -p gpurun_out
TAG=${TAG:-r03}
for spec in "C2:" "C3:" "C4:--poses 20" "C5:--poses 256"; do
  cfg=${spec%%:*}; extra=${spec#*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cast_dyn -s 2 -c 1 \
      -o gpurun_out/${TAG}_k_cast_${cfg} python bench.py --config $cfg $extra --mode cast --steps 1 --warmup 1 --no-e2e --no-cpu --no-latency > /dev/null 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
      --log-file gpurun_out/${TAG}_launches_${cfg}.csv python bench.py --config $cfg $extra --steps 1 --warmup 1 --no-e2e --no-cpu --no-latency > /dev/null 2>&1
done
timeout 600 bash tools/ncu_build.sh c3 && mv gpurun_out/ncu_build_c3.ncu-rep gpurun_out/${TAG}_build_C3.ncu-rep
rm -f gpurun_out/${TAG}_configs.jsonl
for spec in "C1:" "C2:" "C3:" "C4:" "C5:" "C2:--mode refit" "C2:--treelets 1 --leaf-size 1" "C2:--restructure -4 --mode cast"; do
  cfg=${spec%%:*}; extra=${spec#*:}
  timeout 400 python bench.py --config $cfg $extra --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 >> gpurun_out/${TAG}_configs.jsonl
done
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err
