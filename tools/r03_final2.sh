#!/bin/bash
mkdir -p gpurun_out
TAG=r03f
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err
rm -f gpurun_out/${TAG}_configs.jsonl
for cfg in C1 C2 C3 C4 C5; do
  timeout 400 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 >> gpurun_out/${TAG}_configs.jsonl
done
timeout 400 python bench.py --mode refit --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 >> gpurun_out/${TAG}_configs.jsonl
timeout 400 python bench.py --treelets 1 --leaf-size 1 --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 >> gpurun_out/${TAG}_configs.jsonl
for cfg in C2 C3; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
      --log-file gpurun_out/${TAG}_launches_${cfg}.csv python bench.py --config $cfg --steps 1 --warmup 1 --no-e2e --no-cpu --no-latency > /dev/null 2>&1
done
timeout 600 bash tools/ncu_build.sh c3f && mv gpurun_out/ncu_build_c3f.ncu-rep gpurun_out/${TAG}_build_C3.ncu-rep
