#!/bin/bash
# Round-2 measurement session (run under gpurun): ncu --set full of the cast kernel per config,
# launch lists, the C3 build kernels, compute-sanitizer, bench lines per config and the layout A/B.
TAG=${TAG:-r02}
for spec in "C2:" "C3:" "C4:--poses 20" "C5:--poses 256"; do
  cfg=${spec%%:*}; extra=${spec#*:}
  ncu --set full --clock-control none --import-source on -k regex:k_cast_dyn -s 2 -c 1 \
      -o gpurun_out/${TAG}_k_cast_${cfg} python bench.py --config $cfg $extra --mode cast --steps 1 --warmup 1 --no-e2e --no-cpu --no-latency > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
      --log-file gpurun_out/${TAG}_launches_${cfg}.csv python bench.py --config $cfg $extra --steps 1 --warmup 1 --no-e2e --no-cpu --no-latency > /dev/null 2>&1
done
bash tools/ncu_build.sh c3 && mv gpurun_out/ncu_build_c3.ncu-rep gpurun_out/${TAG}_build_C3.ncu-rep
for tool in memcheck racecheck synccheck; do
  echo "== compute-sanitizer --tool $tool python tools/sanitize.py" >> gpurun_out/${TAG}_sanitizer.txt
  timeout 1200 compute-sanitizer --tool $tool python tools/sanitize.py 2>&1 | grep -E "done|SUMMARY|ERROR|Invalid|hazard" | head -20 >> gpurun_out/${TAG}_sanitizer.txt
done
for spec in "C1:" "C2:" "C3:" "C4:" "C5:" "C2:--width 8" "C2:--width 4" "C2:--width 4 --quantized 1" "C2:--restructure 3 --mode cast" "C2:--mode refit"; do
  cfg=${spec%%:*}; extra=${spec#*:}
  python bench.py --config $cfg $extra --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 >> gpurun_out/${TAG}_configs.jsonl
done
