#!/bin/bash
# Round measurement session (run under gpurun): launch lists + one --set full capture of the cast
# kernel per config, and a bench line per config. Outputs land in gpurun_out/.
set -x
TAG=${TAG:-r01}
for cfg in C2 C3; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
      --log-file gpurun_out/${TAG}_launches_${cfg}.csv python bench.py --config $cfg --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_cast -s 2 -c 1 \
      -o gpurun_out/${TAG}_k_cast_${cfg} python bench.py --config $cfg --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"k_onesweep|k_reorder_refit|k_karras" -s 12 -c 3 \
    -o gpurun_out/${TAG}_build_C2 python bench.py --config C2 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
# the C3 (10 M triangles) build, every kernel once, and the G2 voxelizer (NEXT-2)
bash tools/ncu_build.sh c3 && mv gpurun_out/ncu_build_c3.ncu-rep gpurun_out/${TAG}_build_C3.ncu-rep
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/${TAG}_launches_G2.csv python bench.py --config G2 --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_voxelize|k_masks" -s 4 -c 2 \
    -o gpurun_out/${TAG}_vox_G2 python bench.py --config G2 --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph > /dev/null 2>&1
for cfg in C1 C2 C3 C4 C5 G1 G2; do
  python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 >> gpurun_out/${TAG}_configs.jsonl
done
