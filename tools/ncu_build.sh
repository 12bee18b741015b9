#!/bin/bash
# ncu --set full of every build kernel of one warm terrain (C3, 10 M tris) build (run under gpurun).
# usage: tools/ncu_build.sh <tag>   -> gpurun_out/ncu_build_<tag>.ncu-rep
tag=${1:-build}
cat > /tmp/ncu_build_driver.py <<'PY'
import torch, synth, paper_2509_17390_b200 as fgl
m = synth.scene_terrain(3).mesh
v = torch.from_numpy(m.verts).cuda(); t = torch.from_numpy(m.tris).cuda()
s = fgl.Scene(v, t)
s.build(); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
s.build(); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
PY
ncu --set full --clock-control none --import-source on --profile-from-start off -f \
    -o gpurun_out/ncu_build_$tag env PYTHONPATH=$PWD python /tmp/ncu_build_driver.py > gpurun_out/ncu_build_$tag.log 2>&1
