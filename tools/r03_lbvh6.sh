#!/bin/bash
mkdir -p gpurun_out
cat > /tmp/memchk.py <<'PY'
import synth, numpy as np, paper_2509_17390_b200 as fgl, os
for T in (1292, 70001):
    m = synth.scene_c1() if T == 1292 else synth.soup(T, seed=3)
    for tl in (0, 1):
        s = fgl.Scene(m.verts, m.tris, treelets=tl); s.export()
os.environ["FGL_LBVH_GLOBAL"] = "1"
m = synth.soup(70001, seed=3); fgl.Scene(m.verts, m.tris).export()
print("memcheck driver ok")
PY
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python /tmp/memchk.py > gpurun_out/r03_lbvh6_memcheck.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_graph_replay.py tests/test_gpu_refit.py -m gpu -x -q > gpurun_out/r03_lbvh6_tests.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r03_lbvh6_tests.txt
SCENE=terrain timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so > gpurun_out/r03_lbvh6_build_ms.txt 2>&1
timeout 300 bash tools/build_ms.sh paper_2509_17390_b200/libfgl.so >> gpurun_out/r03_lbvh6_build_ms.txt 2>&1
MODE=full bash tools/sweep.sh 'run plain' 'run treelets -- --treelets 1' 'run t_leaf1 -- --treelets 1 --leaf-size 1' > gpurun_out/r03_lbvh6_sweep.txt 2>&1
timeout 600 bash tools/ncu_build.sh lbvh6
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' --csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-latency > gpurun_out/r03_lbvh6_launches_C2.csv 2>/dev/null
