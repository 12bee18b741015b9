#!/bin/bash
# build_ms median for each FGL_LIB variant given (SCENE=rooms|terrain): tools/build_ms.sh lib1 lib2 ...
for lib in "$@"; do
  FGL_LIB=$lib python - <<'PY'
import os, torch, synth, statistics, paper_2509_17390_b200 as fgl
m = synth.scene_terrain(3).mesh if os.environ.get("SCENE") == "terrain" else synth.scene_rooms(2)
v = torch.from_numpy(m.verts).cuda(); t = torch.from_numpy(m.tris).cuda()
s = fgl.Scene(v, t)
ms = []
for i in range(12):
    s.build(); ms.append(s.stats()["build_ms"])
print(f"{os.environ['FGL_LIB']:40s} T={m.T} build_ms median {statistics.median(ms[2:]):.3f}")
PY
done
