"""Compare the fused width-2 build (k_lbvh) with the unfused path (build_ab/libfgl_unfused.so) on the
terrain / rooms scenes: child, range, node64 bitwise; run in two processes (FGL_LIB differs)."""
import os, subprocess, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    import torch, synth, paper_2509_17390_b200 as fgl
    which, out = sys.argv[2], sys.argv[3]
    if which == "terrain":
        m = synth.scene_terrain(3).mesh
    elif which.startswith("soup"):
        m = synth.soup(int(which[4:]), seed=5)
    else:
        m = synth.scene_rooms(2)
    s = fgl.Scene(torch.from_numpy(m.verts).cuda(), torch.from_numpy(m.tris).cuda())
    e = s.export()
    np.savez(out, child=e["child"], range=e["range"], nodes=e["nodes"], node_box=e["node_box"])
    sys.exit(0)

for which in sys.argv[1:] or ["soup3000000", "terrain"]:
    res = {}
    for tag, env in (("fused", {}), ("global", {"FGL_LBVH_GLOBAL": "1"}),
                     ("unfused", {"FGL_LIB": "build_ab/libfgl_unfused.so"})):
        f = f"/tmp/dbg_{which}_{tag}.npz"
        subprocess.check_call([sys.executable, __file__, "--child", which, f], env={**os.environ, **env})
        res[tag] = np.load(f)
    for tag in ("fused", "global"):
        for k in ("child", "range", "nodes", "node_box"):
            a, b = res[tag][k], res["unfused"][k]
            a8, b8 = a.reshape(len(a), -1).view(np.uint8), b.reshape(len(b), -1).view(np.uint8)
            bad = np.nonzero(np.any(a8 != b8, axis=1))[0]
            print(f"{which} {tag:7s} {k:8s} mismatching rows {len(bad)} first {bad[:8].tolist()}")
