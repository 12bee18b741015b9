"""SIMT-loss analysis of the C2 cast (run under gpurun): per-ray node / triangle counts from the
COUNT variant, grouped into the kernel's 32-ray tiles (4 channels x 8 columns of one pose). A warp
runs until its longest ray is done, so sum(max over tile) / sum(mean over tile) bounds the lane
idling that the tile tail alone causes."""
import sys, os
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_17390_b200 as fgl  # noqa: E402
import synth  # noqa: E402

cfg = synth.config("C2", poses=8)
m, pat, poses = cfg["mesh"], cfg["pattern"], cfg["poses"]
s = fgl.Scene(m.verts, m.tris, device="cuda:0")
r = s.cast(poses, pat, counts=True)
nc = r["node_counts"].cpu().numpy().astype(np.float64)  # [P][C][A]
tc = r["tri_counts"].cpu().numpy().astype(np.float64)
P, C, A = nc.shape
for tcn, tan in ((4, 8), (2, 16), (8, 4), (1, 32)):
    x = nc.reshape(P, C // tcn, tcn, A // tan, tan).transpose(0, 1, 3, 2, 4).reshape(-1, tcn * tan)
    y = tc.reshape(P, C // tcn, tcn, A // tan, tan).transpose(0, 1, 3, 2, 4).reshape(-1, tcn * tan)
    w = x * 55 + y * 70  # rough instructions per ray
    print(f"tile {tcn}x{tan}: nodes mean {x.mean():.2f} tile-max mean {x.max(1).mean():.2f} "
          f"eff {x.mean() / x.max(1).mean():.3f}; tris eff {y.mean() / max(y.max(1).mean(), 1e-9):.3f}; "
          f"weighted eff {w.mean() / w.max(1).mean():.3f}")
print("node count percentiles", np.percentile(nc, [5, 25, 50, 75, 95, 99]))
print("tri count percentiles", np.percentile(tc, [5, 25, 50, 75, 95, 99]))
rng = r["range"].cpu().numpy()
print("range percentiles", np.percentile(rng[np.isfinite(rng)], [5, 25, 50, 75, 95]), "miss", np.mean(~np.isfinite(rng)))
