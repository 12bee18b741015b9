"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck): build + casts of
every kind (widths 2 / 4 / 4-quantised / 8, restructured, refitted) + sort + point metrics +
voxelizer / denoise / TSDF / marching cubes on small inputs."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_17390_b200 as fgl  # noqa: E402
import synth  # noqa: E402

cfg = synth.config("C1")
m = cfg["mesh"]
s = fgl.Scene(m.verts, m.tris)
r = s.cast(cfg["poses"], cfg["pattern"], hit_xyz=True, counts=True)
soup = synth.soup(10000, seed=1)
s2 = fgl.Scene(soup.verts, soup.tris)
ros = synth.Rosette(points_per_frame=1007)
s2.cast(synth.random_poses(2, 1, (0, 0, 0), (10, 10, 10)), ros)
o = torch.rand(5000, 3, device="cuda") * 10
d = torch.nn.functional.normalize(torch.randn(5000, 3, device="cuda"), dim=1)
s2.cast_rays(o, d, 0.1, 200.0)
s2.cast_rays(o, d, 0.1, 200.0, bruteforce=True)
s4 = fgl.Scene(soup.verts, soup.tris, width=4)
s4.cast(cfg["poses"], cfg["pattern"])
k = torch.randint(0, 2 ** 62, (50000,), device="cuda", dtype=torch.int64)
v = torch.arange(50000, device="cuda", dtype=torch.int32)
fgl.sort_pairs(k, v, 63)
fgl.cloud_metrics(r["hit_xyz"].reshape(-1, 3), r["hit_xyz"].reshape(-1, 3) + 0.01, 0.02)
# round 2: the compressed 8-wide layout (SAH collapse queue + cast), quantised width 4, treelet
# restructuring, refit, the graph-safe sort epoch (two sorts), voxelizer + masks, denoise, TSDF, MC
s8 = fgl.Scene(soup.verts, soup.tris, width=8)
s8.cast(cfg["poses"], cfg["pattern"])
s8.cast_rays(o, d, 0.1, 200.0)
s8.check()
s4q = fgl.Scene(soup.verts, soup.tris, width=4, quantized=1)
s4q.cast(cfg["poses"], cfg["pattern"])
sr = fgl.Scene(soup.verts, soup.tris, restructure=1)
sr.cast(cfg["poses"], cfg["pattern"])
s.refit(m.verts + np.float32(0.01))
s.cast(cfg["poses"], cfg["pattern"])
fgl.sort_pairs(k, v, 63)
g = synth.gaussians_random(300, 4)
grid = synth.grid_for(g, 20)
gs = fgl.GaussianScene(g.mu, g.quat, g.scale, g.opacity)
vox = gs.voxelize(grid.origin, grid.h, grid.dims, 0.5, density=True)
occ = vox["occupancy"] if isinstance(vox, dict) else vox
dims, sp = grid.dims, (grid.h, grid.h, grid.h)
dn = fgl.denoise(occ, dims, sp, 0.7, 0.35)
phi = fgl.tsdf(dn if isinstance(dn, torch.Tensor) else dn["occupancy"], dims, sp, 3.0 * grid.h)
fgl.marching_cubes(phi, grid.origin, sp, 0.0, normals=True)
torch.cuda.synchronize()
print("sanitize workload done")
