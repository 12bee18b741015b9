import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, time, paper_2509_17390_b200 as fgl
cfg = synth.gauss_config("G2"); g, grid = cfg["gauss"], cfg["grid"]
gs = fgl.GaussianScene(g.mu, g.quat, g.scale, g.opacity, kappa=3.0)
for i in range(3): gs.build(); r = gs.voxelize(grid.origin, grid.h, grid.dims, 0.5)
torch.cuda.synchronize()
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
e0.record()
for i in range(10): gs.build()
e1.record()
for i in range(10): r = gs.voxelize(grid.origin, grid.h, grid.dims, 0.5)
e2.record(); torch.cuda.synchronize()
print("G2 build ms", e0.elapsed_time(e1)/10, "voxelize ms", e1.elapsed_time(e2)/10, "counts", r["counts"].tolist(), "grid", grid.dims)
