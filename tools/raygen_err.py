"""Max |d_gpu - d_oracle| of the exported float32 ray directions vs the oracle's double rays, over
many poses / frames (run under gpurun): the raygen bound the mode-A classifier eps must cover."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_17390_b200 as fgl  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402

worst = {}
for name, cols in (("VLP16", 360), ("HDL64", 2048), ("OS128", 2048), ("VLP32", 1800)):
    for seed in range(4):
        pat = synth.spinning_preset(name, cols, az0_deg=1.25 * seed)
        poses = synth.random_poses(8, seed, (-300, -300, -20), (300, 300, 20))
        o, d = fgl.export_rays(pat, poses)
        oo, dd = oracle.pattern_rays(pat, poses)
        err = np.abs(d.cpu().numpy().astype(np.float64) - dd).max()
        worst[name] = max(worst.get(name, 0.0), err)
ros = synth.rosette_default()
for ff in (0, 999, 123456789, 2 ** 40 // 20000):
    poses = synth.random_poses(4, ff % 97, (-1, -1, -1), (1, 1, 1))
    o, d = fgl.export_rays(ros, poses, first_frame=ff)
    oo, dd = oracle.pattern_rays(ros, poses, ff)
    err = np.abs(d.cpu().numpy().astype(np.float64) - dd).max()
    worst["rosette"] = max(worst.get("rosette", 0.0), err)
for k, v in worst.items():
    print(f"{k:8s} max |d_gpu - d_oracle| = {v:.3e} = 2^{np.log2(v):.2f}")
