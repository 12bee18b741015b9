"""Does concurrent PCIe traffic slow the LBVH build / the cast? Device times of build and cast alone,
and while a 67 MB D2H and an 18 MB H2D copy run on other streams (e2e pipeline conditions)."""
import os, sys, statistics
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_17390_b200 as fgl  # noqa: E402
import synth  # noqa: E402

cfg = synth.config("C2", poses=64)
m, pat = cfg["mesh"], cfg["pattern"]
v = torch.from_numpy(m.verts).cuda(); t = torch.from_numpy(m.tris).cuda()
poses = torch.from_numpy(np.ascontiguousarray(cfg["poses"])).cuda()
s = fgl.Scene(v, t)
out = s.cast(poses, pat)
dbig = torch.empty(67_108_864 // 4, device="cuda"); hbig = torch.empty(67_108_864 // 4).pin_memory()
dsm = torch.empty(18_330_168 // 4, device="cuda"); hsm = torch.empty(18_330_168 // 4).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
vh = torch.from_numpy(m.verts).pin_memory(); th = torch.from_numpy(m.tris).pin_memory()


def timed(fn, dma, upload=None, reps=10):
    res = []
    for _ in range(reps):
        torch.cuda.synchronize()
        if dma:
            with torch.cuda.stream(s1):
                hbig.copy_(dbig, non_blocking=True)
            with torch.cuda.stream(s2):
                if upload is not None:
                    upload.upload(vh, th, sync=False, stream=s2)
                else:
                    dsm.copy_(hsm, non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1))
    return statistics.median(res)


b0 = timed(lambda: s.build(), False)
b1 = timed(lambda: s.build(), True)
c0 = timed(lambda: s.cast(poses, pat, out=out), False)
c1 = timed(lambda: s.cast(poses, pat, out=out), True)
print(f"build alone {b0:.3f} ms, with D2H+H2D copies {b1:.3f} ms; cast alone {c0:.3f} ms, with copies {c1:.3f} ms")
s2u = fgl.Scene(v, t)
b2 = timed(lambda: s.build(), True, upload=s2u)
print(f"build with D2H + another scene's upload (H2D + validate) {b2:.3f} ms")
