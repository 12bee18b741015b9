"""NEXT-1 measurement: point-cloud metrics (§V-A) between a simulated scan of the C2 rooms
and a scan of the same rooms with vertices jittered by 1 cm (both cast by libfgl), on B200.
Times index build + exact nearest neighbours both ways + the metric reduction (CUDA events), and
the oracle's O(mn) scan on a bounded sample. Prints one JSON line."""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_17390_b200 as fgl  # noqa: E402
import synth  # noqa: E402


def main(poses=8, steps=10, tau=0.02):
    cfg = synth.config("C2", poses=poses)
    m = cfg["mesh"]
    jit = synth.Mesh(m.verts + np.random.default_rng(3).normal(scale=0.01, size=m.verts.shape).astype(np.float32),
                     m.tris)
    a = fgl.Scene(m.verts, m.tris).cast(cfg["poses"], cfg["pattern"], hit_xyz=True)["hit_xyz"].reshape(-1, 3)
    b = fgl.Scene(jit.verts, jit.tris).cast(cfg["poses"], cfg["pattern"], hit_xyz=True)["hit_xyz"].reshape(-1, 3)
    a = a[torch.isfinite(a).all(1)].contiguous()
    b = b[torch.isfinite(b).all(1)].contiguous()
    for _ in range(2):
        fgl.cloud_metrics(a, b, tau)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for e in ev:
        e[0].record()
        res = fgl.cloud_metrics(a, b, tau)
        e[1].record()
    torch.cuda.synchronize()
    ms = statistics.median(e[0].elapsed_time(e[1]) for e in ev)
    # NN-only timing (index prebuilt)
    pb = fgl.PointCloud(b)
    for _ in range(2):
        pb.nearest(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        pb.nearest(a)
    e1.record()
    torch.cuda.synchronize()
    nn_ms = e0.elapsed_time(e1) / steps
    # oracle sample
    import oracle
    an, bn = a.cpu().numpy(), b.cpu().numpy()
    idx = np.random.default_rng(0).choice(an.shape[0], 256, replace=False)
    t0 = time.perf_counter()
    oracle.nearest(bn, an[idx])
    dt = time.perf_counter() - t0
    line = {"workload": f"C2 scan ({poses} poses) vs scan of 1 cm-jittered rooms, tau={tau} m",
            "points_a": int(a.shape[0]), "points_b": int(b.shape[0]),
            "metrics_ms": ms, "metrics_queries_per_s": (a.shape[0] + b.shape[0]) / (ms / 1e3),
            "nn_ms": nn_ms, "nn_queries_per_s": a.shape[0] / (nn_ms / 1e3),
            "chamfer_m": res["chamfer"], "precision": res["precision"], "recall": res["recall"],
            "fscore": res["fscore"],
            "cpu_baseline": {"value": 256 / dt, "unit": "nn queries/s", "cores": oracle.threads(), "kind": "oracle",
                             "sample": f"256 queries vs all {bn.shape[0]} points"}}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
