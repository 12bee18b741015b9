"""GPU parity of the point-cloud metrics (NEXT-1; §V-A): exact nearest neighbours from the
LBVH-indexed point scene vs the oracle's O(mn) scan, and Chamfer / precision / recall / F-score
on simulated scans of a mesh and of a perturbed copy."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fgl():
    import paper_2509_17390_b200 as f
    f.lib()
    return f


def _check_nn(pts, q, d, i):
    dref, iref = oracle.nearest(pts, q)
    d = d.cpu().numpy().astype(np.float64)
    i = i.cpu().numpy()
    fin = np.isfinite(q).all(1)
    assert np.all(np.isnan(d[~fin])) and np.all(i[~fin] == -1)
    assert np.allclose(d[fin], dref[fin], rtol=2e-6, atol=1e-7)
    diff = np.nonzero(fin & (i != iref))[0]
    # a different index is only allowed on a near-tie: its exact distance equals the minimum
    for k in diff:
        true_d = np.linalg.norm(pts[i[k]].astype(np.float64) - q[k].astype(np.float64))
        assert abs(true_d - dref[k]) <= 2e-6 * max(dref[k], 1e-3), (k, true_d, dref[k])
    assert diff.size <= max(2, 1e-3 * q.shape[0])


@pytest.mark.parametrize("n,m", [(1, 10), (2, 100), (1000, 3000), (200_000, 20_000)])
def test_nearest_matches_oracle(fgl, n, m):
    rng = np.random.default_rng(n)
    pts = rng.uniform(-5, 5, size=(n, 3)).astype(np.float32)
    q = rng.uniform(-7, 7, size=(m, 3)).astype(np.float32)
    q[: min(m, n) // 3] = pts[: min(m, n) // 3]  # exact hits: distance 0
    q[-1] = np.nan                                   # a missed beam's hit point
    pc = fgl.PointCloud(pts)
    d, i = pc.nearest(q)
    _check_nn(pts, q, d, i)


def test_metrics_special_cases(fgl):
    a = np.random.default_rng(0).uniform(0, 1, (500, 3)).astype(np.float32)
    m = fgl.cloud_metrics(a, a, 0.01)
    assert m["chamfer"] == 0.0 and m["precision"] == m["recall"] == m["fscore"] == 1.0
    m = fgl.cloud_metrics(np.array([[0, 0, 0]], np.float32), np.array([[1, 0, 0]], np.float32), 0.5)
    assert m["chamfer"] == 1.0 and m["fscore"] == 0.0


def _scan(fgl, mesh, cfg):
    s = fgl.Scene(mesh.verts, mesh.tris)
    r = s.cast(cfg["poses"], cfg["pattern"], hit_xyz=True)
    return r["hit_xyz"].reshape(-1, 3)


def test_scan_vs_perturbed_mesh_scan(fgl):
    cfg = synth.config("C1")
    m = cfg["mesh"]
    jit = synth.Mesh(m.verts + np.random.default_rng(3).normal(scale=0.01, size=m.verts.shape).astype(np.float32),
                     m.tris)
    a = _scan(fgl, m, cfg)
    b = _scan(fgl, jit, cfg)
    tau = 0.02
    g = fgl.cloud_metrics(a, b, tau)
    an, bn = a.cpu().numpy(), b.cpu().numpy()
    an, bn = an[np.isfinite(an).all(1)], bn[np.isfinite(bn).all(1)]
    o = oracle.cloud_metrics(an, bn, tau)
    assert g["n_a"] == an.shape[0] and g["n_b"] == bn.shape[0]
    assert abs(g["chamfer"] - o["chamfer"]) <= 1e-6 * o["chamfer"] + 1e-9
    # threshold decisions within rounding of tau may differ
    amb_a = np.sum(np.abs(o["d_ab"] - tau) <= 1e-6 * tau)
    amb_b = np.sum(np.abs(o["d_ba"] - tau) <= 1e-6 * tau)
    assert abs(g["precision"] - o["precision"]) * an.shape[0] <= amb_a + 1e-9
    assert abs(g["recall"] - o["recall"]) * bn.shape[0] <= amb_b + 1e-9
    assert 0.0 < o["chamfer"] < 0.05 and 0 < o["fscore"] <= 1
