"""Pins for the oracle's point-cloud metrics (§V-A): closed forms on
lattices, the SPEC examples, and the metric invariants (symmetry, precision/recall duality,
monotonicity in the threshold, invariance under exact rigid motions)."""
import numpy as np

import oracle as orc


def _lattice(n=6, h=0.5):
    g = np.arange(n) * h
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    return np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1).astype(np.float32)


def test_spec_examples():
    a = _lattice()
    m = orc.cloud_metrics(a, a, 0.01)
    assert m["chamfer"] == 0.0 and m["precision"] == m["recall"] == m["fscore"] == 1.0
    m = orc.cloud_metrics(np.array([[0, 0, 0]], np.float32), np.array([[1, 0, 0]], np.float32), 0.5)
    assert m["chamfer"] == 1.0 and m["fscore"] == 0.0               # single pair -> 1.0
    far = a + np.float32(100.0)
    m = orc.cloud_metrics(a, far, 1.0)
    assert m["precision"] == m["recall"] == m["fscore"] == 0.0      # disjoint beyond tau


def test_shifted_lattice_closed_form():
    # every point of a lattice shifted by s < h/2 along x has its nearest neighbour at distance s
    h, s = 0.5, 0.125
    a = _lattice(8, h)
    b = a + np.array([s, 0, 0], np.float32)
    d, i = orc.nearest(a, b)
    assert np.allclose(d, s, atol=0, rtol=1e-12)
    assert np.array_equal(i, np.arange(a.shape[0]))
    m = orc.cloud_metrics(a, b, 0.2)
    assert abs(m["chamfer"] - s) < 1e-12 and m["fscore"] == 1.0
    m = orc.cloud_metrics(a, b, 0.1)
    assert m["fscore"] == 0.0


def test_ties_go_to_smaller_index():
    p = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0]], np.float32)
    d, i = orc.nearest(p, np.zeros((1, 3), np.float32))
    assert i[0] == 0 and d[0] == 1.0


def test_invariants():
    rng = np.random.default_rng(0)
    a = (np.round(rng.uniform(-4, 4, (700, 3)) * 256) / 256).astype(np.float32)
    b = (np.round(rng.uniform(-4, 4, (500, 3)) * 256) / 256).astype(np.float32)
    mab = orc.cloud_metrics(a, b, 0.3)
    mba = orc.cloud_metrics(b, a, 0.3)
    assert abs(mab["chamfer"] - mba["chamfer"]) < 1e-15                     # symmetry
    assert mab["precision"] == mba["recall"] and mab["recall"] == mba["precision"]  # duality
    f = [orc.cloud_metrics(a, b, t)["fscore"] for t in (0.05, 0.1, 0.2, 0.4, 0.8)]
    assert all(x <= y for x, y in zip(f, f[1:]))                             # monotone in tau
    S = np.array([[0, 0, 1], [1, 0, 0], [0, -1, 0]], np.float64)             # exact signed permutation
    sh = np.array([5.0, -3.0, 2.0])
    ra = (a.astype(np.float64) @ S.T + sh).astype(np.float32)
    rb = (b.astype(np.float64) @ S.T + sh).astype(np.float32)
    mr = orc.cloud_metrics(ra, rb, 0.3)
    assert abs(mr["chamfer"] - mab["chamfer"]) < 1e-12 and mr["fscore"] == mab["fscore"]


def test_brute_force_matches_numpy_definition_on_tiny_clouds():
    rng = np.random.default_rng(1)
    a = rng.normal(size=(40, 3)).astype(np.float32)
    b = rng.normal(size=(30, 3)).astype(np.float32)
    D = np.linalg.norm(a[:, None, :].astype(np.float64) - b[None, :, :].astype(np.float64), axis=2)
    d, i = orc.nearest(b, a)
    assert np.allclose(d, D.min(1), rtol=1e-15) and np.array_equal(i, D.argmin(1))
