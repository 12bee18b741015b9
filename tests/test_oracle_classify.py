"""Pins for the oracle's ambiguity classifier. The classifier decides which rays
have a unique correct float answer. Pins: hand-built degenerate configurations with known
status, and the semantic property the classifier promises: an unambiguous ray keeps its strict
answer under every perturbation smaller than the classifier's epsilon."""
import numpy as np

import synth

TMIN, TMAX = 0.1, 200.0


def _two_tris():
    V = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]], np.float32)
    return V, np.array([[0, 1, 2], [1, 3, 2]], np.int32)


def _classify(orc, V, Tr, o, d, **kw):
    o = np.asarray(o, np.float64).reshape(-1, 3)
    d = np.asarray(d, np.float64).reshape(-1, 3)
    return orc.cast_and_classify(V, Tr, o, d, kw.pop("tmin", TMIN), kw.pop("tmax", TMAX), **kw)


def test_interior_is_unambiguous(orc):
    V, Tr = _two_tris()
    v = _classify(orc, V, Tr, [0.25, 0.25, 2.0], [0, 0, -1])
    assert v.flags[0] == 0 and v.ncand[0] == 1 and v.cid[0, 0] == 0
    assert v.clo[0, 0] <= 2.0 <= v.chi[0, 0]


def test_shared_edge_is_ambiguous_with_both(orc):
    V, Tr = _two_tris()
    v = _classify(orc, V, Tr, [0.5, 0.5, 2.0], [0, 0, -1])
    assert v.flags[0] & orc.AMBIG and v.flags[0] & orc.EDGE
    assert sorted(v.cid[0, :v.ncand[0]]) == [0, 1]
    assert v.k1[0] == 0


def test_silhouette_edge_allows_miss(orc):
    V, Tr = _two_tris()
    # exactly on the outer edge x = 0 of triangle 0: marginal, nothing firm -> a miss is also correct
    v = _classify(orc, V, Tr, [0.0, 0.5, 2.0], [0, 0, -1])
    assert v.flags[0] & orc.AMBIG and v.flags[0] & orc.MISS_OK
    assert list(v.cid[0, :v.ncand[0]]) == [0]
    # 1 mm outside: no candidate at all, unambiguous miss
    v = _classify(orc, V, Tr, [-1e-3, 0.5, 2.0], [0, 0, -1])
    assert v.flags[0] == orc.MISS_OK and v.ncand[0] == 0 and v.k1[0] == -1


def test_grazing_is_ambiguous(orc):
    # triangle tilted 1e-5 rad out of the ray direction: the depth is ill-conditioned
    V = np.array([[0, -1, -1e-4], [10, -1, 1e-4], [0, 1, -1e-4]], np.float32)
    v = _classify(orc, V, np.array([[0, 1, 2]], np.int32), [-1, -0.5, 0.0], [1, 0, 0])
    assert v.k1[0] == 0 and abs(v.t1[0] - 6.0) < 1e-3
    assert v.flags[0] & orc.AMBIG
    assert v.flags[0] & (orc.GRAZE | orc.EDGE)


def test_interval_boundary_is_ambiguous(orc):
    V, Tr = _two_tris()
    v = _classify(orc, V, Tr, [0.25, 0.25, 8.0], [0, 0, -1], tmax=8.0)
    assert v.flags[0] & orc.BOUNDARY and v.flags[0] & orc.AMBIG
    v = _classify(orc, V, Tr, [0.25, 0.25, 7.0], [0, 0, -1], tmax=8.0)
    assert v.flags[0] == 0


def test_stacked_faces_tie_is_ambiguous(orc):
    # two parallel triangles 1e-9 m apart: their depths are not separable in float32
    V = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1e-9], [1, 0, 1e-9], [0, 1, 1e-9]], np.float32)
    Tr = np.array([[0, 1, 2], [3, 4, 5]], np.int32)
    v = _classify(orc, V, Tr, [0.2, 0.2, 3.0], [0, 0, -1])
    assert v.flags[0] & orc.AMBIG and v.ncand[0] == 2
    # 1 cm apart: separable -> unambiguous, nearer one wins
    V[3:, 2] = 0.01
    v = _classify(orc, V, Tr, [0.2, 0.2, 3.0], [0, 0, -1])
    assert v.flags[0] == 0 and v.k1[0] == 1


def test_closed_mesh_never_leaks(orc):
    # from inside a closed box / icosphere every ray has a strict hit and, if ambiguous, candidates
    for m in (synth.box((-1, -1, -1), (1, 2, 3), 0.25), synth.icosphere(3, 10.0)):
        rng = np.random.default_rng(1)
        R = 1500
        o = rng.uniform(-0.5, 0.5, size=(R, 3))
        d = rng.normal(size=(R, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        v = orc.cast_and_classify(m.verts, m.tris, o, d, TMIN, TMAX)
        assert np.all(v.k1 >= 0)
        assert np.all((v.flags & orc.MISS_OK) == 0)
        assert np.all(v.ncand >= 1)


def test_unambiguous_rays_are_stable_under_perturbation(orc):
    """The classifier's promise: below its epsilon, no perturbation of ray origin or direction
    changes an unambiguous ray's nearest triangle. Checked on a dense soup with many near-edge rays."""
    m = synth.soup(600, seed=3, extent=4.0, size=0.6)
    rng = np.random.default_rng(4)
    R = 800
    o = rng.uniform(-2, 6, size=(R, 3)).astype(np.float32).astype(np.float64)
    # aim at vertices and edge midpoints so that many rays are degenerate by construction
    Vd = m.verts.astype(np.float64)
    a = m.tris[rng.integers(0, m.T, R)]
    w = np.where(rng.uniform(size=(R, 1)) < 0.5, 0.5, 1.0)
    tgt = w * Vd[a[:, 0]] + (1 - w) * Vd[a[:, 1]]
    d = tgt - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    v = orc.cast_and_classify(m.verts, m.tris, o, d, TMIN, TMAX, eps_rel=orc.EPS_MODE_B)
    un = ~v.ambiguous
    assert un.sum() > R // 4 and v.ambiguous.sum() > R // 10  # the construction creates both kinds
    assert np.all((v.flags & orc.INCONSISTENT) == 0)
    for trial in range(6):
        scale = orc.EPS_MODE_B * 0.3
        dist = np.where(np.isfinite(v.t1), v.t1, 10.0)
        po = o + rng.normal(size=o.shape) * (scale * np.maximum(dist, 1.0))[:, None] / np.sqrt(3)
        pd = d + rng.normal(size=d.shape) * scale / np.sqrt(3)
        t2, k2 = orc.cast(m.verts, m.tris, po, pd, TMIN, TMAX)
        assert np.array_equal(k2[un], v.k1[un]), trial
    # and ambiguous rays' perturbed answers always lie in the kept candidate set (or a permitted miss)
    t2, k2 = orc.cast(m.verts, m.tris, po, pd, TMIN, TMAX)
    for r in np.nonzero(v.ambiguous & ((v.flags & orc.OVERFLOW) == 0))[0]:
        if k2[r] < 0:
            assert v.flags[r] & orc.MISS_OK
        else:
            assert k2[r] in set(v.cid[r, :v.ncand[r]])


def test_c1_ambiguity_is_rare(orc):
    cfg = synth.config("C1")
    m = cfg["mesh"]
    o, d = orc.pattern_rays(cfg["pattern"], cfg["poses"])
    v = orc.cast_and_classify(m.verts, m.tris, o, d, TMIN, TMAX, eps_rel=orc.EPS_MODE_A)
    assert np.all(v.k1 >= 0)  # inside a closed sphere: 100% hit
    assert v.ambiguous.mean() < 0.01
    assert np.all((v.flags & orc.INCONSISTENT) == 0)
