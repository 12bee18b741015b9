"""Pins for the oracle's nearest-hit scan (Eq. 20; naive baseline P:291-294).

Expectations come from exact rational arithmetic with a *different* formulation (Plucker /
orient3d signs + plane equation), closed forms for planes, boxes and convex polyhedra, and
invariants of the definition (closedness, permutation, duplication, symmetry)."""
import math
from fractions import Fraction as F

import numpy as np
import pytest

import synth

TMIN, TMAX = 0.1, 200.0


# ---------------------------------------------------------------------------------------------
def test_spec_unit_triangle():
    import oracle as orc
    # unit triangle in the plane z = 5, ray from the origin along +z through its centroid: t* = 5 [S:153]
    V = np.array([[0, 0, 5], [1, 0, 5], [0, 1, 5]], np.float32)
    Tr = np.array([[0, 1, 2]], np.int32)
    c = V.astype(np.float64).mean(0)
    o = np.array([[c[0], c[1], 0.0], [c[0], c[1], 0.0]])
    d = np.array([[0, 0, 1.0], [0, 0, -1.0]])
    t, k = orc.cast(V, Tr, o, d, 0.0, 100.0)
    assert t[0] == 5.0 and k[0] == 0
    assert np.isinf(t[1]) and k[1] == -1  # along -z: none [S:154]


# ---------------------------------------------------------------------------------------------
def _exact_first_hit(V, Tr, o, d, tmin, tmax):
    """Exact rational first hit with Plucker-sign inclusion and the plane equation (not MT).
    Returns (t, id, margin) where margin is the smallest relative decision slack seen."""
    o = [F(x) for x in o]
    d = [F(x) for x in d]
    best, bid, margin = None, -1, math.inf
    ts = []
    for k, (a, b, c) in enumerate(Tr):
        P = [[F(float(x)) for x in V[a]], [F(float(x)) for x in V[b]], [F(float(x)) for x in V[c]]]
        rel = [[P[i][j] - o[j] for j in range(3)] for i in range(3)]

        def vol(u, w):  # (u x w) . d
            return (u[1] * w[2] - u[2] * w[1]) * d[0] + (u[2] * w[0] - u[0] * w[2]) * d[1] + (u[0] * w[1] - u[1] * w[0]) * d[2]

        s = [vol(rel[0], rel[1]), vol(rel[1], rel[2]), vol(rel[2], rel[0])]
        e1 = [P[1][j] - P[0][j] for j in range(3)]
        e2 = [P[2][j] - P[0][j] for j in range(3)]
        n = [e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]]
        nd = sum(n[j] * d[j] for j in range(3))
        if nd == 0:
            continue
        tot = abs(s[0]) + abs(s[1]) + abs(s[2])
        inside = (min(s) >= 0 or max(s) <= 0)
        # decision slack: how close the signs are to flipping, relative to their scale
        sl = min(abs(x) for x in s) / tot if tot else 0
        t = sum(n[j] * rel[0][j] for j in range(3)) / nd
        if inside or sl < 1e-6:
            margin = min(margin, float(sl))
        if not inside:
            continue
        if t < tmin or t > tmax:
            margin = min(margin, float(min(abs(t - tmin), abs(t - tmax)) / max(abs(t), 1)))
            continue
        ts.append(t)
        if best is None or t < best:
            best, bid = t, k
    if best is not None:
        for t in ts:
            if t != best:
                margin = min(margin, float(abs(t - best) / best))
    return (float(best) if best is not None else math.inf), bid, margin


@pytest.mark.slow
def test_exact_rational_soup():
    import oracle as orc
    rng = np.random.default_rng(11)
    V = rng.uniform(-1, 1, size=(3 * 24, 3)).astype(np.float32)
    Tr = np.arange(72, dtype=np.int32).reshape(24, 3)
    R = 160
    o = rng.uniform(-3, 3, size=(R, 3)).astype(np.float32).astype(np.float64)
    # aim half of the rays at triangle interiors so that hits are plentiful
    tgt = rng.uniform(-1, 1, size=(R, 3))
    k = rng.integers(0, 24, size=R)
    w = rng.dirichlet([1, 1, 1], size=R)
    aim = np.einsum("ri,rij->rj", w, V[Tr[k]].astype(np.float64))
    tgt[: R // 2] = aim[: R // 2]
    d = (tgt - o).astype(np.float32).astype(np.float64)
    t, kk = orc.cast(V, Tr, o, d, 0.0, 1e9)
    checked = 0
    for r in range(R):
        te, ke, margin = _exact_first_hit(V, Tr, o[r], d[r], 0.0, 1e9)
        if margin < 1e-9:
            continue
        checked += 1
        assert kk[r] == ke, r
        if ke >= 0:
            assert abs(t[r] - te) <= 1e-12 * abs(te)
        else:
            assert np.isinf(t[r])
    assert checked >= R - 4
    assert (kk >= 0).sum() >= R // 2


def test_exact_shared_edge_and_vertices():
    import oracle as orc
    # two triangles sharing the edge (1,0,0)-(0,1,0) in the plane z = 0; dyadic coordinates
    V = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]], np.float32)
    Tr = np.array([[0, 1, 2], [1, 3, 2]], np.int32)
    pts, exp = [], []
    for p, e in [((0, 0), 0), ((1, 0), 0), ((0, 1), 0), ((1, 1), 1),        # vertices: smaller id
                 ((0.5, 0.5), 0),                                           # shared-edge midpoint
                 ((0.25, 0.25), 0), ((0.75, 0.75), 1),                      # interiors
                 ((0.5, 0), 0), ((1, 0.5), 1), ((0, 0.5), 0), ((0.5, 1), 1),  # outer edges (inclusive)
                 ((1.25, 0.5), -1), ((-0.25, 0.5), -1)]:                   # outside
        pts.append(p)
        exp.append(e)
    P = np.array(pts, np.float64)
    R = len(pts)
    o = np.concatenate([P, np.full((R, 1), 2.0)], 1)
    d = np.tile([0.0, 0.0, -1.0], (R, 1))
    t, k = orc.cast(V, Tr, o, d, TMIN, TMAX)
    assert list(k) == exp
    assert np.all(t[np.array(exp) >= 0] == 2.0)
    # back face (from below, going up) is hit: two-sided (R2)
    t, k = orc.cast(V, Tr, np.array([[0.25, 0.25, -3.0]]), np.array([[0, 0, 1.0]]), TMIN, TMAX)
    assert k[0] == 0 and t[0] == 3.0
    # in-plane ray (det = 0): no hit (R16); origin on the plane: t = 0 < t_min: no hit (R17)
    t, k = orc.cast(V, Tr, np.array([[-1, 0.25, 0.0], [0.25, 0.25, 0.0]]),
                    np.array([[1, 0, 0.0], [0, 0, 1.0]]), TMIN, TMAX)
    assert list(k) == [-1, -1]
    # interval is closed: t exactly t_min and exactly t_max both hit (R3)
    o = np.array([[0.25, 0.25, 0.5], [0.25, 0.25, 8.0]])
    d = np.array([[0, 0, -1.0], [0, 0, -1.0]])
    t, k = orc.cast(V, Tr, o, d, 0.5, 8.0)
    assert list(k) == [0, 0] and list(t) == [0.5, 8.0]
    t, k = orc.cast(V, Tr, o, d, 0.5 + 2 ** -40, 8.0 - 2 ** -40)
    assert list(k) == [-1, -1]
    # one ulp either side of the outer edge x = 0
    x = np.nextafter(0.0, 1.0), np.nextafter(0.0, -1.0)
    t, k = orc.cast(V, Tr, np.array([[x[0], 0.5, 1.0], [x[1], 0.5, 1.0]]), np.array([[0, 0, -1.0]] * 2), TMIN, TMAX)
    assert list(k) == [0, -1]


def test_duplicate_triangle_smaller_id_wins():
    import oracle as orc
    V = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], np.float32)
    Tr = np.array([[0, 1, 2], [0, 2, 1], [1, 2, 0]], np.int32)  # same triangle three times
    t, k = orc.cast(V, Tr, np.array([[0.2, 0.3, 1.0]]), np.array([[0, 0, -1.0]]), TMIN, TMAX)
    assert k[0] == 0 and t[0] == 1.0


# ---------------------------------------------------------------------------------------------
def test_floor_grid_closed_form():
    import oracle as orc
    nx, ny, D = 64, 48, 0.25
    m = synth.floor_grid(nx, ny, D, 0.0, -8.0, -6.0)
    rng = np.random.default_rng(3)
    R = 3000
    h = 1.7
    o = np.tile([0.3, -0.2, h], (R, 1))
    e = rng.uniform(-80, -12, R) * np.pi / 180
    th = rng.uniform(0, 2 * np.pi, R)
    d = np.stack([np.cos(e) * np.cos(th), np.cos(e) * np.sin(th), np.sin(e)], 1)
    t, k = orc.cast(m.verts, m.tris, o, d, TMIN, TMAX)
    texp = h / -d[:, 2]
    x = o + texp[:, None] * d
    gx, gy = (x[:, 0] + 8.0) / D, (x[:, 1] + 6.0) / D
    i, j = np.floor(gx), np.floor(gy)
    fx, fy = gx - i, gy - j
    ok = (gx > 1e-6) & (gx < nx - 1e-6) & (gy > 1e-6) & (gy < ny - 1e-6)
    clean = ok & (np.minimum.reduce([fx, 1 - fx, fy, 1 - fy, np.abs(fx - fy)]) > 1e-7)
    kexp = (2 * (i * ny + j) + np.where(fx >= fy, 0, 1)).astype(np.int64)
    assert clean.sum() > 0.9 * R
    assert np.array_equal(k[clean], kexp[clean])
    assert np.allclose(t[clean], texp[clean], rtol=1e-12, atol=0)
    outside = (gx < -1e-6) | (gx > nx + 1e-6) | (gy < -1e-6) | (gy > ny + 1e-6)
    assert outside.sum() > 0 and np.all(k[outside] == -1)


def _box_face_id(lo, hi, h, x):
    """Closed-form triangle id of the point x on the surface of synth.box(lo, hi, h)."""
    n = np.maximum(1, np.ceil((np.asarray(hi) - np.asarray(lo)) / h - 1e-9)).astype(int)
    off = 0
    best = None
    dist = []
    for a in range(3):
        for side, val in ((0, lo[a]), (1, hi[a])):
            dist.append((abs(x[a] - val), a, side, off))
            b, c = (a + 1) % 3, (a + 2) % 3
            off += 2 * n[b] * n[c]
    dmin, a, side, off = min(dist)
    b, c = (a + 1) % 3, (a + 2) % 3
    gu = (x[b] - lo[b]) / (hi[b] - lo[b]) * n[b]
    gw = (x[c] - lo[c]) / (hi[c] - lo[c]) * n[c]
    iu, iw = min(int(gu), n[b] - 1), min(int(gw), n[c] - 1)
    fu, fw = gu - iu, gw - iw
    slack = min(fu, 1 - fu, fw, 1 - fw, abs(fu - fw), sorted(d[0] for d in dist)[1])
    return off + 2 * (iu * n[c] + iw) + (0 if fu >= fw else 1), slack


def test_box_inside_slab_closed_form():
    import oracle as orc
    lo, hi, h = (-1.0, -2.0, -3.0), (2.0, 3.0, 4.0), 0.5
    m = synth.box(lo, hi, h)
    rng = np.random.default_rng(5)
    R = 1500
    o = rng.uniform(np.array(lo) + 0.3, np.array(hi) - 0.3, size=(R, 3))
    d = rng.normal(size=(R, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    t, k = orc.cast(m.verts, m.tris, o, d, TMIN, TMAX)
    # slab exit: t = min_a (bound_a - o_a) / d_a with bound = hi if d_a > 0 else lo
    tb = np.where(d > 0, (np.array(hi) - o) / d, (np.array(lo) - o) / d)
    texp = tb.min(1)
    assert np.all(k >= 0)  # closed box: no leak
    good = 0
    for r in range(R):
        if texp[r] < TMIN + 1e-6:
            continue
        kid, slack = _box_face_id(lo, hi, h, o[r] + texp[r] * d[r])
        assert abs(t[r] - texp[r]) <= 1e-12 * texp[r]
        if slack > 1e-7:
            assert k[r] == kid
            good += 1
    assert good > 0.95 * R
    # from outside: slab entry (SPEC S:153 generalised)
    o2 = np.array([[0.5, 0.5, 10.0], [5.0, 0.25, 0.25]])
    d2 = np.array([[0, 0, -1.0], [-1, 0, 0.0]])
    t2, _ = orc.cast(m.verts, m.tris, o2, d2, TMIN, TMAX)
    assert list(t2) == [6.0, 3.0]
    # pointing away from the scene: all miss [S:477]
    t3, k3 = orc.cast(m.verts, m.tris, np.array([[10.0, 0, 0]] * 3), np.array([[1, 0, 0.0], [0, 1, 0], [0.6, 0.8, 0]]), TMIN, TMAX)
    assert np.all(k3 == -1)


def test_icosphere_convex_polyhedron():
    import oracle as orc
    m = synth.icosphere(3, 10.0)
    V = m.verts.astype(np.float64)
    A, B, C = V[m.tris[:, 0]], V[m.tris[:, 1]], V[m.tris[:, 2]]
    n = np.cross(B - A, C - A)
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    h = np.einsum("ij,ij->i", n, A)
    assert np.all(h > 0)  # outward
    # convexity precondition: every vertex on the inner side of every face plane
    assert np.max(V @ n.T - h[None, :]) < 1e-9
    rng = np.random.default_rng(9)
    R = 2000
    o = rng.uniform(-5, 5, size=(R, 3))
    d = rng.normal(size=(R, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    t, k = orc.cast(m.verts, m.tris, o, d, TMIN, TMAX)
    nd = d @ n.T
    tt = np.where(nd > 0, (h[None, :] - o @ n.T) / np.where(nd > 0, nd, 1), np.inf)
    srt = np.sort(tt, 1)
    kexp = np.argmin(tt, 1)
    clean = (srt[:, 1] - srt[:, 0]) > 1e-9 * srt[:, 0]
    assert clean.mean() > 0.97
    assert np.array_equal(k[clean], kexp[clean])
    assert np.allclose(t, srt[:, 0], rtol=1e-12, atol=0)


def test_sphere_sagitta_bounds_from_centre():
    import oracle as orc
    m = synth.icosphere(3, 10.0)
    V = m.verts.astype(np.float64)
    A, B, C = V[m.tris[:, 0]], V[m.tris[:, 1]], V[m.tris[:, 2]]
    n = np.cross(B - A, C - A)
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    hmin = np.einsum("ij,ij->i", n, A).min()
    rmax = np.linalg.norm(V, axis=1).max()
    p = synth.spinning_preset("VLP32", 360)
    o, d = orc.spinning_rays(p.elev_deg, 360, 0.0, synth.pose((0, 0, 0))[None])
    t, k = orc.cast(m.verts, m.tris, o, d, TMIN, TMAX)
    assert np.all(k >= 0)                                  # every beam hits [S:476, S:596]
    assert t.min() >= hmin - 1e-12 and t.max() <= rmax + 1e-12
    assert np.all(np.abs(t - 10.0) <= 0.02 * 10.0)         # within 2% of 10 m [S:476]


# ---------------------------------------------------------------------------------------------
def test_permutation_and_symmetry_invariance():
    import oracle as orc
    # dyadic mesh so that signed axis permutations and integer translations are exact in float32
    rng = np.random.default_rng(21)
    T = 200
    V = (np.round(rng.uniform(-4, 4, size=(3 * T, 3)) * 1024) / 1024).astype(np.float32)
    Tr = np.arange(3 * T, dtype=np.int32).reshape(T, 3)
    R = 400
    o = np.round(rng.uniform(-6, 6, size=(R, 3)) * 64) / 64
    tgt = V[rng.integers(0, 3 * T, R)].astype(np.float64) * 0.9
    d = tgt - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    t, k = orc.cast(V, Tr, o, d, TMIN, TMAX)
    assert (k >= 0).sum() > R // 3
    # triangle permutation: ranges equal, ids remap
    perm = rng.permutation(T)
    t2, k2 = orc.cast(V, Tr[perm], o, d, TMIN, TMAX)
    assert np.array_equal(t, t2)
    hit = k2 >= 0
    assert np.array_equal(perm[k2[hit]], k[hit]) or np.sum(perm[k2[hit]] != k[hit]) <= 2
    # signed axis permutation + integer translation of mesh and rays (an exact rigid motion)
    S = np.array([[0, -1, 0], [0, 0, 1], [1, 0, 0]], np.float64)
    sh = np.array([3.0, -5.0, 7.0])
    V3 = (V.astype(np.float64) @ S.T + sh).astype(np.float32)
    assert np.array_equal(V3.astype(np.float64), V.astype(np.float64) @ S.T + sh)
    t3, k3 = orc.cast(V3, Tr, o @ S.T + sh, d @ S.T, TMIN, TMAX)
    assert np.allclose(t3[hit], t[hit], rtol=1e-12) and np.array_equal(np.isinf(t3), np.isinf(t))
    assert np.mean(k3 == k) > 0.99
