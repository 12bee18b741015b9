"""Pins of oracle/gauss.py (the NEXT-2 voxelizer oracle) against things other than itself: closed
forms, an independent quaternion route, matrix inversion by the library, brute force, Monte Carlo
containment and set identities (Eqs. 4, 8-12; SPEC voxelizer / lbvh examples)."""
import math

import numpy as np
import pytest

import synth
from oracle import gauss as og


def _one(mu, q, s, o):
    return synth.Gaussians(np.array([mu], np.float32), np.array([q], np.float32), np.array([s], np.float32),
                           np.array([o], np.float32))


def _hamilton(a, b):
    w1, x1, y1, z1 = a
    w2, x2, y2, z2 = b
    return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])


Q90Z = (math.cos(math.pi / 4), 0.0, 0.0, math.sin(math.pi / 4))


def test_rotation_closed_forms():
    assert np.allclose(og.rotation([1, 0, 0, 0])[0], np.eye(3))
    assert np.allclose(og.rotation(Q90Z)[0], [[0, -1, 0], [1, 0, 0], [0, 0, 1]], atol=1e-15)
    # unnormalised input is normalised
    assert np.allclose(og.rotation([2, 0, 0, 0])[0], np.eye(3))


def test_rotation_matches_quaternion_sandwich():
    rng = np.random.default_rng(0)
    for _ in range(50):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        v = rng.normal(size=3)
        rot = _hamilton(_hamilton(q, np.r_[0.0, v]), q * np.array([1, -1, -1, -1]))[1:]
        R = og.rotation(q)[0]
        assert np.allclose(R @ v, rot, atol=1e-12)
        assert np.allclose(R @ R.T, np.eye(3), atol=1e-12) and abs(np.linalg.det(R) - 1) < 1e-12


def test_aabb_spec_examples():
    lo, hi = og.aabb([[1, 2, 3]], [[1, 0, 0, 0]], [[1, 2, 3]], 1.0)
    assert np.allclose(lo, [[0, 0, 0]]) and np.allclose(hi, [[2, 4, 6]])
    lo, hi = og.aabb([[0, 0, 0]], [Q90Z], [[1, 2, 3]], 1.0)
    assert np.allclose(hi, [[2, 1, 3]]) and np.allclose(lo, [[-2, -1, -3]])


def test_aabb_contains_kappa_ellipsoid_monte_carlo():
    rng = np.random.default_rng(1)
    g = synth.gaussians_random(50, 3)
    kappa = 3.0
    lo, hi = og.aabb(g.mu, g.quat, g.scale, kappa)
    R = og.rotation(g.quat)
    for n in range(g.N):
        u = rng.normal(size=(2000, 3))
        u *= (rng.uniform(size=(2000, 1)) ** (1 / 3)) / np.linalg.norm(u, axis=1, keepdims=True)
        u[:8] = np.eye(3)[[0, 1, 2, 0, 1, 2, 0, 1]] * np.array([1, 1, 1, -1, -1, -1, 1, 1])[:, None]  # extreme axes
        x = g.mu[n] + kappa * (u * g.scale[n]) @ R[n].T  # Mahalanobis distance <= kappa
        assert np.all(x >= lo[n] - 1e-12) and np.all(x <= hi[n] + 1e-12)


def test_precision_is_inverse_covariance():
    g = synth.gaussians_random(40, 4)
    A = og.precision(g.quat, g.scale)
    R = og.rotation(g.quat)
    S2 = g.scale.astype(np.float64) ** 2
    for n in range(g.N):
        Sigma = R[n] @ np.diag(S2[n]) @ R[n].T
        assert np.allclose(A[n], np.linalg.inv(Sigma), rtol=1e-9, atol=1e-9 * np.abs(A[n]).max())


def test_density_single_gaussian_values():
    # SPEC gs_assets: x = mu -> 1; isotropic unit scale at distance 1 -> exp(-1/2);
    # s = (2, 1, 1) rotated 90 deg about z, x = mu + (0, 2, 0) -> exp(-1/2)
    g = _one((0, 0, 0), (1, 0, 0, 0), (1, 1, 1), 1.0)
    D, _, _ = og.density_at(g, [[0, 0, 0], [1, 0, 0], [0, 0, 2.5]], 3.0)
    assert np.allclose(D, [1.0, math.exp(-0.5), math.exp(-3.125)])
    g = _one((1, 1, 1), Q90Z, (2, 1, 1), 1.0)
    D, _, _ = og.density_at(g, [[1, 3, 1], [3, 1, 1]], 3.0)
    assert np.allclose(D, [math.exp(-0.5), math.exp(-2.0)])


def test_truncation_at_kappa():
    g = _one((0, 0, 0), (1, 0, 0, 0), (1, 1, 1), 0.7)
    D, fs, _ = og.density_at(g, [[2.999, 0, 0], [3.001, 0, 0]], 3.0)
    assert D[0] == pytest.approx(0.7 * math.exp(-0.5 * 2.999 ** 2)) and D[1] == 0.0
    assert fs[0] == pytest.approx(0.7) and fs[1] == 0.0


def test_single_isotropic_gaussian_occupancy_closed_form():
    # SPEC voxelizer example: s = 1, sigma = 0.8, theta = 0.5, h = 0.25: occupied iff
    # |v - mu| < sqrt(2 ln(0.8 / 0.5)) (inside kappa s = 3, so the truncation never bites)
    g = _one((0, 0, 0), (1, 0, 0, 0), (1, 1, 1), 0.8)
    grid = synth.Grid((-2.0, -2.0, -2.0), 0.25, (16, 16, 16))
    D, _, _ = og.density(g, grid, 3.0)
    V = og.occupancy(D, 0.5)
    r = np.linalg.norm(og.centers(grid.origin, grid.h, grid.dims), axis=-1)
    assert np.array_equal(V, r < math.sqrt(2 * math.log(0.8 / 0.5)))
    # a voxel centre at mu: D = sigma exactly
    grid2 = synth.Grid((-2.125, -2.125, -2.125), 0.25, (17, 17, 17))
    D2, _, _ = og.density(g, grid2, 3.0)
    assert D2[8, 8, 8] == float(np.float32(0.8))


def test_density_forms_agree_with_brute_force():
    g = synth.gaussians_random(60, 5, extent=1.5, scale_median=0.1)
    grid = synth.grid_for(g, 14)
    Db, Fb, Mb = og.density_bruteforce(g, grid, 3.0)
    for Dx, Fx, Mx in (og.density(g, grid, 3.0), og.density_tiled(g, grid, 3.0, 8), og.density_tiled(g, grid, 3.0, 3),
                       og.density_tiled(g, grid, 3.0, 1)):
        assert np.allclose(Dx, Db, rtol=1e-12, atol=1e-15)
        assert np.allclose(Fx, Fb, rtol=1e-12, atol=1e-15)
        assert np.allclose(Mx, Mb, rtol=1e-12, atol=1e-15)
    c = og.centers(grid.origin, grid.h, grid.dims).reshape(-1, 3)[::97]
    D, _, _ = og.density_at(g, c, 3.0)
    assert np.allclose(D, Db.reshape(-1)[::97], rtol=1e-12, atol=1e-15)
    assert Db.max() > 0.5  # the case is not trivially empty


def test_threshold_properties():
    g = synth.gaussians_random(80, 6, extent=1.5, scale_median=0.12)
    grid = synth.grid_for(g, 12)
    D, _, _ = og.density(g, grid, 3.0)
    assert not og.occupancy(D, float(g.opacity.sum()) + 1).any()  # theta above every possible sum
    V1, V2 = og.occupancy(D, 0.2), og.occupancy(D, 0.6)
    assert np.all(V1 | ~V2) and V1.sum() > V2.sum() > 0  # theta1 < theta2 => V2 ⊆ V1


def test_translation_equivariance():
    g = synth.gaussians_random(40, 7, extent=1.0, scale_median=0.1)
    grid = synth.grid_for(g, 10)
    shift = np.array([3, -5, 7]) * 0.5  # exact in binary
    g2 = synth.Gaussians(g.mu + shift.astype(np.float32), g.quat, g.scale, g.opacity)
    grid2 = synth.Grid(tuple(np.asarray(grid.origin) + shift), grid.h, grid.dims)
    D1, _, _ = og.density(g, grid, 3.0)
    D2, _, _ = og.density(g2, grid2, 3.0)
    assert np.allclose(D1, D2, atol=1e-9)


def _interior_loops(V):
    nz, ny, nx = V.shape
    out = np.zeros_like(V)
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                if not V[k, j, i]:
                    continue
                ok = True
                for dk, dj, di in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
                    kk, jj, ii = k + dk, j + dj, i + di
                    if not (0 <= kk < nz and 0 <= jj < ny and 0 <= ii < nx and V[kk, jj, ii]):
                        ok = False
                out[k, j, i] = ok
    return out


def test_masks_closed_forms():
    V = np.zeros((5, 6, 7), bool)
    V[2, 3, 4] = True
    assert not og.interior(V).any() and np.array_equal(og.surface(V), V)
    V = np.zeros((7, 7, 7), bool)
    V[2:5, 2:5, 2:5] = True
    I = og.interior(V)
    assert I.sum() == 1 and I[3, 3, 3] and og.surface(V).sum() == 26
    V = np.zeros((9, 10, 11), bool)
    V[1:8, 2:7, 3:10] = True  # 7 x 5 x 7 block
    assert og.interior(V).sum() == 5 * 3 * 5
    V = np.ones((4, 5, 6), bool)  # the whole grid: boundary voxels are never interior (R27)
    assert og.interior(V).sum() == 2 * 3 * 4


def test_masks_brute_force_and_identities():
    rng = np.random.default_rng(8)
    for p in (0.5, 0.8, 0.95):
        V = rng.uniform(size=(6, 7, 9)) < p
        I, S = og.interior(V), og.surface(V)
        assert np.array_equal(I, _interior_loops(V))
        assert np.array_equal(S | I, V) and not (S & I).any()


def test_unpack_bits_layout():
    dims = (40, 2, 1)
    w = np.zeros((1, 2, 2), np.uint32)
    w[0, 0, 0] = 1 | (1 << 31)
    w[0, 1, 1] = 1 << 7  # voxel x = 39 of row 1
    V = og.unpack_bits(w, dims)
    assert V.shape == (1, 2, 40)
    assert V[0, 0, 0] and V[0, 0, 31] and V[0, 1, 39] and V.sum() == 3


def test_r25_equals_literal_eq9_occupancy_on_g1():
    """R25 (a Gaussian contributes only inside its kappa-ellipsoid) against Eqs. 8-9 read literally
    (every candidate of C_tile contributes exp(-m^2/2) f): the literal density is never
    smaller, exceeds R25's by at most exp(-kappa^2/2) x (sum of f over candidates outside their
    ellipsoid), and the occupancy (Eq. 10) can differ only on voxels within that bound of theta. On
    the G1 workload (theta = 0.5, kappa = 3, B = 8) that is 393 of 262 144 voxels (0.15%), all within
    the bound (R25): the readings agree except on threshold-marginal voxels."""
    cfg = synth.gauss_config("G1")
    g, grid, kappa, theta = cfg["gauss"], cfg["grid"], cfg["kappa"], cfg["theta"]
    Dr, _, _ = og.density_tiled(g, grid, kappa, cfg["tile"])
    Dl, excess = og.density_tiled_literal(g, grid, kappa, cfg["tile"])
    bound = math.exp(-0.5 * kappa * kappa) * excess
    assert np.all(Dl >= Dr - 1e-12)  # the literal sum only adds non-negative terms
    assert np.all(Dl - Dr <= bound * (1 + 1e-12) + 1e-15)
    flip = og.occupancy(Dl, theta) != og.occupancy(Dr, theta)
    near = np.abs(Dr - theta) <= bound + 1e-12
    assert np.all(near[flip])  # a flip is only possible within the bound
    assert flip.sum() <= 0.005 * flip.size, int(flip.sum())
    print(f"R25 vs literal Eq. 9 on G1: {int(flip.sum())} of {flip.size} voxels flip, all within the bound")
    assert og.occupancy(Dr, theta).sum() > 1000  # a non-trivial volume
