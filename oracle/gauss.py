"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py for the rules).

Plain double-precision numpy statement of the Gaussian -> occupancy step of PAPER.md §IV-A
(SURVEY §8(f) NEXT-2): the per-Gaussian AABB (Eq. 4), tile culling (Eq. 8,
P:134-137), density at voxel centres (Eq. 9), the occupancy threshold (Eq. 10,
P:160-166) and the interior / surface masks (Eqs. 11-12). The LBVH over the boxes
(Eqs. 5-7) is the oracle's existing `lbvh` machinery; here the boxes are culled by a plain
overlap test, which is what the BVH query must return (SPEC lbvh query_overlap).

Readings (R24-R28): f(sigma) = sigma (R24); a Gaussian contributes to voxel v only
when its squared Mahalanobis distance m^2 <= kappa^2 (R25, truncation at the kappa-sigma
ellipsoid, which lies inside the Eq. 4 box, so Eq. 8 culling drops nothing); voxel centres
v_ijk = o + (i + 1/2, j + 1/2, k + 1/2) h (R26); a voxel on the grid boundary is never interior
(R27, missing neighbours count as empty).

Pin status: every function is pinned in tests/test_oracle_gauss.py against closed forms (single
isotropic / rotated Gaussians, solid blocks), brute force over all voxel-Gaussian pairs, Monte
Carlo containment and set identities. None is "parity unpinned".
"""
from __future__ import annotations

import numpy as np

# m^2 within this relative band of kappa^2: float32 evaluation may include or drop the term
EDGE_REL = 1e-4


def rotation(quat):
    """R(q) for unit quaternions q = (w, x, y, z) (normalised here), the R_i of Sigma_i =
    R_i S_i S_i^T R_i^T (§III-A). Returns [N][3][3] float64."""
    q = np.asarray(quat, np.float64).reshape(-1, 4)
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    R = np.empty((q.shape[0], 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z)
    R[:, 0, 1] = 2 * (x * y - w * z)
    R[:, 0, 2] = 2 * (x * z + w * y)
    R[:, 1, 0] = 2 * (x * y + w * z)
    R[:, 1, 1] = 1 - 2 * (x * x + z * z)
    R[:, 1, 2] = 2 * (y * z - w * x)
    R[:, 2, 0] = 2 * (x * z - w * y)
    R[:, 2, 1] = 2 * (y * z + w * x)
    R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def aabb(mu, quat, scale, kappa: float):
    """Eq. 4: r_i = kappa |R_i| s_i (|R| elementwise), b_i = [mu_i - r_i, mu_i + r_i].
    Returns (lo, hi), float64 [N][3]."""
    R = rotation(quat)
    s = np.asarray(scale, np.float64).reshape(-1, 3)
    r = kappa * np.einsum("nij,nj->ni", np.abs(R), s)
    m = np.asarray(mu, np.float64).reshape(-1, 3)
    return m - r, m + r


def precision(quat, scale):
    """Sigma_i^-1 = R_i diag(1 / s_i^2) R_i^T, float64 [N][3][3]."""
    R = rotation(quat)
    s = np.asarray(scale, np.float64).reshape(-1, 3)
    return np.einsum("nij,nj,nkj->nik", R, 1.0 / (s * s), R)


def centers(origin, h: float, dims):
    """Voxel centres v_ijk = o + (i + 1/2, j + 1/2, k + 1/2) h (R26), float64 [nz][ny][nx][3]."""
    nx, ny, nz = (int(d) for d in dims)
    o = np.asarray(origin, np.float64)
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    return np.stack([o[0] + (i + 0.5) * h, o[1] + (j + 0.5) * h, o[2] + (k + 0.5) * h], axis=-1)


def _accumulate(D, fsum, marg, v, mu, A, f, kappa, sel):
    """Add Gaussian (mu, A = Sigma^-1, weight f) to the voxels `sel` (index tuple) of D."""
    d = v[sel] - mu
    m2 = np.einsum("...i,ij,...j->...", d, A, d)
    inside = m2 <= kappa * kappa
    g = np.where(inside, np.exp(-0.5 * m2), 0.0) * f
    D[sel] += g
    fsum[sel] += np.where(inside, f, 0.0)
    near = np.abs(m2 - kappa * kappa) <= EDGE_REL * kappa * kappa
    marg[sel] += np.where(near, np.exp(-0.5 * m2) * f, 0.0)


def density_bruteforce(g, grid, kappa: float):
    """Eq. 9 by its definition over every (voxel, Gaussian) pair, with the R25 truncation.
    Returns (D, fsum, marg), float64 [nz][ny][nx]: density, the sum of f over contributing
    Gaussians, and the contribution of Gaussians whose m^2 is within EDGE_REL of kappa^2."""
    v = centers(grid.origin, grid.h, grid.dims)
    A = precision(g.quat, g.scale)
    mu = g.mu.astype(np.float64)
    f = g.opacity.astype(np.float64)  # R24: f(sigma) = sigma
    D = np.zeros(v.shape[:3])
    fsum, marg = np.zeros_like(D), np.zeros_like(D)
    allv = (slice(None),) * 3
    for n in range(g.N):
        _accumulate(D, fsum, marg, v, mu[n], A[n], f[n], kappa, allv)
    return D, fsum, marg


def tile_candidates(box_lo, box_hi, tlo, thi):
    """Eq. 8: indices i with b_i ∩ B_tile ≠ ∅ (closed boxes)."""
    ok = np.all((box_lo <= thi) & (box_hi >= tlo), axis=1)
    return np.nonzero(ok)[0]


def density_tiled(g, grid, kappa: float, tile: int = 8):
    """Eqs. 8-9 in the paper's order: for every tile of tile^3 voxels, the candidate set C_tile of
    Gaussians whose Eq. 4 box meets the box spanned by the tile's voxel centres (Eq. 8), then each
    voxel of the tile sums over C_tile (Eq. 9, R25 truncation). Returns (D, fsum, marg)."""
    v = centers(grid.origin, grid.h, grid.dims)
    lo, hi = aabb(g.mu, g.quat, g.scale, kappa)
    A = precision(g.quat, g.scale)
    mu = g.mu.astype(np.float64)
    f = g.opacity.astype(np.float64)
    nx, ny, nz = grid.dims
    D = np.zeros((nz, ny, nx))
    fsum, marg = np.zeros_like(D), np.zeros_like(D)
    for z0 in range(0, nz, tile):
        for y0 in range(0, ny, tile):
            for x0 in range(0, nx, tile):
                sel = (slice(z0, min(z0 + tile, nz)), slice(y0, min(y0 + tile, ny)), slice(x0, min(x0 + tile, nx)))
                tv = v[sel].reshape(-1, 3)
                for n in tile_candidates(lo, hi, tv.min(axis=0), tv.max(axis=0)):
                    _accumulate(D, fsum, marg, v, mu[n], A[n], f[n], kappa, sel)
    return D, fsum, marg


def density_tiled_literal(g, grid, kappa: float, tile: int = 8):
    """Eqs. 8-9 read literally (no R25 truncation): every voxel of a tile sums exp(-m^2/2) f over
    the WHOLE candidate set C_tile of Eq. 8, however far outside the kappa ellipsoid a candidate's
    m^2 lies. The result depends on the tile partition (the reason for R25); it is kept as the
    literal reading against which R25 is pinned (tests/test_oracle_gauss.py). Returns (D, excess)
    where excess is the sum over candidates with m^2 > kappa^2 of f (each such term is below
    exp(-kappa^2/2) f, so |D_literal - D_R25| <= exp(-kappa^2/2) excess)."""
    v = centers(grid.origin, grid.h, grid.dims)
    lo, hi = aabb(g.mu, g.quat, g.scale, kappa)
    A = precision(g.quat, g.scale)
    mu = g.mu.astype(np.float64)
    f = g.opacity.astype(np.float64)
    nx, ny, nz = grid.dims
    D = np.zeros((nz, ny, nx))
    excess = np.zeros_like(D)
    for z0 in range(0, nz, tile):
        for y0 in range(0, ny, tile):
            for x0 in range(0, nx, tile):
                sel = (slice(z0, min(z0 + tile, nz)), slice(y0, min(y0 + tile, ny)), slice(x0, min(x0 + tile, nx)))
                tv = v[sel].reshape(-1, 3)
                for n in tile_candidates(lo, hi, tv.min(axis=0), tv.max(axis=0)):
                    d = v[sel] - mu[n]
                    m2 = np.einsum("...i,ij,...j->...", d, A[n], d)
                    D[sel] += np.exp(-0.5 * m2) * f[n]
                    excess[sel] += np.where(m2 > kappa * kappa, f[n], 0.0)
    return D, excess


def density(g, grid, kappa: float):
    """Eq. 9 with R25, each Gaussian scattered to the voxels whose centres lie in its Eq. 4 box
    (the kappa ellipsoid lies inside that box, so nothing else can receive a contribution).
    Same result as density_bruteforce; the fast form the tests use. Returns (D, fsum, marg)."""
    v = centers(grid.origin, grid.h, grid.dims)
    lo, hi = aabb(g.mu, g.quat, g.scale, kappa)
    A = precision(g.quat, g.scale)
    mu = g.mu.astype(np.float64)
    f = g.opacity.astype(np.float64)
    o = np.asarray(grid.origin, np.float64)
    dims = np.asarray(grid.dims)
    D = np.zeros(v.shape[:3])
    fsum, marg = np.zeros_like(D), np.zeros_like(D)
    # voxel i has centre o + (i + 1/2) h: the centres inside [lo, hi] are i in [ceil(a), floor(b)]
    i0 = np.maximum(np.ceil((lo - o) / grid.h - 0.5).astype(np.int64) - 1, 0)
    i1 = np.minimum(np.floor((hi - o) / grid.h - 0.5).astype(np.int64) + 1, dims - 1)
    for n in range(g.N):
        if np.any(i1[n] < i0[n]):
            continue
        sel = (slice(i0[n, 2], i1[n, 2] + 1), slice(i0[n, 1], i1[n, 1] + 1), slice(i0[n, 0], i1[n, 0] + 1))
        _accumulate(D, fsum, marg, v, mu[n], A[n], f[n], kappa, sel)
    return D, fsum, marg


def density_at(g, points, kappa: float):
    """Eq. 9 with R25 at arbitrary points (sampled parity at full size): [M] (D, fsum, marg)."""
    p = np.asarray(points, np.float64).reshape(-1, 3)
    lo, hi = aabb(g.mu, g.quat, g.scale, kappa)
    A = precision(g.quat, g.scale)
    mu = g.mu.astype(np.float64)
    f = g.opacity.astype(np.float64)
    out = np.zeros((3, p.shape[0]))
    for m in range(p.shape[0]):
        cand = np.nonzero(np.all((lo <= p[m]) & (hi >= p[m]), axis=1))[0]
        d = p[m] - mu[cand]
        m2 = np.einsum("ni,nij,nj->n", d, A[cand], d)
        inside = m2 <= kappa * kappa
        e = np.exp(-0.5 * m2) * f[cand]
        out[0, m] = np.sum(np.where(inside, e, 0.0))
        out[1, m] = np.sum(np.where(inside, f[cand], 0.0))
        out[2, m] = np.sum(np.where(np.abs(m2 - kappa * kappa) <= EDGE_REL * kappa * kappa, e, 0.0))
    return out[0], out[1], out[2]


def tol_density(fsum):
    """Allowed |D_gpu - D| for a float32 evaluation: 1e-4 of the summed weights
    (m^2 relative error <~ 1e-5 after tile-relative offsets, exp2 and summation rounding) + 1e-6."""
    return 1e-4 * fsum + 1e-6


def occupancy(D, theta: float):
    """Eq. 10: V = D > theta (strict)."""
    return np.asarray(D) > theta


def interior(V):
    """Eq. 11: V and all six face neighbours occupied; outside the grid counts as
    empty (R27)."""
    V = np.asarray(V, bool)
    P = np.zeros(tuple(n + 2 for n in V.shape), bool)
    P[1:-1, 1:-1, 1:-1] = V
    c = (slice(1, -1),) * 3
    out = V.copy()
    for ax in range(3):
        for sgn in (-1, 1):
            sl = list(c)
            sl[ax] = slice(1 + sgn, P.shape[ax] - 1 + sgn)
            out &= P[tuple(sl)]
    return out


def surface(V):
    """Eq. 12: Surf = V and not Int."""
    V = np.asarray(V, bool)
    return V & ~interior(V)


def unpack_bits(words, dims):
    """Bit-packed volume (uint32 [nz][ny][ceil(nx / 32)], bit b of word w = voxel 32 w + b) ->
    bool [nz][ny][nx]. Test helper for the device layout."""
    nx, ny, nz = dims
    w = np.asarray(words, np.uint32).reshape(nz, ny, -1)
    bits = np.unpackbits(w.view(np.uint8).reshape(nz, ny, -1), axis=-1, bitorder="little")
    return bits[:, :, :nx].astype(bool)
