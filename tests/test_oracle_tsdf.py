"""Pins of oracle/tsdf.py (the NEXT-3 TSDF + Marching Cubes oracle): scipy.ndimage routines for
the blur, the flood fill and the taxicab shells; closed forms for boxes and cavities; mesh
invariants (closed 2-manifold, consistent outward orientation, Euler characteristic, enclosed
volume) for every one of the 254 non-trivial cube cases, spheres and random fields."""
import math

import numpy as np
import pytest
from scipy import ndimage

from oracle import tsdf as ot


# ---- Eqs. 13-14 --------------------------------------------------------------------------------
@pytest.mark.parametrize("sigma_vox", [0.4, 1.0, 1.7])
def test_blur_matches_scipy(sigma_vox):
    rng = np.random.default_rng(0)
    V = rng.uniform(size=(7, 9, 11)) < 0.4
    h = 0.05
    B = ot.blur(V, sigma_vox * h, (h, h, h))
    R = max(1, math.ceil(3 * sigma_vox))
    ref = V.astype(np.float64)
    for ax in (2, 1, 0):
        ref = ndimage.gaussian_filter1d(ref, sigma_vox, axis=ax, mode="constant", cval=0.0,
                                        truncate=(R - 0.25) / sigma_vox)
    assert np.allclose(B, ref, atol=1e-13)
    assert abs(ot.gauss_weights(sigma_vox).sum() - 1) < 1e-15


def test_blur_anisotropic_spacing_and_constant_interior():
    V = np.ones((9, 9, 21), bool)
    B = ot.blur(V, 0.1, (0.05, 0.1, 0.2))  # sigma = 2, 1, 0.5 voxels along x, y, z (radius 6, 3, 2)
    assert B[4, 4, 10] == pytest.approx(1.0, abs=1e-12)  # farther than every radius from the border
    assert B[4, 4, 0] < B[4, 0, 10] < B[0, 4, 10] < 1  # x blurs widest, z least
    assert np.array_equal(ot.rethreshold(B, 0.5), B >= 0.5)


# ---- Eqs. 15-17 --------------------------------------------------------------------------------
def _outside_scipy(V):
    free = np.pad(~V, 1, constant_values=True)
    lab, _ = ndimage.label(free)  # default structure = 6-connectivity
    return (lab == lab[0, 0, 0])[1:-1, 1:-1, 1:-1]


def test_outside_matches_scipy_label():
    rng = np.random.default_rng(1)
    for p in (0.3, 0.5, 0.65):
        V = rng.uniform(size=(10, 12, 9)) < p
        assert np.array_equal(ot.outside(V), _outside_scipy(V))


def test_hollow_box_cavity_is_inside():
    V = np.zeros((9, 9, 9), bool)
    V[2:7, 2:7, 2:7] = True
    V[3:6, 3:6, 3:6] = False  # enclosed void
    O = ot.outside(V)
    assert not O[3:6, 3:6, 3:6].any() and O[0, 0, 0] and O[1, 4, 4]
    V[3, 4, 2] = False  # tunnel to the cavity? (2 is the wall at x=2 -> opens the void)
    assert ot.outside(V)[4, 4, 4]


def test_shells_are_taxicab_distance_to_s0():
    rng = np.random.default_rng(2)
    V = ndimage.binary_closing(rng.uniform(size=(14, 13, 12)) < 0.45)
    S = ot.boundary_set(V)
    # S_0 by its definition with the frame free, pinned on a hand case
    W = np.zeros((3, 3, 3), bool)
    W[1, 1, 1] = True
    assert ot.boundary_set(W).sum() == 7  # the voxel + its 6 neighbours
    ref = ndimage.distance_transform_cdt(~S, metric="taxicab")
    for m_max in (0, 2, 5):
        k = ot.shells(V, m_max)
        exp = np.where(ref <= m_max, ref, -1)
        assert np.array_equal(k, exp)


def test_tsdf_closed_forms():
    V = np.zeros((11, 11, 11), bool)
    V[3:8, 3:8, 3:8] = True
    h = 0.1
    phi, kappa = ot.tsdf(V, (h, h, h), 0.25)  # band: ceil(0.25 / 0.1) = 3 shells
    assert phi.dtype == np.float32
    # S_0 = the block's outer layer and the free layer around it (kappa 0); the centre voxel is two
    # shells deeper: phi = -(2 * h) in float32, inside the r = 0.25 band
    assert kappa[5, 5, 5] == 2 and phi[5, 5, 5] == -(np.float32(2) * np.float32(h))
    assert phi[3, 5, 5] == 0 and phi[2, 5, 5] == 0  # both sides of the interface
    assert phi[1, 5, 5] == np.float32(1) * np.float32(0.1) and phi[0, 5, 5] == np.float32(2) * np.float32(0.1)


def test_tsdf_band_and_signs():
    V = np.zeros((15, 15, 15), bool)
    V[2:13, 2:13, 2:13] = True
    phi, kappa = ot.tsdf(V, (0.1, 0.1, 0.1), 0.3)
    assert phi[7, 7, 7] == np.float32(-0.3)  # kappa 5 > band: -r
    assert np.all(phi[~V] >= 0) and np.all(phi[V & (kappa != 0)] < 0)
    assert np.all(np.abs(phi) <= np.float32(0.3))


# ---- Eq. 18 ------------------------------------------------------------------------------------
def _check_closed_oriented(verts, tris):
    """Every undirected edge in exactly two triangles, with opposite directions."""
    assert len(tris) > 0
    d = {}
    for t in tris:
        for a, b in ((t[0], t[1]), (t[1], t[2]), (t[2], t[0])):
            assert (a, b) not in d, "directed edge repeated: inconsistent orientation"
            d[(a, b)] = 1
    for (a, b) in d:
        assert (b, a) in d, "boundary edge: not watertight"
    E = len(d) // 2
    return len(verts) - E + len(tris)  # Euler characteristic


def _volume(verts, tris):
    a, b, c = verts[tris[:, 0]], verts[tris[:, 1]], verts[tris[:, 2]]
    return np.einsum("ij,ij->i", a, np.cross(b, c)).sum() / 6.0


def test_all_256_cube_cases_closed_and_outward():
    n_ok = 0
    for case in range(1, 255):
        phi = np.ones((4, 4, 4), np.float32)  # pad with outside corners so the surface closes
        for c in range(8):
            if (case >> c) & 1:
                phi[1 + ((c >> 2) & 1), 1 + ((c >> 1) & 1), 1 + (c & 1)] = -1.0
        V, T = ot.marching_cubes(phi, (0, 0, 0), (1, 1, 1))
        chi = _check_closed_oriented(V, T)
        comps = ndimage.label(phi < 0)[1]
        assert chi == 2 * comps  # each inside component is wrapped by its own sphere
        assert _volume(V, T) > 0  # outward orientation
        n_ok += 1
    assert n_ok == 254


def test_single_corner_case_geometry():
    phi = np.ones((3, 3, 3), np.float32)
    phi[1, 1, 1] = -1.0
    V, T = ot.marching_cubes(phi, (0, 0, 0), (1, 1, 1))
    assert len(V) == 6 and len(T) == 8  # an octahedron around the voxel centre (1.5,1.5,1.5)
    assert np.allclose(np.sort(np.abs(V - 1.5).sum(axis=1)), 0.5)
    assert _volume(V, T) == pytest.approx(4 / 3 * 0.5 ** 3)  # octahedron of radius 1/2


@pytest.mark.parametrize("R", [3.3, 5.7])
def test_sphere_sdf(R):
    n = int(2 * R + 6)
    g = np.arange(n) + 0.5 - n / 2
    Z, Y, X = np.meshgrid(g, g, g, indexing="ij")
    phi = (np.sqrt(X * X + Y * Y + Z * Z) - R).astype(np.float32)
    V, T, N = ot.marching_cubes(phi, (-n / 2, -n / 2, -n / 2), (1, 1, 1), normals=True)
    assert _check_closed_oriented(V, T) == 2
    vol = _volume(V, T)
    assert abs(vol / (4 / 3 * math.pi * R ** 3) - 1) < 0.8 / R ** 2  # chord error O((h / R)^2)
    assert np.all(np.abs(np.linalg.norm(V, axis=1) - R) < 0.1)
    radial = V / np.linalg.norm(V, axis=1, keepdims=True)
    assert np.all(np.einsum("ij,ij->i", N, radial) > 0.95)


def test_random_fields_always_watertight():
    rng = np.random.default_rng(3)
    for _ in range(20):
        phi = np.ones((8, 8, 8), np.float32)
        phi[1:-1, 1:-1, 1:-1] = rng.choice([-1.0, 1.0], size=(6, 6, 6)).astype(np.float32)
        V, T = ot.marching_cubes(phi, (0, 0, 0), (1, 1, 1))
        if len(T):
            _check_closed_oriented(V, T)
            assert _volume(V, T) > 0


def test_vertices_on_linear_edges_exact():
    phi = np.zeros((2, 2, 3), np.float32)
    phi[..., 0], phi[..., 1], phi[..., 2] = -1.0, 3.0, 7.0  # zero crossing at x = 0.25 of cell 0
    V, T = ot.marching_cubes(phi, (0, 0, 0), (2.0, 1.0, 1.0))
    assert len(V) == 4 and np.allclose(V[:, 0], 1.0 + 0.25 * 2.0)
    assert len(T) == 2  # one quad, open (the surface leaves the grid)


def test_centroid_fans_only_where_needed():
    """Loops fanned around a centre vertex exist (through ambiguous faces) but are rare, and every
    other loop keeps the one-vertex-per-crossing-edge property."""
    n_loops = n_centre = 0
    for case in range(1, 255):
        for loop in ot.cube_polygons([(case >> c) & 1 for c in range(8)]):
            n_loops += 1
            n_centre += not ot.fan_ok(loop)
            assert 3 <= len(loop) <= 12
    assert 0 < n_centre < n_loops // 4


def test_pipeline_on_occupancy_sphere():
    """Eqs. 15-18 end to end on a voxelised ball: a closed surface around it, volume close to the
    ball's, every vertex within the band of the voxel surface."""
    n, R, h = 24, 7.5, 0.1
    g = np.arange(n) + 0.5 - n / 2
    Z, Y, X = np.meshgrid(g, g, g, indexing="ij")
    V = X * X + Y * Y + Z * Z <= R * R
    phi, _ = ot.tsdf(V, (h, h, h), 3 * h)
    verts, tris = ot.marching_cubes(phi, (0.0, 0.0, 0.0), (h, h, h))
    assert _check_closed_oriented(verts, tris) == 2
    vol = _volume(verts, tris)
    assert 0.6 < vol / (V.sum() * h ** 3) < 1.05  # the iso = 0 surface sits on the inner boundary layer


def test_quantile_matches_numpy_inverted_cdf():
    rng = np.random.default_rng(9)
    for n in (1, 7, 1000):
        v = rng.uniform(size=n).astype(np.float32)
        v[: n // 3] = 0.0  # ties, as the blurred occupancy has
        for q in (0.0, 0.1, 0.5, 0.9, 0.999, 1.0):
            assert ot.quantile(v, q) == np.quantile(v, q, method="inverted_cdf")
    v = np.arange(10, dtype=np.float32)
    assert ot.quantile(v, 1.0) == 9 and ot.quantile(v, 0.0) == 0 and ot.quantile(v, 0.35) == 3
    assert ot.rethreshold_quantile(v, 0.75).sum() == 3
