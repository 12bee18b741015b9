"""GPU parity of the occupancy -> mesh path (Eqs. 13-18) against
oracle/tsdf.py, through the C ABI (paper_2509_17390_b200.denoise / tsdf / marching_cubes)."""
import numpy as np
import pytest
import torch
from scipy import ndimage

import synth
from oracle import gauss as og
from oracle import tsdf as ot

pytestmark = pytest.mark.gpu

fgl = pytest.importorskip("paper_2509_17390_b200")


def _pack(V):
    """bool [nz][ny][nx] -> device bit volume uint32 [nz][ny][ceil(nx/32)] (test helper)."""
    nz, ny, nx = V.shape
    nw = (nx + 31) // 32
    P = np.zeros((nz, ny, nw * 32), bool)
    P[..., :nx] = V
    b = np.packbits(P.reshape(nz, ny, nw * 4, 8), axis=-1, bitorder="little").reshape(nz, ny, nw * 4)
    return torch.from_numpy(b.view(np.int32).copy()).cuda()


def _volumes():
    rng = np.random.default_rng(0)
    out = []
    out.append(ndimage.binary_closing(rng.uniform(size=(20, 23, 37)) < 0.45))  # ragged nx
    V = np.zeros((12, 13, 40), bool)
    V[2:10, 2:11, 3:30] = True
    V[4:8, 4:9, 6:20] = False  # hollow box with a cavity
    out.append(V)
    g = np.arange(33) + 0.5 - 16.5
    Z, Y, X = np.meshgrid(g, g, g, indexing="ij")
    out.append(X * X + Y * Y + Z * Z <= 12.2 ** 2)  # ball touching nothing
    out.append(rng.uniform(size=(7, 5, 70)) < 0.6)  # noisy, thin in z
    out.append(np.ones((4, 4, 4), bool))  # full grid
    out.append(np.zeros((3, 5, 33), bool))  # empty grid
    W = rng.uniform(size=(3, 4, 1100)) < 0.97  # long rows: 35 words (> one warp), long free runs
    W[1, 2, 40:1060] = False
    out.append(W)
    return out


@pytest.mark.parametrize("case", range(7))
def test_tsdf_bit_exact(case):
    V = _volumes()[case]
    nz, ny, nx = V.shape
    for sp, r in (((0.1, 0.1, 0.1), 0.3), ((0.05, 0.1, 0.2), 0.22)):
        phi = fgl.tsdf(_pack(V), (nx, ny, nz), sp, r).cpu().numpy()
        ref, _ = ot.tsdf(V, sp, r)
        assert np.array_equal(phi.view(np.uint32), ref.view(np.uint32)), (case, sp)


@pytest.mark.parametrize("sigma_vox,shape", [(0.6, (18, 21, 45)), (0.9, (7, 9, 64)), (1.2, (5, 40, 33)),
                                             (1.5, (18, 21, 45)), (0.3, (3, 4, 97))])
def test_denoise_parity(sigma_vox, shape):
    # R = ceil(3 sigma) = 2, 3, 4 (word-per-thread x pass, full / ragged last words), 5 (gather x pass), 1
    rng = np.random.default_rng(1)
    V = rng.uniform(size=shape) < 0.5
    nz, ny, nx = V.shape
    h = 0.05
    tau = 0.5
    out, vp = fgl.denoise(_pack(V), (nx, ny, nz), (h, h, h), sigma_vox * h, tau, vprime=True)
    ref = ot.blur(V, sigma_vox * h, (h, h, h))
    assert np.max(np.abs(vp.cpu().numpy() - ref)) < 1e-5
    Vg = og.unpack_bits(out.cpu().numpy().view(np.uint32), (nx, ny, nz))
    marginal = np.abs(ref - tau) <= 1e-5
    assert np.array_equal(Vg[~marginal], ot.rethreshold(ref, tau)[~marginal])
    assert np.array_equal(Vg, vp.cpu().numpy() >= tau)  # the GPU thresholds its own V' exactly


def _mc_compare(phi, origin, sp, iso=0.0):
    phi_d = torch.from_numpy(np.ascontiguousarray(phi, np.float32)).cuda()
    r = fgl.marching_cubes(phi_d, origin, sp, iso, normals=True)
    V, T, N = ot.marching_cubes(phi, origin, sp, iso, normals=True)
    vg, tg, ng = (r[k].cpu().numpy() for k in ("verts", "tris", "normals"))
    assert tg.shape == T.shape and np.array_equal(tg, T)
    assert vg.shape == V.shape
    ext = float(np.max(np.asarray(sp) * np.asarray(phi.shape[::-1]))) + float(np.max(np.abs(origin)))
    assert np.max(np.abs(vg - V), initial=0.0) <= 2e-6 * ext
    ok = np.linalg.norm(N, axis=1) > 0.5
    assert np.max(np.abs(ng[ok] - N[ok]), initial=0.0) < 1e-3
    return vg, tg


def test_mc_all_cube_cases():
    # every 8-corner pattern once, each in its own padded cell of one grid
    phi = np.ones((4, 4, 4 * 256), np.float32)
    for case in range(256):
        for c in range(8):
            if (case >> c) & 1:
                phi[1 + ((c >> 2) & 1), 1 + ((c >> 1) & 1), 4 * case + 1 + (c & 1)] = -1.0
    _mc_compare(phi, (0.0, 0.0, 0.0), (1.0, 1.0, 1.0))


def test_mc_sphere_and_random_fields():
    n, R = 29, 10.3
    g = np.arange(n) + 0.5 - n / 2
    Z, Y, X = np.meshgrid(g, g, g, indexing="ij")
    _mc_compare((np.sqrt(X * X + Y * Y + Z * Z) - R).astype(np.float32), (-1.5, 2.0, 0.25), (0.1, 0.1, 0.1))
    rng = np.random.default_rng(4)
    phi = rng.normal(size=(9, 11, 47)).astype(np.float32)
    _mc_compare(phi, (0.0, 0.0, 0.0), (0.2, 0.1, 0.05), iso=0.1)


@pytest.mark.parametrize("case", [0, 1, 2, 3])
def test_tsdf_then_mc(case):
    V = _volumes()[case]
    nz, ny, nx = V.shape
    sp = (0.1, 0.1, 0.1)
    phi = fgl.tsdf(_pack(V), (nx, ny, nz), sp, 0.3).cpu().numpy()
    vg, tg = _mc_compare(phi, (1.0, -2.0, 0.5), sp)
    if case in (1, 2):  # surfaces inside the grid: closed, consistently oriented
        e = np.concatenate([tg[:, [0, 1]], tg[:, [1, 2]], tg[:, [2, 0]]])
        fwd = set(map(tuple, e))
        assert len(fwd) == len(e) and all((b, a) in fwd for a, b in fwd)


def test_mc_counts_and_capacity():
    n, R = 21, 7.1
    g = np.arange(n) + 0.5 - n / 2
    Z, Y, X = np.meshgrid(g, g, g, indexing="ij")
    phi = torch.from_numpy((np.sqrt(X * X + Y * Y + Z * Z) - R).astype(np.float32)).cuda()
    full = fgl.marching_cubes(phi, (0, 0, 0), (1, 1, 1))
    nv, nt = full["verts"].shape[0], full["tris"].shape[0]
    small = dict(verts=torch.full((10, 3), -7.0, device="cuda"), tris=torch.full((5, 3), -7, dtype=torch.int32,
                                                                               device="cuda"),
                 counts=torch.zeros(2, dtype=torch.int64, device="cuda"))
    fgl.marching_cubes(phi, (0, 0, 0), (1, 1, 1), out=small)
    assert small["counts"].tolist() == [nv, nt]
    assert torch.equal(small["verts"], full["verts"][:10]) and torch.equal(small["tris"], full["tris"][:5])


def test_gaussians_to_mesh_to_cast():
    """The paper's pipeline end to end on the GPU: 3DGS -> occupancy -> TSDF -> MC mesh -> LBVH ->
    cast; the mesh is closed and every beam from a point far outside hits it or misses it exactly
    as the oracle cast of the same mesh says."""
    g = synth.gaussians_on_mesh(synth.icosphere(3, 1.0), 30000, 31, tangent_median=0.05, normal_scale=0.03)
    grid = synth.grid_for(g, 48, pad=3)
    gs = fgl.GaussianScene(g.mu, g.quat, g.scale, g.opacity)
    occ = gs.voxelize(grid.origin, grid.h, grid.dims, 0.3, masks=False)["occupancy"]
    sp = (grid.h,) * 3
    phi = fgl.tsdf(occ, grid.dims, sp, 3 * grid.h)
    m = fgl.marching_cubes(phi, grid.origin, sp)
    verts, tris = m["verts"], m["tris"]
    tg = tris.cpu().numpy()
    e = np.concatenate([tg[:, [0, 1]], tg[:, [1, 2]], tg[:, [2, 0]]])
    fwd = set(map(tuple, e))
    assert len(fwd) == len(e) and all((b, a) in fwd for a, b in fwd)  # watertight, oriented
    sc = fgl.Scene(verts, tris)
    pat = synth.spinning_preset("VLP16")
    pose = synth.pose((0.0, 0.0, 0.05))  # the sphere's centre: every beam must hit the closed mesh
    res = sc.cast(pose[None], pat)
    assert torch.all(res["tri_id"] >= 0)
    rng = res["range"].cpu().numpy()
    assert np.all((rng > 0.6) & (rng < 1.4))


@pytest.mark.parametrize("q", [0.0, 0.3, 0.75, 0.98, 1.0])
def test_denoise_quantile(q):
    rng = np.random.default_rng(2)
    V = rng.uniform(size=(17, 19, 41)) < 0.4
    nz, ny, nx = V.shape
    h = 0.05
    out, thr, vp = fgl.denoise_quantile(_pack(V), (nx, ny, nz), (h, h, h), 0.9 * h, q, vprime=True)
    vpn = vp.cpu().numpy()
    # the selection is exact on the GPU's own float32 V' (same decision, same precision)
    assert thr.item() == ot.quantile(vpn, q)
    Vg = og.unpack_bits(out.cpu().numpy().view(np.uint32), (nx, ny, nz))
    assert np.array_equal(Vg, ot.rethreshold_quantile(vpn, q))
    ref = ot.blur(V, 0.9 * h, (h, h, h))
    assert np.max(np.abs(vpn - ref)) < 1e-5
