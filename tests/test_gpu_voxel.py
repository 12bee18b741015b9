"""GPU parity of the Gaussian -> occupancy path (Eqs. 4, 8-12)
against oracle/gauss.py, through the C ABI (paper_2509_17390_b200.GaussianScene)."""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import gauss as og

pytestmark = pytest.mark.gpu

fgl = pytest.importorskip("paper_2509_17390_b200")


def _vox(g, grid, theta, kappa=3.0, **kw):
    gs = fgl.GaussianScene(g.mu, g.quat, g.scale, g.opacity, kappa=kappa)
    r = gs.voxelize(grid.origin, grid.h, grid.dims, theta, density=True, **kw)
    torch.cuda.synchronize()
    out = {k: v.cpu().numpy() for k, v in r.items()}
    out["scene"] = gs
    return out


def _check_against_oracle(g, grid, theta, kappa=3.0, max_marginal=0.01):
    r = _vox(g, grid, theta, kappa)
    D, fsum, marg = og.density(g, grid, kappa)
    tol = og.tol_density(fsum) + marg
    Dg = r["density"].astype(np.float64)
    bad = np.abs(Dg - D) > tol
    assert not bad.any(), (int(bad.sum()), float(np.abs(Dg - D).max()))
    Vg = og.unpack_bits(r["occupancy"].view(np.uint32), grid.dims)
    Vo = og.occupancy(D, theta)
    marginal = np.abs(D - theta) <= tol
    assert np.array_equal(Vg[~marginal], Vo[~marginal])
    assert marginal.mean() <= max_marginal
    # the GPU thresholds its own density (Eq. 10) exactly
    assert np.array_equal(Vg, r["density"] > np.float32(theta))
    # Eqs. 11-12 are integer work: bit-exact against the oracle masks of the GPU's V
    Sg = og.unpack_bits(r["surface"].view(np.uint32), grid.dims)
    Ig = og.unpack_bits(r["interior"].view(np.uint32), grid.dims)
    assert np.array_equal(Ig, og.interior(Vg)) and np.array_equal(Sg, og.surface(Vg))
    c = r["counts"]
    assert c[0] == Vg.sum() and c[1] == Sg.sum() and c[3] == 0
    # padding bits of the last word of each row stay zero
    nx = grid.dims[0]
    if nx % 32:
        assert not np.any(r["occupancy"].view(np.uint32)[..., -1] >> np.uint32(nx % 32))
    return r, D, Vo


def test_g1_parity():
    cfg = synth.gauss_config("G1")
    r, D, Vo = _check_against_oracle(cfg["gauss"], cfg["grid"], cfg["theta"], cfg["kappa"])
    assert Vo.sum() > 1000 and (~Vo).sum() > 1000  # a non-trivial occupancy
    assert r["counts"][2] > 0


@pytest.mark.parametrize("dims", [(37, 29, 13), (1, 1, 1), (33, 8, 9), (70, 3, 17)])
def test_ragged_grids(dims):
    g = synth.gaussians_random(300, 21, extent=2.0, scale_median=0.12)
    h = 2.2 / max(dims)
    grid = synth.Grid((-0.1, -0.1, -0.1), float(np.float32(h)), dims)
    _check_against_oracle(g, grid, 0.4)


@pytest.mark.parametrize("kappa", [1.0, 2.0, 3.0])
def test_kappa(kappa):
    g = synth.gaussians_random(400, 22, extent=2.0, scale_median=0.1)
    _check_against_oracle(g, synth.grid_for(g, 40), 0.3, kappa)


def test_surface_splats_parity():
    m = synth.merge([synth.box((0.0, 0.0, 0.0), (2.0, 1.5, 1.0), 0.1), synth.icosphere(2, 0.4, (1.0, 0.7, 1.5))])
    g = synth.gaussians_on_mesh(m, 20000, 23)
    _check_against_oracle(g, synth.grid_for(g, 96), 0.5)


def test_single_gaussian_closed_form():
    g = synth.Gaussians(np.zeros((1, 3), np.float32), np.array([[1, 0, 0, 0]], np.float32),
                        np.ones((1, 3), np.float32), np.array([0.8], np.float32))
    grid = synth.Grid((-2.0, -2.0, -2.0), 0.25, (16, 16, 16))
    r = _vox(g, grid, 0.5)
    V = og.unpack_bits(r["occupancy"].view(np.uint32), grid.dims)
    rad = np.linalg.norm(og.centers(grid.origin, grid.h, grid.dims), axis=-1)
    assert np.array_equal(V, rad < math.sqrt(2 * math.log(0.8 / 0.5)))


def test_threshold_extremes_and_outside():
    g = synth.gaussians_random(200, 24, extent=1.0, scale_median=0.1)
    grid = synth.grid_for(g, 20)
    r = _vox(g, grid, float(g.opacity.sum()) + 1.0)
    assert not r["occupancy"].any() and r["counts"][0] == 0
    r = _vox(g, grid, -1.0)  # D >= 0 > theta everywhere: full grid, interior = all but the boundary
    V = og.unpack_bits(r["occupancy"].view(np.uint32), grid.dims)
    I = og.unpack_bits(r["interior"].view(np.uint32), grid.dims)
    nx, ny, nz = grid.dims
    assert V.all() and I.sum() == (nx - 2) * (ny - 2) * (nz - 2)
    far = synth.Grid((100.0, 100.0, 100.0), grid.h, grid.dims)  # every Gaussian is outside the grid
    r = _vox(g, far, 0.1)
    assert not r["occupancy"].any() and not r["density"].any() and r["counts"][2] == 0


def test_deterministic():
    cfg = synth.gauss_config("G1")
    a = _vox(cfg["gauss"], cfg["grid"], 0.5)
    b = _vox(cfg["gauss"], cfg["grid"], 0.5)
    assert np.array_equal(a["density"].view(np.uint32), b["density"].view(np.uint32))
    assert np.array_equal(a["occupancy"], b["occupancy"])


def test_eq4_boxes_conservative():
    g = synth.gaussians_random(500, 25)
    gs = fgl.GaussianScene(g.mu, g.quat, g.scale, g.opacity, kappa=3.0)
    ex = gs.scene.export()
    lo, hi = og.aabb(g.mu, g.quat, g.scale, 3.0)
    perm = ex["perm"].astype(np.int64)
    lb = ex["leaf_box"].astype(np.float64)
    assert np.all(lb[:, :3] <= lo[perm]) and np.all(lb[:, 3:] >= hi[perm])
    ext = hi[perm] - lo[perm]
    assert np.all(lo[perm] - lb[:, :3] <= 1e-5 * ext + 1e-6) and np.all(lb[:, 3:] - hi[perm] <= 1e-5 * ext + 1e-6)
    # the tree over the boxes is a valid Eq. 6-7 hierarchy: every node box is the union of its leaves
    nb, rng = ex["node_box"], ex["range"]
    for i in range(0, len(rng), 37):
        a, b = rng[i]
        assert np.array_equal(nb[i, :3], lb[a:b + 1, :3].min(axis=0).astype(np.float32))
        assert np.array_equal(nb[i, 3:], lb[a:b + 1, 3:].max(axis=0).astype(np.float32))


def test_errors():
    g = synth.gaussians_random(10, 26)
    bad = g.scale.copy()
    bad[3, 1] = 0.0
    with pytest.raises(fgl.FglError) as e:
        fgl.GaussianScene(g.mu, g.quat, bad, g.opacity)
    assert e.value.status == 2
    op = g.opacity.copy()
    op[0] = 1.5
    with pytest.raises(fgl.FglError):
        fgl.GaussianScene(g.mu, g.quat, g.scale, op)
    with pytest.raises(fgl.FglError):
        fgl.GaussianScene(g.mu, g.quat, g.scale, g.opacity, kappa=0.5)
    gs = fgl.GaussianScene(g.mu, g.quat, g.scale, g.opacity)
    pat = synth.spinning_preset("VLP16")
    with pytest.raises(fgl.FglError) as e:
        gs.scene.cast(synth.pose((0, 0, 0))[None], pat)
    assert e.value.status == 1
    m = synth.scene_c1()
    sc = fgl.Scene(m.verts, m.tris)
    assert fgl.lib().fgl_voxelize(sc._h, None, None, None, None, None, None, None) == 1


def test_g2_full_size_sampled():
    """Full G2 (1 M surface splats, 512 voxels on the long axis): sampled voxel densities against
    the oracle one by one, plus whole-volume invariants."""
    cfg = synth.gauss_config("G2")
    g, grid, theta = cfg["gauss"], cfg["grid"], cfg["theta"]
    gs = fgl.GaussianScene(g.mu, g.quat, g.scale, g.opacity, kappa=cfg["kappa"])
    r = gs.voxelize(grid.origin, grid.h, grid.dims, theta, density=True)
    torch.cuda.synchronize()
    dens = r["density"]
    occ = r["occupancy"].cpu().numpy().view(np.uint32)
    nx, ny, nz = grid.dims
    rng = np.random.default_rng(5)
    flat = dens.reshape(-1)
    hot = torch.nonzero(flat > 0.05).reshape(-1).cpu().numpy()
    idx = np.concatenate([rng.choice(hot, 150, replace=False), rng.integers(0, flat.numel(), 50)])
    k, rem = np.divmod(idx, nx * ny)
    j, i = np.divmod(rem, nx)
    pts = np.stack([grid.origin[0] + (i + 0.5) * grid.h, grid.origin[1] + (j + 0.5) * grid.h,
                    grid.origin[2] + (k + 0.5) * grid.h], axis=1)
    D, fsum, marg = og.density_at(g, pts, cfg["kappa"])
    Dg = flat[torch.from_numpy(idx).to(flat.device)].cpu().numpy().astype(np.float64)
    assert np.all(np.abs(Dg - D) <= og.tol_density(fsum) + marg)
    V = og.unpack_bits(occ, grid.dims)
    c = r["counts"].cpu().numpy()
    assert c[0] == V.sum() and c[3] == 0 and 0.001 < V.mean() < 0.5
    S = og.unpack_bits(r["surface"].cpu().numpy().view(np.uint32), grid.dims)
    I = og.unpack_bits(r["interior"].cpu().numpy().view(np.uint32), grid.dims)
    assert np.array_equal(S | I, V) and not (S & I).any() and c[1] == S.sum()
    assert np.array_equal(I, og.interior(V))
