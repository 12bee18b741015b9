"""The compressed 8-wide node layout ("node96q", width 8; P:130
layout, P:297 memory-conscious traversal) — built by the SAH collapse of the Karras tree
(csrc/wide.cu) and traversed by the persistent cast kernel:

* tree validity, decoded from the exported node bytes: every triangle in exactly one leaf of at
  most 3 triangles (a contiguous range of the Morton order), every decoded 8-bit child box
  (p + q 2^e, rounded outward) contains the exact box of the child's triangles, and the cast's
  stack bound holds;
* cast parity against the CPU ORACLE (mode B, the kernel's exact float32 rays) on C1 (all rays),
  C2, C3, C4 and C5 samples, random rays through a soup with a ragged last tile, degenerate
  meshes (T = 1, 2, 3), and after a refit — the same gate as the binary layout
  (tests/test_gpu_cast.py)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fgl():
    import paper_2509_17390_b200 as f
    f.lib()
    return f


def _parity(verdict, rng, tid, max_amb=0.01, label=""):
    j = oracle.judge(verdict, rng, tid)
    msg = f"{label}: n={j['n']} ambiguous={j['ambiguous']} unamb_mismatch={len(j['unamb_mismatch'])} " \
          f"amb_outside={len(j['amb_outside'])}"
    assert len(j["unamb_mismatch"]) == 0, msg
    assert len(j["amb_outside"]) == 0, msg
    assert j["ambiguous"] / max(j["n"], 1) <= max_amb, msg
    return j


def decode_node96q(buf: np.ndarray, n: int):
    """(lo[8][3], hi[8][3] in float64 exactly, refs[8], valid mask) of wide node n."""
    b = buf.view(np.uint8).reshape(-1)[96 * n:96 * n + 96]
    f = b[:16].view(np.float32)
    meta = int(b[12:16].view(np.uint32)[0])
    q = b[16:64]
    refs = b[64:96].view(np.int32).copy()
    lo = np.zeros((8, 3))
    hi = np.zeros((8, 3))
    for a in range(3):
        E = (meta >> (8 * a)) & 0xFF
        step = np.ldexp(1.0, E - 142)
        ql = q[16 * a:16 * a + 8]
        qh = q[16 * a + 8:16 * a + 16]
        lo[:, a] = float(f[a]) + ql.astype(np.float64) * step
        hi[:, a] = float(f[a]) + qh.astype(np.float64) * step
    valid = (meta >> 24) & 0xFF
    return lo, hi, refs, valid


def check_tree(fgl, scene, T):
    e = scene.export()
    buf = e["nodes4"]
    tri = e["tri48"].reshape(T, 12).astype(np.float64)
    tv = tri[:, [0, 1, 2, 4, 5, 6, 8, 9, 10]].reshape(T, 3, 3)
    tlo, thi = tv.min(1), tv.max(1)
    cover = np.zeros(T, np.int32)
    n_nodes = 0
    max_need = 0

    def visit(n, need):
        nonlocal n_nodes, max_need
        n_nodes += 1
        lo, hi, refs, valid = decode_node96q(buf, n)
        nvalid = bin(valid).count("1")
        assert nvalid >= 1
        max_need = max(max_need, need + nvalid)
        box_lo, box_hi = np.full(3, np.inf), np.full(3, -np.inf)
        for k in range(8):
            if not (valid >> k) & 1:
                assert refs[k] == np.iinfo(np.int32).min
                continue
            r = int(refs[k])
            if r >= 0:
                clo, chi = visit(r, need + nvalid - 1)
            else:
                v = ~r
                first, cnt = v >> 3, (v & 7) + 1
                assert 1 <= cnt <= 3
                cover[first:first + cnt] += 1
                clo, chi = tlo[first:first + cnt].min(0), thi[first:first + cnt].max(0)
            assert np.all(lo[k] <= clo) and np.all(hi[k] >= chi), (n, k, lo[k], clo, hi[k], chi)
            box_lo, box_hi = np.minimum(box_lo, clo), np.maximum(box_hi, chi)
        return box_lo, box_hi

    import sys
    sys.setrecursionlimit(10000)
    visit(0, 0)
    assert np.all(cover == 1), (np.sum(cover == 0), np.sum(cover > 1))
    assert n_nodes <= max(T - 1, 1)
    return n_nodes, max_need


@pytest.mark.parametrize("name", ["tiny1", "tiny2", "tiny3", "dups", "c1", "soup"])
def test_node96q_tree_valid(fgl, name):
    meshes = {
        "tiny1": synth.Mesh(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 2]], np.float32), np.array([[0, 1, 2]], np.int32)),
        "tiny2": synth.Mesh(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]], np.float32),
                            np.array([[0, 1, 2], [1, 3, 2]], np.int32)),
        "tiny3": synth.Mesh(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0], [2, 0, 1]], np.float32),
                            np.array([[0, 1, 2], [1, 3, 2], [1, 4, 3]], np.int32)),
        "dups": synth.Mesh(np.tile(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], np.float32), (50, 1)),
                           np.arange(150, dtype=np.int32).reshape(50, 3)),
        "c1": synth.scene_c1(),
        "soup": synth.soup(20011, seed=7),
    }
    m = meshes[name]
    s = fgl.Scene(m.verts, m.tris, width=8)
    n_nodes, need = check_tree(fgl, s, m.T)
    assert need <= 192
    # a wide tree over T triangles needs at least T / 24 nodes (8 leaves of <= 3 triangles each)
    assert n_nodes >= (m.T + 23) // 24


def _mode_b(fgl, cfg, n_sample, seed, first_frame=0, scene=None):
    m, pat, poses = cfg["mesh"], cfg["pattern"], cfg["poses"]
    s = scene or fgl.Scene(m.verts, m.tris, width=8)
    res = s.cast(poses, pat, first_frame=first_frame)
    rng = res["range"].reshape(-1).cpu().numpy()
    tid = res["tri_id"].reshape(-1).cpu().numpy()
    idx = np.arange(rng.size) if n_sample >= rng.size else \
        np.sort(np.random.default_rng(seed).choice(rng.size, n_sample, replace=False))
    o, d = fgl.export_rays(pat, poses, first_frame=first_frame)
    o = o.cpu().numpy().astype(np.float64)[idx]
    d = d.cpu().numpy().astype(np.float64)[idx]
    v = oracle.cast_and_classify(m.verts, m.tris, o, d, pat.t_min, pat.t_max, eps_rel=oracle.EPS_MODE_B)
    return v, rng[idx], tid[idx], s


@pytest.mark.parametrize("name,kw,n,ff", [("C1", {}, 10 ** 9, 0), ("C2", {"poses": 2}, 4096, 0),
                                          ("C3", {}, 2048, 0), ("C4", {"poses": 5}, 1500, 17),
                                          ("C5", {"poses": 4}, 1024, 0)])
def test_width8_oracle_parity(fgl, name, kw, n, ff):
    cfg = synth.config(name, **kw)
    v, rng, tid, s = _mode_b(fgl, cfg, n, seed=11, first_frame=ff)
    _parity(v, rng, tid, label=f"{name} width 8")
    s.check()


def test_width8_soup_random_rays_ragged(fgl):
    m = synth.soup(100_000, seed=7)
    s = fgl.Scene(m.verts, m.tris, width=8)
    rng = np.random.default_rng(1)
    R = 1000 + 17
    o = rng.uniform(-2, 12, size=(R, 3)).astype(np.float32)
    tgt = m.verts[m.tris[rng.integers(0, m.T, R)]].mean(1)
    d = tgt - o
    d = (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)
    r, t = s.cast_rays(o, d, 0.0, 1e3)
    v = oracle.cast_and_classify(m.verts, m.tris, o.astype(np.float64), d.astype(np.float64), 0.0, 1e3)
    _parity(v, r.cpu().numpy(), t.cpu().numpy(), max_amb=0.05, label="soup width 8")


@pytest.mark.parametrize("T", [1, 2, 3, 5])
def test_width8_tiny_meshes(fgl, T):
    rng = np.random.default_rng(T)
    v = rng.uniform(-1, 1, size=(3 * T, 3)).astype(np.float32)
    v[:, 0] += 3.0
    m = synth.Mesh(v, np.arange(3 * T, dtype=np.int32).reshape(T, 3))
    s = fgl.Scene(m.verts, m.tris, width=8)
    check_tree(fgl, s, T)
    R = 4096
    o = np.zeros((R, 3), np.float32)
    d = rng.normal(size=(R, 3))
    d[:, 0] = np.abs(d[:, 0]) * 4
    d = (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)
    r, t = s.cast_rays(o, d, 0.0, 1e3)
    vv = oracle.cast_and_classify(m.verts, m.tris, o.astype(np.float64), d.astype(np.float64), 0.0, 1e3)
    _parity(vv, r.cpu().numpy(), t.cpu().numpy(), max_amb=0.05, label=f"T={T} width 8")


def test_width8_refit(fgl):
    cfg = synth.config("C1")
    m = cfg["mesh"]
    s = fgl.Scene(m.verts, m.tris, width=8)
    rng = np.random.default_rng(5)
    v2 = (m.verts + rng.normal(scale=0.05, size=m.verts.shape)).astype(np.float32)
    s.refit(v2)
    check_tree(fgl, s, m.T)
    cfg2 = dict(cfg)
    cfg2["mesh"] = synth.Mesh(v2, m.tris)
    v, rng_, tid, _ = _mode_b(fgl, cfg2, 10 ** 9, 0, scene=s)
    _parity(v, rng_, tid, label="C1 refit width 8")


def test_width8_hit_points_counts_and_determinism(fgl):
    """Optional outputs of the width-8 cast: hit points x* = o + t d, the Eq. 21 counters,
    and bitwise determinism across casts."""
    cfg = synth.config("C1")
    m, pat, poses = cfg["mesh"], cfg["pattern"], cfg["poses"]
    s = fgl.Scene(m.verts, m.tris, width=8)
    r = s.cast(poses, pat, hit_xyz=True, counts=True)
    r2 = s.cast(poses, pat)
    assert np.array_equal(r["range"].cpu().numpy().view(np.int32), r2["range"].cpu().numpy().view(np.int32))
    assert np.array_equal(r["tri_id"].cpu().numpy(), r2["tri_id"].cpu().numpy())
    o, d = fgl.export_rays(pat, poses)
    rng = r["range"].reshape(-1).cpu().numpy().astype(np.float64)
    x = r["hit_xyz"].reshape(-1, 3).cpu().numpy().astype(np.float64)
    exp = o.cpu().numpy().astype(np.float64) + rng[:, None] * d.cpu().numpy().astype(np.float64)
    assert np.allclose(x, exp, rtol=0, atol=1e-5 + 1e-6 * np.abs(exp).max())
    nc = r["node_counts"].cpu().numpy()
    assert nc.min() >= 1 and nc.mean() < 20  # wide nodes: few visits per ray on C1
    assert r["tri_counts"].cpu().numpy().min() >= 1
