"""NEXT-4 refit for deforming meshes (fgl_scene_refit): the kept tree gets the exact Eq. 7 boxes of
the new positions (bit-exact against the oracle's post-order refit on the same leaf order and
topology), and casts on the refitted scene meet the oracle's acceptance on the deformed mesh."""
import math

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


def _deform(verts, amp, phase=0.0):
    v = verts.astype(np.float64)
    d = np.stack([np.sin(0.7 * v[:, 1] + phase), np.cos(0.5 * v[:, 2] - phase), np.sin(0.3 * v[:, 0] + 2 * phase)], 1)
    return (v + amp * d).astype(np.float32)


@pytest.mark.parametrize("width,quant", [(2, 0), (4, 0), (4, 1)])
def test_refit_boxes_exact(fgl, width, quant):
    m = synth.soup(20000, seed=3)
    s = fgl.Scene(m.verts, m.tris, width=width, quantized=quant)
    e0 = s.export()
    v2 = _deform(m.verts, 0.2)
    s.refit(v2)
    e1 = s.export()
    assert np.array_equal(e1["perm"], e0["perm"]) and np.array_equal(e1["child"], e0["child"])
    leaf, node = oracle.refit(v2, m.tris, e0["perm"], e0["child"])
    assert np.array_equal(e1["leaf_box"], leaf) and np.array_equal(e1["node_box"], node)
    assert not np.array_equal(e1["node_box"], e0["node_box"])


def test_refit_cast_parity_c1(fgl):
    cfg = synth.config("C1")
    m, pat, poses = cfg["mesh"], cfg["pattern"], cfg["poses"]
    s = fgl.Scene(m.verts, m.tris)
    for k, amp in enumerate((0.05, 0.3, 1.0)):
        v2 = _deform(m.verts, amp, phase=0.3 * k)
        s.refit(v2)
        res = s.cast(poses, pat)
        rng = res["range"].reshape(-1).cpu().numpy()
        tid = res["tri_id"].reshape(-1).cpu().numpy()
        o, d = fgl.export_rays(pat, poses)
        vd = oracle.cast_and_classify(v2, m.tris, o.cpu().numpy().astype(np.float64),
                                      d.cpu().numpy().astype(np.float64), pat.t_min, pat.t_max,
                                      eps_rel=oracle.EPS_MODE_B)
        j = oracle.judge(vd, rng, tid)
        assert len(j["unamb_mismatch"]) == 0 and len(j["amb_outside"]) == 0
        assert j["ambiguous"] <= 0.01 * j["n"]


def test_refit_rooms_sampled_and_matches_rebuild(fgl):
    m = synth.scene_rooms(2)
    s = fgl.Scene(m.verts, m.tris)
    v2 = _deform(m.verts, 0.02)
    s.refit(v2)
    fresh = fgl.Scene(v2, m.tris)
    pat = synth.spinning_preset("HDL64")
    poses = synth.poses_yaw_offsets((9.0, 7.5, 1.5), 2, 0.01)
    a = s.cast(poses, pat)
    b = fresh.cast(poses, pat)
    # the same first hits through two different trees (rounding-decided rays aside)
    same = (a["tri_id"] == b["tri_id"]).float().mean().item()
    assert same > 0.9999
    assert torch.allclose(a["range"][a["tri_id"] == b["tri_id"]], b["range"][a["tri_id"] == b["tri_id"]])
    st = s.stats()
    assert st["build_ms"] > 0


def test_refit_errors(fgl):
    m = synth.scene_c1()
    s = fgl.Scene(m.verts, m.tris)
    with pytest.raises(fgl.FglError) as e:
        s.refit(m.verts[:-3])
    assert e.value.status == 1
    bad = m.verts.copy()
    bad[5, 1] = math.nan
    with pytest.raises(fgl.FglError) as e:
        s.refit(bad)
    assert e.value.status == 2
    u = fgl.Scene(build=False)
    with pytest.raises(fgl.FglError):
        u.refit(m.verts)


# ---- NEXT-4 treelet restructuring --------------------------------------------------------------
def _tree_checks(ex, T):
    child, nb, lb = ex["child"], ex["node_box"].astype(np.float64), ex["leaf_box"].astype(np.float64)
    seen = np.zeros(T, int)
    stack, depth = [(0, 0)], 0
    lo = np.zeros((T - 1, 3))
    while stack:
        n, d = stack.pop()
        depth = max(depth, d)
        for c in child[n]:
            if c < 0:
                seen[~c] += 1
            else:
                stack.append((c, d + 1))
    assert np.all(seen == 1)  # every triangle exactly once
    # every node box is the union of its two children's boxes (Eq. 7 on the new topology)
    def box(c):
        return lb[~c] if c < 0 else nb[c]
    for n in range(T - 1):
        a, b = box(child[n][0]), box(child[n][1])
        assert np.array_equal(nb[n, :3], np.minimum(a[:3], b[:3])) and np.array_equal(nb[n, 3:], np.maximum(a[3:], b[3:]))
    return depth


@pytest.mark.parametrize("passes", [1, 3, -1, -3, -6])  # < 0: parallel depth-partition passes
def test_restructure_tree_valid_and_cast_parity(fgl, passes):
    cfg = synth.config("C1")
    m, pat, poses = cfg["mesh"], cfg["pattern"], cfg["poses"]
    s = fgl.Scene(m.verts, m.tris, restructure=passes)
    depth = _tree_checks(s.export(), m.T)
    assert depth < 90
    res = s.cast(poses, pat)
    o, d = fgl.export_rays(pat, poses)
    vd = oracle.cast_and_classify(m.verts, m.tris, o.cpu().numpy().astype(np.float64),
                                  d.cpu().numpy().astype(np.float64), pat.t_min, pat.t_max, eps_rel=oracle.EPS_MODE_B)
    j = oracle.judge(vd, res["range"].reshape(-1).cpu().numpy(), res["tri_id"].reshape(-1).cpu().numpy())
    assert len(j["unamb_mismatch"]) == 0 and len(j["amb_outside"]) == 0
    s.check()  # the stack bound of the restructured tree was met (no refused cast)


@pytest.mark.parametrize("passes", [2, -3])
def test_restructure_rooms_same_hits_fewer_nodes(fgl, passes):
    m = synth.scene_rooms(2)
    plain = fgl.Scene(m.verts, m.tris)
    rs = fgl.Scene(m.verts, m.tris, restructure=passes)
    assert _tree_checks(rs.export(), m.T) < 90
    pat = synth.spinning_preset("HDL64")
    poses = synth.poses_yaw_offsets((9.0, 7.5, 1.5), 2, 0.01)
    a = plain.cast(poses, pat, counts=True)
    b = rs.cast(poses, pat, counts=True)
    assert (a["tri_id"] == b["tri_id"]).float().mean().item() > 0.9999
    assert b["node_counts"].float().mean().item() < a["node_counts"].float().mean().item() + 1.5
    # a refit of the restructured tree keeps it exact
    v2 = _deform(m.verts, 0.02)
    rs.refit(v2)
    fresh = fgl.Scene(v2, m.tris)
    c1, c2 = rs.cast(poses, pat), fresh.cast(poses, pat)
    assert (c1["tri_id"] == c2["tri_id"]).float().mean().item() > 0.9999


# ---- bottom-up 4-leaf treelets inside the fused build (fgl_build_opts.treelets) ----------------
def _node64_checks(nodes, tri48, T, leaf_size):
    """Walk the traversal nodes from the root: every triangle reached exactly once, every child box
    the exact union of the triangles below it; returns the tree height (edges to the deepest leaf)."""
    f = nodes.view(np.float32).reshape(-1, 16)
    ii = nodes.view(np.int32).reshape(-1, 16)
    V = tri48.reshape(T, 3, 4)[:, :, :3]
    seen = np.zeros(T, int)

    def walk(n):  # -> (lo, hi, height)
        a, b, c, d = f[n, 0:4], f[n, 4:8], f[n, 8:12], ii[n, 12:16]
        boxes = [np.array([a[0], a[2], c[0], a[1], a[3], c[1]]), np.array([b[0], b[2], c[2], b[1], b[3], c[3]])]
        lo, hi, hh = np.full(3, np.inf, np.float32), np.full(3, -np.inf, np.float32), 0
        for s in range(2):
            ref = int(d[s])
            if ref >= 0:
                l, h, k = walk(ref)
            else:
                v = ~ref
                first, cnt = v >> 3, (v & 7) + 1
                assert cnt <= leaf_size
                seen[first:first + cnt] += 1
                sub = V[first:first + cnt].reshape(-1, 3)
                l, h, k = sub.min(0), sub.max(0), 0
            assert np.array_equal(boxes[s], np.concatenate([l, h]))
            lo, hi, hh = np.minimum(lo, l), np.maximum(hi, h), max(hh, k + 1)
        return lo, hi, hh

    import sys
    sys.setrecursionlimit(10000)
    height = walk(0)[2]
    assert np.all(seen == 1)
    return height


@pytest.mark.parametrize("mesh,leaf_size", [("c1", 2), ("c1", 1), ("soup", 2), ("soup", 4), ("dups", 2)])
def test_treelets_tree_valid_and_cast_parity(fgl, mesh, leaf_size):
    m = {"c1": lambda: synth.scene_c1(), "soup": lambda: synth.soup(20011, seed=3),
         "dups": lambda: synth.Mesh(np.tile(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], np.float32), (1500, 1)),
                                    np.arange(4500, dtype=np.int32).reshape(1500, 3))}[mesh]()
    s = fgl.Scene(m.verts, m.tris, treelets=1, leaf_size=leaf_size)
    ex = s.export()
    assert _tree_checks(ex, m.T) < 90
    height = _node64_checks(ex["nodes"], ex["tri48"], m.T, leaf_size)
    plain = fgl.Scene(m.verts, m.tris, leaf_size=leaf_size).export()
    assert height <= _node64_checks(plain["nodes"], plain["tri48"], m.T, leaf_size) + 40
    if mesh != "c1":
        return
    cfg = synth.config("C1")
    pat, poses = cfg["pattern"], cfg["poses"]
    res = s.cast(poses, pat)
    o, d = fgl.export_rays(pat, poses)
    vd = oracle.cast_and_classify(m.verts, m.tris, o.cpu().numpy().astype(np.float64),
                                  d.cpu().numpy().astype(np.float64), pat.t_min, pat.t_max, eps_rel=oracle.EPS_MODE_B)
    j = oracle.judge(vd, res["range"].reshape(-1).cpu().numpy(), res["tri_id"].reshape(-1).cpu().numpy())
    assert len(j["unamb_mismatch"]) == 0 and len(j["amb_outside"]) == 0
    s.check()


def test_treelets_rooms_same_hits_fewer_nodes(fgl):
    m = synth.scene_rooms(2)
    plain = fgl.Scene(m.verts, m.tris)
    ts = fgl.Scene(m.verts, m.tris, treelets=1)
    pat = synth.spinning_preset("HDL64")
    poses = synth.poses_yaw_offsets((9.0, 7.5, 1.5), 2, 0.01)
    a = plain.cast(poses, pat, counts=True)
    b = ts.cast(poses, pat, counts=True)
    assert (a["tri_id"] == b["tri_id"]).float().mean().item() > 0.9999
    assert torch.allclose(a["range"][a["tri_id"] == b["tri_id"]], b["range"][a["tri_id"] == b["tri_id"]])
    na, nb = a["node_counts"].float().mean().item(), b["node_counts"].float().mean().item()
    ta, tb = a["tri_counts"].float().mean().item(), b["tri_counts"].float().mean().item()
    assert nb + tb < na + ta  # fewer visits + tests per ray
    ts.check()
    # graph-replayed treelet builds are reproducible bit for bit
    e1 = ts.export()
    ts.build()
    e2 = ts.export()
    for k in ("nodes", "tri48", "child"):
        assert e1[k].tobytes() == e2[k].tobytes(), k
    # refit of the treelet tree stays exact
    v2 = _deform(m.verts, 0.02)
    ts.refit(v2)
    fresh = fgl.Scene(v2, m.tris)
    c1, c2 = ts.cast(poses, pat), fresh.cast(poses, pat)
    assert (c1["tri_id"] == c2["tri_id"]).float().mean().item() > 0.9999


def test_treelets_option_errors(fgl):
    m = synth.scene_c1()
    for kw in (dict(treelets=2), dict(treelets=1, width=4), dict(treelets=1, restructure=-2)):
        with pytest.raises(fgl.FglError) as e:
            fgl.Scene(m.verts, m.tris, **kw)
        assert e.value.status == 1, kw
