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
