"""GPU parity of the LBVH build rows (§IV-A, Eqs. 5-7) against the oracle,
through the C ABI: Morton codes, the stable radix sort, the Karras radix tree and the Eq. 7
refit must be bit-exact; the leaf-order triangle records and the traversal nodes are checked
element by element against the oracle's tree."""
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


def _meshes():
    return {
        "tiny1": synth.Mesh(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 2]], np.float32), np.array([[0, 1, 2]], np.int32)),
        "tiny2": synth.Mesh(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]], np.float32),
                            np.array([[0, 1, 2], [1, 3, 2]], np.int32)),
        "dups": synth.Mesh(np.tile(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], np.float32), (50, 1)),
                           np.arange(150, dtype=np.int32).reshape(50, 3)),
        "c1": synth.scene_c1(),
        "soup": synth.soup(20011, seed=7),
    }


def _decode_nodes(nodes, T, leaf_size):
    """Walk the traversal nodes (DESIGN.md §5 node64 layout) from the root; return the list of
    (box of child, ('leaf', first, count) | ('node', idx)) per visited slot, and leaf coverage."""
    f = nodes.view(np.float32).reshape(-1, 16)
    ii = nodes.view(np.int32).reshape(-1, 16)
    cover = np.zeros(T, np.int32)
    out = []
    stack = [0]
    while stack:
        i = stack.pop()
        a, b, c, d = f[i, 0:4], f[i, 4:8], f[i, 8:12], ii[i, 12:16]
        boxes = [np.array([a[0], a[2], c[0], a[1], a[3], c[1]]), np.array([b[0], b[2], c[2], b[1], b[3], c[3]])]
        for s in range(2):
            ref = int(d[s])
            if ref == -2 ** 31:
                continue
            if ref >= 0:
                out.append((boxes[s], ("node", ref)))
                stack.append(ref)
            else:
                v = ~ref
                first, cnt = v >> 3, (v & 7) + 1
                assert cnt <= leaf_size
                cover[first:first + cnt] += 1
                out.append((boxes[s], ("leaf", first, cnt)))
    return out, cover


def _depth_oracle(child, n):
    d = np.zeros(max(n - 1, 0), np.int64)
    stack = [(0, 0)] if n >= 2 else []
    while stack:
        i, k = stack.pop()
        d[i] = k
        for c in child[i]:
            if c >= 0:
                stack.append((c, k + 1))
    return d


def _check_nodes4q(g, o, m, T, leaf_size):
    """8-bit quantised 4-wide nodes (node64q): decoded child boxes contain the exact union of their
    triangles (outward rounding) and are at most one quantum (+ rounding) larger per side."""
    raw = g["nodes4"].view(np.uint8).reshape(-1)
    V = m.verts[m.tris[o["perm"]]]
    cover = np.zeros(T, np.int32)
    stack = [0]
    while stack:
        i = stack.pop()
        rec = raw[64 * i:64 * (i + 1)]
        f0 = rec[:16].view(np.float32)
        bits = int(rec[12:16].view(np.uint32)[0])
        q0 = rec[16:32].view(np.uint32)
        q1 = rec[32:48].view(np.int32)
        q2 = rec[48:64].view(np.int32)
        mask = bits >> 24
        scale = [2.0 ** (((bits >> (8 * a)) & 0xFF) - 127) for a in range(3)]
        qwords = [int(q0[0]), int(q0[1]), int(q0[2]), int(q0[3]), int(q1[0]) & 0xFFFFFFFF, int(q1[1]) & 0xFFFFFFFF]
        refs = [int(q1[2]), int(q1[3]), int(q2[0]), int(q2[1])]
        for k in range(4):
            if not (mask >> k) & 1:
                assert refs[k] == -2 ** 31
                continue
            ref = refs[k]
            if ref >= 0:
                fr, l = o["range"][ref]
                c = l - fr + 1
                stack.append(ref)
            else:
                v = ~ref
                fr, c = v >> 3, (v & 7) + 1
                cover[fr:fr + c] += 1
            sub = V[fr:fr + c].reshape(-1, 3).astype(np.float64)
            for a in range(3):
                qlo = (qwords[2 * a] >> (8 * k)) & 0xFF
                qhi = (qwords[2 * a + 1] >> (8 * k)) & 0xFF
                lo = float(f0[a]) + qlo * scale[a]
                hi = float(f0[a]) + qhi * scale[a]
                assert lo <= sub[:, a].min() and hi >= sub[:, a].max()       # conservative
                assert sub[:, a].min() - lo <= scale[a] * 1.001 + 1e-30       # tight (one quantum)
                assert hi - sub[:, a].max() <= scale[a] * 1.001 + 1e-30
    assert np.all(cover == 1)


def _check_nodes4(g, o, m, T, leaf_size):
    """4-wide nodes (DESIGN.md §5 node128): walk from the root; every child box is the exact union
    of its triangles; leaves cover each sorted position once; internal children are the even-depth
    binary nodes two levels down; depths match the oracle tree."""
    if T >= 2:
        assert np.array_equal(g["depth"], _depth_oracle(o["child"], T))
    f = g["nodes4"].view(np.float32).reshape(-1, 32)
    ii = g["nodes4"].view(np.int32).reshape(-1, 32)
    V = m.verts[m.tris[o["perm"]]]
    cover = np.zeros(T, np.int32)
    stack = [0]
    while stack:
        i = stack.pop()
        refs = ii[i, 24:28]
        assert ii[i, 28] == np.sum(refs != -2 ** 31)
        for k in range(4):
            ref = int(refs[k])
            box = np.array([f[i, 0 + k], f[i, 8 + k], f[i, 16 + k], f[i, 4 + k], f[i, 12 + k], f[i, 20 + k]])
            if ref == -2 ** 31:
                assert np.all(box == np.float32(3.0e38))
                continue
            if ref >= 0:
                fr, l = o["range"][ref]
                c = l - fr + 1
                assert c > leaf_size and g["depth"][ref] % 2 == 0
                stack.append(ref)
            else:
                v = ~ref
                fr, c = v >> 3, (v & 7) + 1
                assert c <= leaf_size or (T == 1)
                cover[fr:fr + c] += 1
            sub = V[fr:fr + c].reshape(-1, 3)
            assert np.array_equal(box, np.concatenate([sub.min(0), sub.max(0)]))
    assert np.all(cover == 1)


@pytest.mark.parametrize("name", ["tiny1", "tiny2", "dups", "c1", "soup"])
@pytest.mark.parametrize("leaf_size,cubic,width,bits,quant", [(1, 0, 2, 21, 0), (4, 0, 2, 16, 0), (8, 0, 2, 10, 0),
                                                              (4, 1, 2, 21, 0), (2, 1, 2, 13, 0), (2, 1, 4, 16, 0),
                                                              (1, 1, 4, 21, 0), (5, 0, 4, 7, 0), (2, 1, 4, 13, 1),
                                                              (4, 0, 4, 21, 1)])
def test_build_matches_oracle(fgl, name, leaf_size, cubic, width, bits, quant):
    m = _meshes()[name]
    s = fgl.Scene(m.verts, m.tris, leaf_size=leaf_size, morton_box=0 if cubic else 1, width=width, morton_bits=bits,
                  quantized=quant)
    g = s.export()
    o = oracle.lbvh(m.verts, m.tris, bits=bits, cubic=bool(cubic))
    T = m.T
    assert np.array_equal(g["scene_box"][:3], o["lo"]) and np.array_equal(g["scene_box"][3:], o["hi"])
    assert np.array_equal(g["codes"], o["code"])                       # Eq. 5
    assert np.array_equal(g["sorted_keys"], o["sorted_keys"])          # sort: keys
    assert np.array_equal(g["perm"], o["perm"])                        # sort: stable order
    assert np.array_equal(g["child"], o["child"])                      # Eq. 6 radix tree
    assert np.array_equal(g["range"], o["range"])
    assert np.array_equal(g["leaf_box"], o["leaf_box"])                # Eq. 7 leaves
    assert np.array_equal(g["node_box"], o["node_box"])                # Eq. 7 unions
    # leaf-order triangle records: exact input vertices + original id
    tri = g["tri48"].reshape(T, 3, 4)
    assert np.array_equal(tri[:, :, :3], m.verts[m.tris[o["perm"]]])
    assert np.array_equal(tri[:, 0, 3].view(np.int32), o["perm"].astype(np.int32))
    # traversal nodes: every reachable child box is the exact union of its triangles, leaves cover
    # every sorted position exactly once
    if width == 4 and quant:
        if T >= 2:
            _check_nodes4q(g, o, m, T, leaf_size)
        return
    if width == 4:
        _check_nodes4(g, o, m, T, leaf_size)
        return
    visited, cover = _decode_nodes(g["nodes"], T, leaf_size)
    assert np.all(cover == 1)
    V = m.verts[m.tris[o["perm"]]]
    for box, ref in visited:
        if ref[0] == "leaf":
            f, c = ref[1], ref[2]
        else:
            f, l = o["range"][ref[1]]
            c = l - f + 1
            assert c > leaf_size
        sub = V[f:f + c].reshape(-1, 3)
        assert np.array_equal(box, np.concatenate([sub.min(0), sub.max(0)]))


@pytest.mark.parametrize("T", [2, 3, 511, 512, 513, 1024, 1025, 4097, 65537])
@pytest.mark.parametrize("leaf_size", [1, 2])
def test_fused_tree_at_chunk_edges(fgl, T, leaf_size):
    """The default width-2 build meets siblings in shared memory inside 512-leaf chunks and through
    global slots across them (k_lbvh): ragged last chunks (one leaf), exact chunk multiples and many
    chunks must give the oracle's Eq. 6 tree and exact Eq. 7 node boxes; duplicated centroids force
    the index tie-break across chunk boundaries."""
    m = synth.soup(T, seed=T)
    if T > 600:  # 600 identical triangles: a run of equal codes that straddles a chunk boundary
        m.verts[:3 * 600] = np.tile(m.verts[:3], (600, 1))
    s = fgl.Scene(m.verts, m.tris, leaf_size=leaf_size)
    g = s.export()
    o = oracle.lbvh(m.verts, m.tris, bits=10, cubic=True)
    for k_g, k_o in (("perm", "perm"), ("child", "child"), ("range", "range"), ("node_box", "node_box")):
        assert np.array_equal(g[k_g], o[k_o]), k_g
    visited, cover = _decode_nodes(g["nodes"], T, leaf_size)
    assert np.all(cover == 1)
    V = m.verts[m.tris[o["perm"]]]
    for box, ref in visited:
        if ref[0] == "leaf":
            f, c = ref[1], ref[2]
        else:
            f, l = o["range"][ref[1]]
            c = l - f + 1
            assert c > leaf_size
        sub = V[f:f + c].reshape(-1, 3)
        assert np.array_equal(box, np.concatenate([sub.min(0), sub.max(0)]))


@pytest.mark.parametrize("T,mode", [(1025, 1), (70001, 1), (70001, 2), (70001, 4), (300007, 6)])
def test_fused_tree_global_fallback(fgl, T, mode, monkeypatch):
    """FGL_LBVH_GLOBAL sends boundary subtrees through the global-slot climb (k_lbvh_top, the path
    taken when a chunk or a group overflows its shared-memory unit budget): every chunk (1), every
    odd chunk (2), every odd group above the chunks (4) — partial overflow poisons everything above
    it — must give the same Eq. 6 tree and node64s as the hierarchical levels."""
    m = synth.soup(T, seed=11)
    a = fgl.Scene(m.verts, m.tris).export()
    monkeypatch.setenv("FGL_LBVH_GLOBAL", str(mode))
    b = fgl.Scene(m.verts, m.tris).export()
    for k in ("child", "range", "nodes", "tri48", "node_box"):
        assert a[k].tobytes() == b[k].tobytes(), k
    o = oracle.lbvh(m.verts, m.tris, bits=10, cubic=True)
    assert np.array_equal(b["child"], o["child"]) and np.array_equal(b["range"], o["range"])


def test_fused_tree_terrain_full_size(fgl, monkeypatch):
    """C3's 10 M-triangle terrain (39 k chunks, 7 levels above them, duplicate codes): every node's
    children tile its leaf range (the radix-tree invariant of Eq. 6), every node but the root has
    one parent, and the tree is bitwise the one the all-global fallback builds."""
    m = synth.scene_terrain(3).mesh
    v, t = torch.from_numpy(m.verts).cuda(), torch.from_numpy(m.tris).cuda()
    a = fgl.Scene(v, t).export()
    child, rng = a["child"].astype(np.int64), a["range"].astype(np.int64)
    lo = np.where(child >= 0, rng[np.maximum(child, 0), 0], ~child)
    hi = np.where(child >= 0, rng[np.maximum(child, 0), 1], ~child)
    assert np.array_equal(lo[:, 0], rng[:, 0]) and np.array_equal(hi[:, 1], rng[:, 1])
    assert np.array_equal(hi[:, 0] + 1, lo[:, 1])
    assert rng[0, 0] == 0 and rng[0, 1] == m.T - 1
    internal = child[child >= 0]
    assert np.array_equal(np.sort(internal), np.arange(1, m.T - 1))
    monkeypatch.setenv("FGL_LBVH_GLOBAL", "1")
    b = fgl.Scene(v, t).export()
    for k in ("child", "range", "nodes", "tri48"):
        assert a[k].tobytes() == b[k].tobytes(), k


def test_build_is_deterministic(fgl):
    m = synth.soup(5000, seed=1)
    a = fgl.Scene(m.verts, m.tris).export()
    b = fgl.Scene(m.verts, m.tris).export()
    for k in a:
        assert a[k].tobytes() == b[k].tobytes(), k  # bitwise (node refs viewed as float may be NaN)


def test_build_rooms_full_size(fgl):
    m = synth.scene_rooms(2)
    s = fgl.Scene(m.verts, m.tris)
    g = s.export()
    o = oracle.lbvh(m.verts, m.tris, bits=10, cubic=True)  # library defaults below 2^22: b = 10, cubic box (R7, R22)
    for k_g, k_o in (("codes", "code"), ("sorted_keys", "sorted_keys"), ("perm", "perm"), ("child", "child"),
                     ("range", "range"), ("leaf_box", "leaf_box"), ("node_box", "node_box")):
        assert np.array_equal(g[k_g], o[k_o]), k_g
    st = s.stats()
    assert st["triangles"] == m.T and st["build_ms"] > 0 and st["morton_bits"] == 10


@pytest.mark.parametrize("n", [0, 1, 2, 3, 4095, 4096, 4097, 100_003, 1_000_000, 5_000_011])
@pytest.mark.parametrize("bits", [8, 30, 63, 64])
def test_sort_pairs_matches_oracle(fgl, n, bits):
    rng = np.random.default_rng(n + bits)
    hi = 2 ** bits if bits < 64 else 2 ** 64
    keys = rng.integers(0, min(hi, 2 ** 63), size=n, dtype=np.uint64)
    if bits == 64:
        keys |= (rng.integers(0, 2, size=n).astype(np.uint64) << np.uint64(63))
    if n > 10:
        keys[: n // 3] = keys[n // 3: 2 * (n // 3)]  # plenty of duplicates
    vals = np.arange(n, dtype=np.uint32)
    k = torch.from_numpy(keys.view(np.int64).copy()).cuda()
    v = torch.from_numpy(vals.view(np.int32).copy()).cuda()
    fgl.sort_pairs(k, v, key_bits=bits)
    sk, perm = oracle.stable_sort(keys)
    assert np.array_equal(k.cpu().numpy().view(np.uint64), sk)
    assert np.array_equal(v.cpu().numpy().view(np.uint32), perm)


def test_morton_primitive_matches_oracle(fgl):
    rng = np.random.default_rng(5)
    pts = rng.normal(size=(50000, 3)).astype(np.float32)
    lo, hi = oracle.scene_box(pts)
    for bits in (1, 7, 10, 21):
        g = fgl.morton_codes(torch.from_numpy(pts).cuda(), lo, hi, bits).cpu().numpy().view(np.uint64)
        assert np.array_equal(g, oracle.morton(pts, lo, hi, bits))


def test_sort_reduce_then_scan_path_matches_oracle():
    """The reduce-then-scan pass variant of the radix sort (off by default; forced here through
    FGL_SORT_RTS_MIN) gives the same stable order as the oracle, key-value and packed key-only
    (the latter through a full LBVH build compared with the default build)."""
    import os
    import subprocess
    import sys
    ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import numpy as np, torch, oracle, synth, paper_2509_17390_b200 as fgl
rng = np.random.default_rng(3)
n = 300_001
keys = rng.integers(0, 2 ** 40, n, dtype=np.int64).astype(np.uint64)
keys[::7] = keys[1::7][: len(keys[::7])]  # duplicates: stability matters
vals = np.arange(n, dtype=np.uint32)
k, v = fgl.sort_pairs(torch.from_numpy(keys.view(np.int64)).cuda(), torch.from_numpy(vals.view(np.int32)).cuda(), 40)
ok_, ov_ = oracle.stable_sort(keys, vals)
assert np.array_equal(k.cpu().numpy().view(np.uint64), ok_) and np.array_equal(v.cpu().numpy().view(np.uint32), ov_)
m = synth.soup(200_003, seed=9)
e = fgl.Scene(m.verts, m.tris).export()
import hashlib
print("OK", hashlib.sha256(e["sorted_keys"].tobytes() + e["nodes"].tobytes() + e["tri48"].tobytes()).hexdigest())
'''
    env = dict(os.environ, FGL_SORT_RTS_MIN="1")
    r1 = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=ROOT, timeout=600)
    assert r1.returncode == 0 and "OK" in r1.stdout, r1.stderr[-2000:]
    r0 = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r0.returncode == 0 and r0.stdout == r1.stdout, (r0.stdout, r1.stdout)
