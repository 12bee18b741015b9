"""Pins for the oracle's LBVH steps (§IV-A, Eqs. 5-7): Morton codes against exact
integer cases and a bit-string decode, the stable order by its defining properties, the radix
tree against the textbook worked example (Karras 2012, Fig. 3) and the defining prefix
properties on random keys, the refit against brute-force subtree unions."""
import numpy as np
import pytest

import synth


def test_centroid_exact_on_integer_triangles(orc):
    V = np.array([[0, 0, 0], [3, 6, 9], [6, 0, 3], [-3, 3, 0]], np.float32)
    Tr = np.array([[0, 1, 2], [1, 2, 3]], np.int32)
    c = orc.centroids(V, Tr)
    assert np.array_equal(c, [[3, 2, 4], [2, 3, 4]])


def test_scene_box_is_exact_bounds(orc):
    rng = np.random.default_rng(0)
    c = rng.normal(size=(1000, 3)).astype(np.float32)
    lo, hi = orc.scene_box(c)
    assert np.array_equal(lo, c.min(0)) and np.array_equal(hi, c.max(0))


def _decode(code, bits):
    s = bin(int(code))[2:].zfill(3 * bits)[::-1]  # s[i] = bit i
    return [int(s[a::3][::-1], 2) for a in range(3)]


def test_morton_closed_forms(orc):
    lo = np.zeros(3, np.float32)
    for bits in (1, 5, 10, 21):
        hi = np.full(3, 2.0 ** bits, np.float32)  # L = 2^b: scale 1, q = floor(c)
        assert orc.morton(np.zeros((1, 3), np.float32), lo, hi, bits)[0] == 0         # origin -> 0 [S:123]
        top = orc.morton(hi[None], lo, hi, bits)[0]                                  # clamp at 2^b - 1
        assert top == 2 ** (3 * bits) - 1
    hi1 = np.ones(3, np.float32)
    assert orc.morton(np.array([[0.75, 0.5, 0.9]], np.float32), lo, hi1, 1)[0] == 7  # upper half -> 7 [S:124]
    hi = np.full(3, 2.0 ** 21, np.float32)
    axes = orc.morton(np.array([[1.5, 0, 0], [0, 1.5, 0], [0, 0, 1.5]], np.float32), lo, hi, 21)
    assert list(axes) == [1, 2, 4]  # x lowest


def test_morton_decode_matches_integer_cells(orc):
    rng = np.random.default_rng(1)
    for bits in (3, 10, 21):
        q = rng.integers(0, 2 ** bits, size=(500, 3))
        frac = rng.uniform(0, 0.99, size=(500, 3))
        c = (q + frac).astype(np.float32)
        q = np.floor(c).astype(np.int64)  # float32 rounding may carry into the next cell
        lo = np.zeros(3, np.float32)
        hi = np.full(3, 2.0 ** bits, np.float32)
        code = orc.morton(c, lo, hi, bits)
        for i in range(500):
            assert _decode(code[i], bits) == [min(int(x), 2 ** bits - 1) for x in q[i]]


def test_morton_flat_axis(orc):
    c = np.array([[0, 1, 5], [4, 3, 5]], np.float32)
    lo, hi = orc.scene_box(c)
    code = orc.morton(c, lo, hi, 2)
    assert [(_decode(x, 2)[2]) for x in code] == [0, 0]


def test_stable_sort_properties(orc):
    rng = np.random.default_rng(2)
    for n in (0, 1, 2, 17, 5000):
        keys = rng.integers(0, 40, size=n).astype(np.uint64) << np.uint64(rng.integers(0, 50))
        sk, perm = orc.stable_sort(keys)
        assert sorted(perm.tolist()) == list(range(n))                  # a permutation
        assert np.array_equal(keys[perm], sk)
        assert np.all(sk[1:] >= sk[:-1])                                  # ordered
        eq = sk[1:] == sk[:-1]
        assert np.all(perm[1:][eq] > perm[:-1][eq])                        # stable


def test_radix_tree_karras_worked_example(orc):
    # Karras 2012, Fig. 3: keys 00001 00010 00100 00101 10011 11000 11001 11110.
    # Hand derivation: root [0,7] splits after 3 (first bit); node 3 = [0,3] splits after 1;
    # node 1 = [0,1] -> leaves 0,1; node 2 = [2,3] -> leaves 2,3; node 4 = [4,7] splits after 4
    # -> leaf 4, node 5 = [5,7] splits after 6 -> node 6 = [5,6] (leaves 5,6), leaf 7.
    keys = np.array([1, 2, 4, 5, 19, 24, 25, 30], np.uint64)
    child, rng = orc.radix_tree(keys)
    L = lambda j: ~j
    assert child.tolist() == [[3, 4], [L(0), L(1)], [L(2), L(3)], [1, 2], [L(4), 5], [6, L(7)], [L(5), L(6)]]
    assert rng.tolist() == [[0, 7], [0, 1], [2, 3], [0, 3], [4, 7], [5, 7], [5, 6]]


def _aug(k, i):
    return (int(k) << 32) | i


def _check_tree(keys, child, rng):
    n = len(keys)
    seen_int, seen_leaf = [0] * (n - 1), [0] * n
    for i in range(n - 1):
        f, l = rng[i]
        assert i in (f, l)                                  # node index is an end of its range
        a, b = _aug(keys[f], f), _aug(keys[l], l)
        lam = 96 - (a ^ b).bit_length()                      # common prefix length of the range
        bit = 95 - lam                                       # first differing bit
        for s, c in enumerate(child[i]):
            if c < 0:
                cf = cl = ~c
                seen_leaf[~c] += 1
            else:
                cf, cl = rng[c]
                seen_int[c] += 1
            for j in range(cf, cl + 1):
                x = _aug(keys[j], j)
                assert (x >> (bit + 1)) == (a >> (bit + 1))  # shares the range prefix
                assert ((x >> bit) & 1) == s                 # left = 0, right = 1 at the split bit
        lo_c = child[i][0]
        hi_c = child[i][1]
        lend = ~lo_c if lo_c < 0 else rng[lo_c][1]
        rbeg = ~hi_c if hi_c < 0 else rng[hi_c][0]
        assert (f, l) == ((~lo_c if lo_c < 0 else rng[lo_c][0]), (~hi_c if hi_c < 0 else rng[hi_c][1]))
        assert rbeg == lend + 1
    assert seen_int[0] == 0 and all(x == 1 for x in seen_int[1:])
    assert all(x == 1 for x in seen_leaf)


def test_radix_tree_prefix_properties(orc):
    rng = np.random.default_rng(3)
    for n in (2, 3, 5, 64, 300):
        for dup in (False, True):
            hi = 8 if dup else 2 ** 63
            keys = np.sort(rng.integers(0, hi, size=n, dtype=np.uint64))
            child, rr = orc.radix_tree(keys)
            _check_tree(keys.tolist(), child.tolist(), rr.tolist())
    keys = np.zeros(9, np.uint64)  # all equal: index fallback builds a balanced-by-bits tree
    child, rr = orc.radix_tree(keys)
    _check_tree(keys.tolist(), child.tolist(), rr.tolist())


def test_refit_is_exact_union(orc):
    m = synth.soup(700, seed=5)
    b = orc.lbvh(m.verts, m.tris)
    V = m.verts[m.tris[b["perm"]]]  # [n][3][3] in sorted order
    lo_t, hi_t = V.min(1), V.max(1)
    assert np.array_equal(b["leaf_box"][:, :3], lo_t) and np.array_equal(b["leaf_box"][:, 3:], hi_t)
    for i, (f, l) in enumerate(b["range"]):
        assert np.array_equal(b["node_box"][i, :3], lo_t[f:l + 1].min(0))
        assert np.array_equal(b["node_box"][i, 3:], hi_t[f:l + 1].max(0))
    # root covers everything
    assert np.array_equal(b["node_box"][0, :3], m.verts[m.tris].reshape(-1, 3).min(0))


def test_single_triangle_tree(orc):
    V = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 2]], np.float32)
    b = orc.lbvh(V, np.array([[0, 1, 2]], np.int32))
    assert b["child"].shape == (0, 2) and np.array_equal(b["leaf_box"][0], [0, 0, 0, 1, 1, 2])


def test_morton_cubic_box_uses_longest_extent(orc):
    # R22: with a cubic box every axis is scaled by the longest extent: for lo = 0 and a longest
    # extent of 2^b the cells are unit cubes on all axes, q = floor(c), whatever the other extents
    bits = 10
    lo = np.zeros(3, np.float32)
    hi = np.array([2.0 ** bits, 5.0, 3.0], np.float32)
    rng = np.random.default_rng(7)
    c = np.stack([rng.uniform(0, 2 ** bits, 300), rng.uniform(0, 5, 300), rng.uniform(0, 3, 300)], 1).astype(np.float32)
    code = orc.morton(c, lo, hi, bits, cubic=True)
    for i in range(300):
        assert _decode(code[i], bits) == [min(int(np.floor(x)), 2 ** bits - 1) for x in c[i]]
    # per-axis (Eq. 5) scales y by 2^b / 5 instead
    code2 = orc.morton(c, lo, hi, bits)
    assert _decode(code2[0], bits)[1] == int(np.floor(np.float32(c[0, 1]) * np.float32(2.0 ** bits / 5.0)))
