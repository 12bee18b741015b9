"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py for the rules).

Plain numpy statement of the mesh-reconstruction steps of PAPER.md §IV-B:
binary denoising (Eq. 13) and fixed / quantile re-thresholding (Eq. 14), the
narrow-band TSDF — outside flood fill from the padded frame, boundary set S_0 (Eq. 15,
P:206-208), layered shells kappa(x) and delta = kappa v_min (Eq. 16), phi =
clip(s delta, -r, r) (Eq. 17) — and Marching Cubes on phi (Eq. 18).

Readings (R29-R34): the Gaussian kernel is truncated at ceil(3 sigma) voxels and
normalised, outside the grid counts as empty (R29); outside = the free voxels 6-connected to
the padded frame, i.e. to the grid boundary (R30); S_0 includes both sides of every V-change,
the frame counting as free (R31); beyond the band phi = s r (R32); phi is formed in float32
(R33: sign and cube decisions are float decisions, taken in the kernel's precision); the cube
polygonisation is face-consistent Marching Cubes — on every cube face the inside corners are
cut off one run at a time (diagonal faces keep their two inside corners apart), segments chain
into loops, each loop is fanned from its lowest edge unless a fan diagonal would lie in a cube
face (then it is fanned around its centroid), edge vertices are numbered by global edge id (R34).

Pin status: pinned in tests/test_oracle_tsdf.py against scipy.ndimage (gaussian_filter1d,
label, distance_transform_cdt), closed forms (solid and hollow boxes, spheres) and mesh
invariants (watertight 2-manifold, outward orientation, enclosed volume, Euler characteristic).
None is "parity unpinned".
"""
from __future__ import annotations

import math

import numpy as np


# ---- Eqs. 13-14: denoise + re-threshold ----------------------------------------------------
def gauss_weights(sigma_vox: float):
    """Normalised 1-D Gaussian weights on [-R, R], R = max(1, ceil(3 sigma)) (R29)."""
    R = max(1, int(math.ceil(3.0 * sigma_vox)))
    k = np.arange(-R, R + 1, dtype=np.float64)
    w = np.exp(-0.5 * (k / sigma_vox) ** 2)
    return w / w.sum()


def blur(V, sigma_m: float, spacing):
    """Eq. 13: V' = G_sigma * V, separable along x, y, z with sigma_a = sigma / s_a voxels and zero
    outside the grid (R29). V: [nz][ny][nx] (bool or float). Returns float64."""
    out = np.asarray(V, np.float64)
    for ax_arr, s in ((2, spacing[0]), (1, spacing[1]), (0, spacing[2])):
        w = gauss_weights(sigma_m / s)
        R = (len(w) - 1) // 2
        pad = [(0, 0)] * 3
        pad[ax_arr] = (R, R)
        P = np.pad(out, pad)
        acc = np.zeros_like(out)
        n = out.shape[ax_arr]
        for t in range(2 * R + 1):
            sl = [slice(None)] * 3
            sl[ax_arr] = slice(t, t + n)
            acc += w[t] * P[tuple(sl)]
        out = acc
    return out


def rethreshold(Vp, tau: float):
    """Eq. 14a: V~ = V' >= tau."""
    return np.asarray(Vp) >= tau


def quantile(Vp, q: float):
    """Quantile_q(V') of Eq. 14b read as the inverted-CDF quantile (R35): the value of 1-based rank
    max(1, ceil(q N)) in ascending order."""
    v = np.sort(np.asarray(Vp).reshape(-1))
    k = min(max(1, int(math.ceil(q * v.size))), v.size)
    return v[k - 1]


def rethreshold_quantile(Vp, q: float):
    """Eq. 14b: V~ = V' >= Quantile_q(V')."""
    return np.asarray(Vp) >= quantile(Vp, q)


# ---- Eqs. 15-17: narrow-band TSDF ------------------------------------------------------------
def _nbr_or(M):
    """For every voxel, OR of its six face neighbours (outside the grid = False)."""
    P = np.pad(M, 1)
    c = slice(1, -1)
    out = np.zeros_like(M)
    for ax in range(3):
        for d in (-1, 1):
            sl = [c, c, c]
            sl[ax] = slice(1 + d, P.shape[ax] - 1 + d)
            out |= P[tuple(sl)]
    return out


def outside(V):
    """Free voxels 6-connected to the padded frame Gamma (R30): the fixed point of 'free and
    (on the grid boundary or next to an outside voxel)' by iterated dilation."""
    free = ~np.asarray(V, bool)
    border = np.zeros_like(free)
    border[0, :, :] = border[-1, :, :] = True
    border[:, 0, :] = border[:, -1, :] = True
    border[:, :, 0] = border[:, :, -1] = True
    O = free & border
    while True:
        nxt = O | (free & _nbr_or(O))
        if np.array_equal(nxt, O):
            return O
        O = nxt


def boundary_set(V):
    """Eq. 15: S_0 = {x : some 6-neighbour y has V(y) != V(x)}, the frame counting as free (R31)."""
    V = np.asarray(V, bool)
    P = np.pad(V, 1)  # frame = free
    c = slice(1, -1)
    S = np.zeros_like(V)
    for ax in range(3):
        for d in (-1, 1):
            sl = [c, c, c]
            sl[ax] = slice(1 + d, P.shape[ax] - 1 + d)
            S |= P[tuple(sl)] != V
    return S


def shells(V, m_max: int):
    """Layered propagation from S_0: kappa = 0 on S_0, kappa = m on the voxels first
    reached by the m-th 6-neighbour expansion; -1 where not reached within m_max shells."""
    S = boundary_set(V)
    kappa = np.where(S, 0, -1).astype(np.int64)
    vis = S.copy()
    for m in range(1, m_max + 1):
        new = _nbr_or(vis) & ~vis
        if not new.any():
            break
        kappa[new] = m
        vis |= new
    return kappa


def tsdf(V, spacing, r: float):
    """Eqs. 16-17: phi = clip(s(x) kappa(x) v_min, -r, r), s = +1 outside (R30) else -1; the
    product and the clip in float32 (R33); voxels beyond the band get s r (R32)."""
    V = np.asarray(V, bool)
    vmin = np.float32(min(spacing))
    r32 = np.float32(r)
    m_max = int(math.ceil(float(r32) / float(vmin))) if vmin > 0 else 0
    kappa = shells(V, m_max)
    s = np.where(outside(V), np.float32(1), np.float32(-1))
    d = np.where(kappa >= 0, kappa.astype(np.float32) * vmin, r32).astype(np.float32)
    d = np.minimum(d, r32)
    return (s * d).astype(np.float32), kappa


# ---- Eq. 18: Marching Cubes ------------------------------------------------------------------
# corner c = dx + 2 dy + 4 dz of the cube whose lowest corner is voxel (i, j, k)
_CORNER = [(c & 1, (c >> 1) & 1, (c >> 2) & 1) for c in range(8)]


def _faces():
    """The six faces as corner lists ordered counter-clockwise seen from outside the cube."""
    faces = []
    for ax in range(3):
        for side in (0, 1):
            cs = [c for c in range(8) if _CORNER[c][ax] == side]
            n = np.zeros(3)
            n[ax] = 1.0 if side else -1.0
            ctr = np.mean([_CORNER[c] for c in cs], axis=0)
            u = np.zeros(3)
            u[(ax + 1) % 3] = 1.0
            v = np.cross(n, u)
            ang = [math.atan2(np.dot(np.subtract(_CORNER[c], ctr), v), np.dot(np.subtract(_CORNER[c], ctr), u))
                   for c in cs]
            faces.append([cs[i] for i in np.argsort(ang)])  # increasing angle about n = CCW from outside
    return faces


_FACES = _faces()


def _edge(a, b):
    """Local edge between adjacent corners a, b: (lower corner, axis)."""
    lo = min(a, b, key=lambda c: sum(_CORNER[c]))
    ax = [t for t in range(3) if _CORNER[a][t] != _CORNER[b][t]][0]
    return lo, ax


def _edge_rank(e):
    """Global edge ids of one cube's edges are ordered by (dz, dy, dx, axis) of (lower corner, axis)."""
    c, ax = e
    dx, dy, dz = _CORNER[c]
    return (dz, dy, dx, ax)


def cube_polygons(inside):
    """Loops of local edges for one cube (inside[c] for the 8 corners): on each face the inside
    corners are cut off run by run (two diagonal inside corners stay apart), each segment goes
    from the edge entering the run to the edge leaving it (CCW seen from outside), segments chain
    into loops, each loop starts at its lowest-ranked edge (R34)."""
    nxt = {}
    for f in _FACES:
        b = [bool(inside[c]) for c in f]
        if all(b) or not any(b):
            continue
        for s in range(4):  # a run starts at s: b[s] and not b[s-1]
            if b[s] and not b[s - 1]:
                t = s
                while b[(t + 1) % 4]:
                    t = (t + 1) % 4
                e_in = _edge(f[s - 1], f[s])
                e_out = _edge(f[t], f[(t + 1) % 4])
                assert e_in not in nxt
                nxt[e_in] = e_out
    loops = []
    left = set(nxt)
    while left:
        start = min(left, key=_edge_rank)
        loop = [start]
        left.discard(start)
        e = nxt[start]
        while e != start:
            loop.append(e)
            left.discard(e)
            e = nxt[e]
        loops.append(loop)
    return loops


def _same_face(e1, e2):
    """Do two local edges lie on a common cube face?"""
    pts = {e1[0], e2[0], _edge_end(e1), _edge_end(e2)}
    return any(pts <= set(f) for f in _FACES)


def _edge_end(e):
    c, ax = e
    return c | (1 << ax)


def fan_ok(loop):
    """A loop is fanned from its first edge unless a fan diagonal (v0, v_k), 2 <= k <= m-2, joins
    two vertices on one cube face (possible only through an ambiguous face): such a diagonal would
    lie in the face and be shared with the neighbouring cube's fan (R34)."""
    return all(not _same_face(loop[0], loop[k]) for k in range(2, len(loop) - 1))


def marching_cubes(phi, origin, spacing, iso: float = 0.0, normals: bool = False):
    """Eq. 18 on the voxel-centre lattice of phi [nz][ny][nx]: corner c is inside iff
    phi < iso (float32 comparison, R33); one vertex per crossing edge at p_a + t (p_b - p_a),
    t = (iso - phi_a) / (phi_b - phi_a) (double), numbered by increasing global edge id
    3 (k ny nx + j nx + i) + axis; each loop becomes the fan (v0, v_k, v_k+1) from its first
    vertex, or, when fan_ok fails, the fan (c, v_k, v_k+1) (k cyclic) around an extra vertex c = the
    mean of its vertices, numbered after all edge vertices in emission order; cubes in (k, j, i)
    order, loops in order of their first edge (R34). Returns (verts float64 [V][3], tris int64
    [T][3] [, normals]): normals = normalised interpolation of the central-difference gradient of
    phi (one-sided on the grid boundary); a centre vertex takes the normalised mean of its loop's."""
    phi = np.asarray(phi, np.float32)
    nz, ny, nx = phi.shape
    iso32 = np.float32(iso)
    ins = phi < iso32
    o = np.asarray(origin, np.float64)
    sp = np.asarray(spacing, np.float64)
    # crossing edges and their vertex ids (global edge id order)
    eid_list = []
    for ax in range(3):
        sl_a = [slice(None)] * 3
        sl_b = [slice(None)] * 3
        arr_ax = 2 - ax
        sl_a[arr_ax] = slice(0, phi.shape[arr_ax] - 1)
        sl_b[arr_ax] = slice(1, phi.shape[arr_ax])
        cross = ins[tuple(sl_a)] != ins[tuple(sl_b)]
        k, j, i = np.nonzero(cross)
        eid_list.append(3 * ((k * ny + j) * nx + i) + ax)
    eids = np.sort(np.concatenate(eid_list))
    vid = {int(e): n for n, e in enumerate(eids)}
    verts = np.empty((len(eids), 3))
    grad = None
    if normals:
        grad = np.stack([np.gradient(phi.astype(np.float64), sp[a], axis=2 - a) if phi.shape[2 - a] > 1
                         else np.zeros(phi.shape) for a in range(3)], axis=-1)
    nrm = np.zeros((len(eids), 3))
    for n, e in enumerate(eids):
        ax = int(e % 3)
        lin = int(e // 3)
        k, rem = divmod(lin, nx * ny)
        j, i = divmod(rem, nx)
        a = np.array([i, j, k])
        b = a.copy()
        b[ax] += 1
        pa, pb = float(phi[a[2], a[1], a[0]]), float(phi[b[2], b[1], b[0]])
        t = (float(iso32) - pa) / (pb - pa)
        xa = o + (a + 0.5) * sp
        xb = o + (b + 0.5) * sp
        verts[n] = xa + t * (xb - xa)
        if normals:
            g = (1 - t) * grad[a[2], a[1], a[0]] + t * grad[b[2], b[1], b[0]]
            ln = np.linalg.norm(g)
            nrm[n] = g / ln if ln > 0 else 0.0
    tris = []
    extra, extra_n = [], []
    cache = {}
    for k in range(nz - 1):
        for j in range(ny - 1):
            for i in range(nx - 1):
                idx = 0
                for c in range(8):
                    dx, dy, dz = _CORNER[c]
                    if ins[k + dz, j + dy, i + dx]:
                        idx |= 1 << c
                if idx == 0 or idx == 255:
                    continue
                if idx not in cache:
                    cache[idx] = [(lp, fan_ok(lp)) for lp in cube_polygons([(idx >> c) & 1 for c in range(8)])]
                for loop, ok in cache[idx]:
                    g = []
                    for (c, ax) in loop:
                        dx, dy, dz = _CORNER[c]
                        g.append(vid[3 * (((k + dz) * ny + (j + dy)) * nx + (i + dx)) + ax])
                    if ok:
                        for m in range(1, len(g) - 1):
                            tris.append((g[0], g[m], g[m + 1]))
                    else:
                        cid = len(eids) + len(extra)
                        extra.append(verts[g].mean(axis=0))
                        mn = nrm[g].mean(axis=0)
                        ln = np.linalg.norm(mn)
                        extra_n.append(mn / ln if ln > 0 else mn)
                        for m in range(len(g)):
                            tris.append((cid, g[m], g[(m + 1) % len(g)]))
    tris = np.asarray(tris, np.int64).reshape(-1, 3)
    if extra:
        verts = np.concatenate([verts, np.asarray(extra)])
        nrm = np.concatenate([nrm, np.asarray(extra_n)])
    if not normals:
        return verts, tris
    return verts, tris, nrm
