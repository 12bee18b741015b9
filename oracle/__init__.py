"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain CPU double-precision implementation of the LiDAR first-return cast (§IV-C, Eqs.
19-20) and of the LBVH build steps it depends on (§IV-A, Eqs. 5-7), in
oracle/oracle.c, plus this ctypes/numpy wrapper. Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg may import it. It shares no code with the CUDA
path in paper_2509_17390_b200/ and never imports it.

Pin status: every function below is pinned by tests/test_oracle_*.py against
closed forms, exact-rational brute force, textbook special cases or invariants. None is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_double, c_float, c_int, c_int32, c_int64, c_uint32, c_uint64, c_void_p

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

AMBIG, EDGE, BOUNDARY, GRAZE, OVERFLOW, MISS_OK, INCONSISTENT = 1, 2, 4, 8, 16, 32, 64
EPS_MODE_B = 2.0 ** -20   # oracle consumes the exact float32 rays the kernel used
EPS_MODE_A = 2.0 ** -19   # oracle generates its own rays in double (+ float32 raygen error <= 2^-21)


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, OpenMP, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared", "-ffp-contract=off",
               "-fno-fast-math", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = c_void_p
        sig = {
            "orc_set_threads": (None, [c_int]),
            "orc_get_threads": (c_int, []),
            "orc_spinning_rays": (None, [P, c_int32, c_int32, c_double, P, c_int64, P, P]),
            "orc_rosette_rays": (None, [c_int32, c_uint32, c_uint32, c_uint32, c_double, P, c_int64, c_int64, P, P]),
            "orc_cast": (None, [P, P, c_int64, P, P, c_int64, c_double, c_double, P, P]),
            "orc_classify": (None, [P, P, c_int64, P, P, c_int64, c_double, c_double, c_double, P, P, c_int32,
                                    P, P, P, P, P]),
            "orc_centroids": (None, [P, P, c_int64, P]),
            "orc_scene_box": (None, [P, c_int64, P, P]),
            "orc_morton": (None, [P, c_int64, P, P, c_int, c_int, P]),
            "orc_stable_sort": (None, [P, P, c_int64, P, P]),
            "orc_radix_tree": (c_int, [P, c_int64, P, P]),
            "orc_refit": (None, [P, P, P, c_int64, P, P, P]),
            "orc_nearest": (None, [P, c_int64, P, c_int64, P, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _p(a):
    return a.ctypes.data_as(c_void_p) if a is not None else None


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def threads() -> int:
    return int(lib().orc_get_threads())


# --- ray generation (Eq. 19) -----------------------------------------------------------------
def spinning_rays(elev_deg, columns: int, az0_deg: float, poses):
    e = _c(elev_deg, np.float32)
    P_ = _c(poses, np.float32).reshape(-1, 3, 4)
    n = P_.shape[0] * e.shape[0] * columns
    o = np.empty((n, 3))
    d = np.empty((n, 3))
    lib().orc_spinning_rays(_p(e), e.shape[0], int(columns), float(az0_deg), _p(P_), P_.shape[0], _p(o), _p(d))
    return o, d


def rosette_rays(N: int, inc1: int, inc2: int, phase2_0: int, half_fov_deg: float, poses, first_frame: int = 0):
    P_ = _c(poses, np.float32).reshape(-1, 3, 4)
    n = P_.shape[0] * N
    o = np.empty((n, 3))
    d = np.empty((n, 3))
    lib().orc_rosette_rays(int(N), int(inc1) & 0xFFFFFFFF, int(inc2) & 0xFFFFFFFF, int(phase2_0) & 0xFFFFFFFF,
                           float(half_fov_deg), _p(P_), P_.shape[0], int(first_frame), _p(o), _p(d))
    return o, d


def pattern_rays(pattern, poses, first_frame: int = 0):
    """Rays of a synth.Spinning / synth.Rosette pattern (dispatch on the parameter object)."""
    if hasattr(pattern, "elev_deg"):
        return spinning_rays(pattern.elev_deg, pattern.columns, pattern.az0_deg, poses)
    return rosette_rays(pattern.points_per_frame, pattern.inc1, pattern.inc2, pattern.phase2_0,
                        pattern.half_fov_deg, poses, first_frame)


# --- nearest hit (Eq. 20) --------------------------------------------------------------------
def cast(verts, tris, orig, dir, t_min: float, t_max: float):
    v = _c(verts, np.float32)
    t = _c(tris, np.int32)
    o = _c(orig, np.float64)
    d = _c(dir, np.float64)
    R = o.shape[0]
    tt = np.empty(R)
    ii = np.empty(R, dtype=np.int32)
    lib().orc_cast(_p(v), _p(t), t.shape[0], _p(o), _p(d), R, float(t_min), float(t_max), _p(tt), _p(ii))
    return tt, ii


class Verdict:
    """Classifier output for R rays: flags, kept-candidate lists (id, t_lo, t_hi)."""

    def __init__(self, t1, k1, flags, ncand, cid, clo, chi):
        self.t1, self.k1, self.flags, self.ncand = t1, k1, flags, ncand
        self.cid, self.clo, self.chi = cid, clo, chi

    @property
    def ambiguous(self):
        return (self.flags & AMBIG) != 0


def classify(verts, tris, orig, dir, t_min, t_max, t1, k1, eps_rel=EPS_MODE_B, kmax=16):
    v = _c(verts, np.float32)
    t = _c(tris, np.int32)
    o = _c(orig, np.float64)
    d = _c(dir, np.float64)
    t1 = _c(t1, np.float64)
    k1 = _c(k1, np.int32)
    R = o.shape[0]
    flags = np.empty(R, np.int32)
    nc = np.empty(R, np.int32)
    cid = np.full((R, kmax), -1, np.int32)
    clo = np.full((R, kmax), np.nan)
    chi = np.full((R, kmax), np.nan)
    lib().orc_classify(_p(v), _p(t), t.shape[0], _p(o), _p(d), R, float(t_min), float(t_max), float(eps_rel),
                       _p(t1), _p(k1), int(kmax), _p(flags), _p(nc), _p(cid), _p(clo), _p(chi))
    return Verdict(t1, k1, flags, nc, cid, clo, chi)


def cast_and_classify(verts, tris, orig, dir, t_min, t_max, eps_rel=EPS_MODE_B, kmax=16):
    t1, k1 = cast(verts, tris, orig, dir, t_min, t_max)
    return classify(verts, tris, orig, dir, t_min, t_max, t1, k1, eps_rel, kmax)


def tol(t):
    """North-star range tolerance: 1e-4 * range + 1e-5 m."""
    return 1e-4 * np.abs(t) + 1e-5


def judge(verdict: Verdict, rng, tid):
    """Compare a cast result (range, tri_id) with the oracle verdict ray by ray.
    Returns dict(n, ambiguous, unamb_mismatch, amb_outside, bad_index) (index arrays)."""
    rng = np.asarray(rng, np.float64)
    tid = np.asarray(tid, np.int64)
    v = verdict
    amb = v.ambiguous
    t1 = v.t1
    k1 = v.k1.astype(np.int64)
    # unambiguous rays: exact id, range within tolerance (miss: +inf and -1)
    hit = k1 >= 0
    ok_u = np.where(hit, (tid == k1) & (np.abs(rng - np.where(hit, t1, 0)) <= tol(np.where(hit, t1, 0))),
                    (tid == -1) & np.isinf(rng))
    bad_u = np.nonzero(~amb & ~ok_u)[0]
    # ambiguous rays: a kept candidate within its depth interval (+ tolerance), or a permitted miss
    bad_a = []
    kmax = v.cid.shape[1]
    for r in np.nonzero(amb)[0]:
        if tid[r] < 0:
            if not ((v.flags[r] & MISS_OK) and np.isinf(rng[r])):
                bad_a.append(r)
            continue
        if v.flags[r] & OVERFLOW:
            ok = True  # candidate list truncated; accept a member or anything beyond the listed ones
            m = np.nonzero(v.cid[r] == tid[r])[0]
            if m.size:
                i = m[0]
                ok = v.clo[r, i] - tol(v.clo[r, i]) <= rng[r] <= v.chi[r, i] + tol(v.chi[r, i])
        else:
            m = np.nonzero(v.cid[r, :min(v.ncand[r], kmax)] == tid[r])[0]
            ok = bool(m.size) and (v.clo[r, m[0]] - tol(v.clo[r, m[0]]) <= rng[r] <= v.chi[r, m[0]] + tol(v.chi[r, m[0]]))
        if not ok:
            bad_a.append(r)
    return dict(n=int(rng.shape[0]), ambiguous=int(amb.sum()), unamb_mismatch=bad_u,
                amb_outside=np.array(bad_a, dtype=np.int64))


# --- LBVH build (Eqs. 5-7) -------------------------------------------------------------------
def centroids(verts, tris):
    v = _c(verts, np.float32)
    t = _c(tris, np.int32)
    c = np.empty((t.shape[0], 3), np.float32)
    lib().orc_centroids(_p(v), _p(t), t.shape[0], _p(c))
    return c


def scene_box(cent):
    c = _c(cent, np.float32)
    lo = np.empty(3, np.float32)
    hi = np.empty(3, np.float32)
    lib().orc_scene_box(_p(c), c.shape[0], _p(lo), _p(hi))
    return lo, hi


def morton(cent, lo, hi, bits: int = 21, cubic: bool = False):
    c = _c(cent, np.float32)
    code = np.empty(c.shape[0], np.uint64)
    lib().orc_morton(_p(c), c.shape[0], _p(_c(lo, np.float32)), _p(_c(hi, np.float32)), int(bits), int(cubic),
                     _p(code))
    return code


def stable_sort(keys, vals=None):
    k = _c(keys, np.uint64)
    v = None if vals is None else _c(vals, np.uint32)
    sk = np.empty_like(k)
    sv = np.empty(k.shape[0], np.uint32)
    lib().orc_stable_sort(_p(k), _p(v), k.shape[0], _p(sk), _p(sv))
    return sk, sv


def radix_tree(sorted_keys):
    k = _c(sorted_keys, np.uint64)
    n = k.shape[0]
    child = np.zeros((max(n - 1, 0), 2), np.int32)
    rng = np.zeros((max(n - 1, 0), 2), np.int32)
    rc = lib().orc_radix_tree(_p(k), n, _p(child), _p(rng))
    if rc:
        raise RuntimeError("radix tree: wrong internal node count")
    return child, rng


def refit(verts, tris, perm, child):
    v = _c(verts, np.float32)
    t = _c(tris, np.int32)
    p = _c(perm, np.uint32)
    c = _c(child, np.int32)
    n = p.shape[0]
    leaf = np.empty((n, 6), np.float32)
    node = np.empty((max(n - 1, 0), 6), np.float32)
    lib().orc_refit(_p(v), _p(t), _p(p), n, _p(c), _p(leaf), _p(node))
    return leaf, node


def lbvh(verts, tris, bits: int = 21, cubic: bool = False):
    """All LBVH steps in paper order: centroids -> box -> Eq. 5 -> sort -> Eq. 6 tree -> Eq. 7."""
    cent = centroids(verts, tris)
    lo, hi = scene_box(cent)
    code = morton(cent, lo, hi, bits, cubic)
    sk, perm = stable_sort(code)
    child, rng = radix_tree(sk) if len(sk) >= 2 else (np.zeros((0, 2), np.int32), np.zeros((0, 2), np.int32))
    leaf, node = refit(verts, tris, perm, child)
    return dict(cent=cent, lo=lo, hi=hi, code=code, sorted_keys=sk, perm=perm, child=child, range=rng,
                leaf_box=leaf, node_box=node)


# --- point-cloud metrics (§V-A; reading R23) ------------------------------------------
def nearest(points, queries):
    """Exact nearest neighbour of every query in `points` (double distances, ties -> smaller index)."""
    p = _c(points, np.float32).reshape(-1, 3)
    q = _c(queries, np.float32).reshape(-1, 3)
    d = np.empty(q.shape[0])
    i = np.empty(q.shape[0], np.int32)
    lib().orc_nearest(_p(p), p.shape[0], _p(q), q.shape[0], _p(d), _p(i))
    return d, i


def cloud_metrics(a, b, tau):
    """Symmetric Chamfer distance (unsquared distances, mean of the two directed means), precision
    (fraction of a within tau of b), recall (fraction of b within tau of a) and F-score (harmonic
    mean; 0 when P + R = 0). "Within" is d <= tau (R23)."""
    dab, _ = nearest(b, a)
    dba, _ = nearest(a, b)
    cd = 0.5 * (dab.mean() + dba.mean())
    prec = float(np.mean(dab <= tau))
    rec = float(np.mean(dba <= tau))
    f = 2 * prec * rec / (prec + rec) if prec + rec > 0 else 0.0
    return dict(chamfer=float(cd), precision=prec, recall=rec, fscore=f, d_ab=dab, d_ba=dba)
