"""Thin ctypes binding of libfgl.so (include/fgl.h) — argument marshalling only.

Every step of the cast path runs in the library's sm_100a kernels; this module only passes
torch device pointers, sizes and the current CUDA stream through the C ABI. There is no CPU
fallback: if libfgl.so is missing or no CUDA device is present the calls raise.

PAPER.md anchors: mesh M, pose T_s, pattern d_j (Eq. 19),
nearest hit t_j* / rho_j (Eq. 20), LBVH build (§IV-A).
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, Structure, c_char_p, c_float, c_int, c_int32, c_int64, c_uint32, c_uint64, c_void_p

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FGL_LIB") or os.path.join(HERE, "libfgl.so")  # FGL_LIB: A/B builds

OK, E_USAGE, E_DATA, E_RESOURCE, E_CUDA = range(5)
HOST, DEVICE, ASYNC = 0, 1, 4


class FglError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"fgl status {status}: {msg}")
        self.status = status


class BuildOpts(Structure):
    _fields_ = [("morton_bits", c_int32), ("leaf_size", c_int32), ("morton_box", c_int32), ("width", c_int32),
                ("quantized", c_int32), ("restructure", c_int32), ("treelets", c_int32), ("reserved", c_int32 * 1)]


class Stats(Structure):
    _fields_ = [("triangles", c_int64), ("vertices", c_int64), ("nodes", c_int64), ("device_bytes", c_int64),
                ("scene_lo", c_float * 3), ("scene_hi", c_float * 3), ("build_ms", c_float),
                ("morton_bits", c_int32), ("leaf_size", c_int32)]


class SpinningC(Structure):
    _fields_ = [("channels", c_int32), ("columns", c_int32), ("elev_deg", c_void_p), ("az0_deg", c_float),
                ("t_min", c_float), ("t_max", c_float)]


class RosetteC(Structure):
    _fields_ = [("points_per_frame", c_int32), ("inc1", c_uint32), ("inc2", c_uint32), ("phase2_0", c_uint32),
                ("half_fov_deg", c_float), ("t_min", c_float), ("t_max", c_float)]


class GridC(Structure):
    _fields_ = [("origin", c_float * 3), ("spacing", c_float), ("dims", c_int32 * 3), ("tile", c_int32),
                ("theta", c_float), ("reserved", c_int32 * 3)]


class ExportC(Structure):
    _fields_ = [(n, c_void_p) for n in ("scene_box", "codes", "sorted_keys", "perm", "child", "range", "leaf_box",
                                        "node_box", "tri48", "nodes", "nodes4", "depth")]


# name: (restype, argtypes)
_SIGS = {
    "fgl_scene_create": (c_int, [c_int, POINTER(c_void_p)]),
    "fgl_scene_destroy": (None, [c_void_p]),
    "fgl_scene_upload_mesh": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_int, c_void_p]),
    "fgl_scene_build": (c_int, [c_void_p, c_void_p, c_void_p]),
    "fgl_scene_stats": (c_int, [c_void_p, POINTER(Stats)]),
    "fgl_scene_refit": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_void_p]),
    "fgl_scene_check": (c_int, [c_void_p, c_void_p]),
    "fgl_cast_spinning": (c_int, [c_void_p, POINTER(SpinningC), c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_void_p, c_void_p]),
    "fgl_cast_rosette": (c_int, [c_void_p, POINTER(RosetteC), c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                 c_void_p, c_void_p, c_void_p]),
    "fgl_cast_rays": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_float, c_float, c_void_p, c_void_p, c_void_p]),
    "fgl_cast_rays_bruteforce": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_float, c_float, c_void_p, c_void_p,
                                         c_void_p]),
    "fgl_export_rays_spinning": (c_int, [POINTER(SpinningC), c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "fgl_export_rays_rosette": (c_int, [POINTER(RosetteC), c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p]),
    "fgl_scene_export": (c_int, [c_void_p, POINTER(ExportC), c_void_p]),
    "fgl_morton_codes": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_int32, c_void_p, c_void_p]),
    "fgl_sort_pairs": (c_int, [c_void_p, c_void_p, c_int64, c_int32, c_void_p]),
    "fgl_cast_spinning_gather": (c_int, [c_void_p, POINTER(SpinningC), c_void_p, c_int64, c_int64, c_void_p, c_void_p,
                                         c_int32, c_void_p]),
    "fgl_cast_spinning_gather_signal": (c_int, [c_void_p, POINTER(SpinningC), c_void_p, c_int64, c_int64, c_void_p,
                                                c_void_p, c_void_p, c_int32, c_void_p]),
    "fgl_wait_flag": (c_int, [c_void_p, c_int32, c_void_p]),
    "fgl_l2_read_probe": (c_int, [c_void_p, c_int64, c_int32, c_void_p, c_void_p]),
    "fgl_scene_upload_points": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_void_p]),
    "fgl_nearest": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "fgl_cloud_metrics": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_float, c_void_p, c_void_p]),
    "fgl_scene_upload_gaussians": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_float, c_int,
                                           c_void_p]),
    "fgl_voxelize": (c_int, [c_void_p, POINTER(GridC), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "fgl_denoise": (c_int, [c_void_p, c_void_p, c_void_p, c_float, c_float, c_void_p, c_void_p, c_void_p]),
    "fgl_denoise_quantile": (c_int, [c_void_p, c_void_p, c_void_p, c_float, c_float, c_void_p, c_void_p, c_void_p,
                                     c_void_p]),
    "fgl_tsdf": (c_int, [c_void_p, c_void_p, c_void_p, c_float, c_void_p, c_void_p]),
    "fgl_marching_cubes": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_float, c_void_p, c_void_p, c_int64,
                                   c_void_p, c_int64, c_void_p, c_void_p]),
    "fgl_alloc": (c_int, [c_int, c_int64, POINTER(c_void_p)]),
    "fgl_free": (c_int, [c_void_p]),
    "fgl_ipc_get_handle": (c_int, [c_void_p, c_void_p]),
    "fgl_ipc_open_handle": (c_int, [c_int, c_void_p, POINTER(c_void_p)]),
    "fgl_ipc_close_handle": (c_int, [c_void_p]),
    "fgl_last_error": (c_char_p, []),
    "fgl_version": (c_char_p, []),
    "fgl_abi_version": (c_int32, []),
    "fgl_kernel_launches": (c_int64, []),
}
SYMBOLS = tuple(_SIGS)

_lib = None


def lib():
    """Load libfgl.so (in-tree). Raises loudly if it is missing: there is no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libfgl.so not found at {LIB_PATH}; run __graft_entry__.build() "
                              "(python paper_2509_17390_b200/_build.py)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int):
    if status != OK:
        raise FglError(status, lib().fgl_last_error().decode(errors="replace"))


def _stream(stream=None) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


def _ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())


def _dev(t: torch.Tensor, dtype, device, shape=None) -> torch.Tensor:
    t = torch.as_tensor(t).to(device=device, dtype=dtype).contiguous()
    if shape is not None:
        t = t.reshape(shape)
    return t


def spinning_struct(pattern):
    """fgl_spinning from any object with elev_deg, columns, az0_deg, t_min, t_max."""
    e = np.ascontiguousarray(np.asarray(pattern.elev_deg, dtype=np.float32))
    s = SpinningC(int(e.shape[0]), int(pattern.columns), e.ctypes.data, float(getattr(pattern, "az0_deg", 0.0)),
                  float(pattern.t_min), float(pattern.t_max))
    s._keep = e
    return s


def rosette_struct(pattern):
    return RosetteC(int(pattern.points_per_frame), int(pattern.inc1) & 0xFFFFFFFF, int(pattern.inc2) & 0xFFFFFFFF,
                    int(pattern.phase2_0) & 0xFFFFFFFF, float(pattern.half_fov_deg), float(pattern.t_min),
                    float(pattern.t_max))


def is_spinning(pattern) -> bool:
    return hasattr(pattern, "elev_deg")


def rays_per_pose(pattern) -> int:
    if is_spinning(pattern):
        return int(len(pattern.elev_deg)) * int(pattern.columns)
    return int(pattern.points_per_frame)


class Scene:
    """A triangle mesh on one GPU with its LBVH. `Scene(verts, tris)` uploads (validating) and
    builds; `cast(poses, pattern)` returns (range, tri_id) device tensors."""

    def __init__(self, verts=None, tris=None, device=None, build: bool = True, morton_bits: int = 0,
                 leaf_size: int = 0, morton_box: int = 0, width: int = 0, quantized: int = 0, restructure: int = 0,
                 treelets: int = 0, stream=None):
        """leaf_size / width 0 = library defaults; morton_box 0 = cubic (R22), 1 = per-axis (Eq. 5)."""
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        h = c_void_p()
        _check(lib().fgl_scene_create(self.device.index or 0, ctypes.byref(h)))
        self._h = h
        self.morton_bits, self.leaf_size, self.morton_box, self.width = morton_bits, leaf_size, morton_box, width
        self.quantized = quantized
        self.restructure = restructure
        self.treelets = treelets
        self.T = 0
        if verts is not None:
            self.upload(verts, tris, stream)
            if build:
                self.build(stream=stream)

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            try:
                _lib.fgl_scene_destroy(h)
            except Exception:
                pass
        self._h = None

    __del__ = close

    # ---- upload / build -------------------------------------------------------------------
    def upload(self, verts, tris, stream=None, sync: bool = True):
        """Copy + validate the mesh. sync=False: no host synchronisation (CUDA-graph capturable);
        call check() to surface a validation error."""
        on_dev = isinstance(verts, torch.Tensor) and verts.is_cuda
        if on_dev:
            v = verts.to(torch.float32).contiguous()
            t = tris.to(torch.int32).contiguous()
            kind, pv, pt = DEVICE, v.data_ptr(), t.data_ptr()
        else:
            v = np.ascontiguousarray(np.asarray(verts if not isinstance(verts, torch.Tensor) else verts.numpy(),
                                                dtype=np.float32))
            t = np.ascontiguousarray(np.asarray(tris if not isinstance(tris, torch.Tensor) else tris.numpy(),
                                                dtype=np.int32))
            kind, pv, pt = HOST, v.ctypes.data, t.ctypes.data
        V = int(v.shape[0]) if v.ndim > 1 else int(v.size) // 3
        T = int(t.shape[0]) if t.ndim > 1 else int(t.size) // 3
        _check(lib().fgl_scene_upload_mesh(self._h, pv, V, pt, T, kind | (0 if sync else ASYNC), _stream(stream)))
        self.T, self.V = T, V
        return self

    def build(self, morton_bits: int | None = None, leaf_size: int | None = None, morton_box: int | None = None,
              width: int | None = None, stream=None):
        mb = self.morton_box if morton_box is None else morton_box
        o = BuildOpts(morton_bits or self.morton_bits, leaf_size or self.leaf_size, int(mb),
                      int(width or self.width), int(self.quantized), int(self.restructure), int(self.treelets),
                      (c_int32 * 1)())
        _check(lib().fgl_scene_build(self._h, ctypes.byref(o), _stream(stream)))
        return self

    def refit(self, verts, stream=None, sync: bool = True):
        """New positions for the same vertices (NEXT-4): boxes and nodes recomputed, tree kept."""
        if isinstance(verts, torch.Tensor) and verts.is_cuda:
            v = verts.to(torch.float32).contiguous()
            kind, pv = DEVICE, v.data_ptr()
        else:
            v = np.ascontiguousarray(np.asarray(verts.cpu().numpy() if isinstance(verts, torch.Tensor) else verts,
                                                dtype=np.float32))
            kind, pv = HOST, v.ctypes.data
        V = int(np.prod(tuple(v.shape))) // 3
        _check(lib().fgl_scene_refit(self._h, pv, V, kind | (0 if sync else ASYNC), _stream(stream)))
        self._refit_keep = v
        return self

    def check(self, stream=None):
        """Synchronise and raise FglError if the last upload failed validation."""
        _check(lib().fgl_scene_check(self._h, _stream(stream)))
        return self

    def stats(self) -> dict:
        s = Stats()
        _check(lib().fgl_scene_stats(self._h, ctypes.byref(s)))
        return dict(triangles=s.triangles, vertices=s.vertices, nodes=s.nodes, device_bytes=s.device_bytes,
                    scene_lo=list(s.scene_lo), scene_hi=list(s.scene_hi), build_ms=s.build_ms,
                    morton_bits=s.morton_bits, leaf_size=s.leaf_size)

    # ---- casts -----------------------------------------------------------------------------
    def cast(self, poses, pattern, first_frame: int = 0, out=None, hit_xyz: bool = False, counts: bool = False,
             stream=None):
        """Cast every beam of `pattern` from every pose. Returns dict(range, tri_id[, hit_xyz,
        node_counts, tri_counts]) of device tensors shaped [P][C][A] (spinning) or [P][N]."""
        dev = self.device
        poses = _dev(poses, torch.float32, dev).reshape(-1, 3, 4)
        P = int(poses.shape[0])
        if is_spinning(pattern):
            shape = (P, len(pattern.elev_deg), int(pattern.columns))
        else:
            shape = (P, int(pattern.points_per_frame))
        if out is None:
            out = {}
        rng = out.get("range")
        if rng is None:
            rng = torch.empty(shape, dtype=torch.float32, device=dev)
        tid = out.get("tri_id")
        if tid is None:
            tid = torch.empty(shape, dtype=torch.int32, device=dev)
        hx = torch.empty(shape + (3,), dtype=torch.float32, device=dev) if hit_xyz else None
        nc = torch.empty(shape, dtype=torch.int32, device=dev) if counts else None
        tc = torch.empty(shape, dtype=torch.int32, device=dev) if counts else None
        st = _stream(stream)
        if is_spinning(pattern):
            s = spinning_struct(pattern)
            _check(lib().fgl_cast_spinning(self._h, ctypes.byref(s), poses.data_ptr(), P, rng.data_ptr(),
                                           tid.data_ptr(), _ptr(hx), _ptr(nc), _ptr(tc), st))
        else:
            s = rosette_struct(pattern)
            _check(lib().fgl_cast_rosette(self._h, ctypes.byref(s), poses.data_ptr(), P, int(first_frame),
                                          rng.data_ptr(), tid.data_ptr(), _ptr(hx), _ptr(nc), _ptr(tc), st))
        res = dict(range=rng, tri_id=tid)
        if hit_xyz:
            res["hit_xyz"] = hx
        if counts:
            res["node_counts"], res["tri_counts"] = nc, tc
        return res

    def cast_to_host(self, poses, pattern, range_out: torch.Tensor, tri_id_out: torch.Tensor, chunks: int = 8,
                     first_frame: int = 0, copy_stream=None, scratch=None, wait: bool = True):
        """Cast and stream the results to (pinned) host tensors, overlapping the device-to-host copy
        of chunk k with the cast of chunk k+1 (the copy runs on `copy_stream`). Returns when the
        copies are enqueued; the caller synchronises. `scratch` (optional) = dict(range, tri_id)
        device tensors of the full output shape, reused across calls. wait=False: the current
        stream does not wait for the copies; the returned event marks their completion."""
        dev = self.device
        cur = torch.cuda.current_stream(dev)
        cs = copy_stream or torch.cuda.Stream(device=dev)
        poses = _dev(poses, torch.float32, dev).reshape(-1, 3, 4)
        P = int(poses.shape[0])
        own_scratch = scratch is None
        if own_scratch:
            scratch = dict(range=torch.empty(range_out.shape, dtype=torch.float32, device=dev),
                           tri_id=torch.empty(tri_id_out.shape, dtype=torch.int32, device=dev))
            # the copies read it on `cs`: keep the allocator from reusing it before they finish
            scratch["range"].record_stream(cs)
            scratch["tri_id"].record_stream(cs)
        step = max(1, -(-P // max(1, chunks)))
        for a in range(0, P, step):
            b = min(P, a + step)
            self.cast(poses[a:b], pattern, first_frame=first_frame + a,
                      out=dict(range=scratch["range"][a:b], tri_id=scratch["tri_id"][a:b]))
            ev = torch.cuda.Event()
            ev.record(cur)
            cs.wait_event(ev)
            with torch.cuda.stream(cs):
                range_out[a:b].copy_(scratch["range"][a:b], non_blocking=True)
                tri_id_out[a:b].copy_(scratch["tri_id"][a:b], non_blocking=True)
        if wait:
            cur.wait_stream(cs)
            return range_out, tri_id_out
        done = torch.cuda.Event()
        done.record(cs)
        return done

    def cast_rays(self, orig, dir, t_min: float, t_max: float, bruteforce: bool = False, stream=None):
        o = _dev(orig, torch.float32, self.device, (-1, 3))
        d = _dev(dir, torch.float32, self.device, (-1, 3))
        R = int(o.shape[0])
        rng = torch.empty(R, dtype=torch.float32, device=self.device)
        tid = torch.empty(R, dtype=torch.int32, device=self.device)
        f = lib().fgl_cast_rays_bruteforce if bruteforce else lib().fgl_cast_rays
        _check(f(self._h, o.data_ptr(), d.data_ptr(), R, float(t_min), float(t_max), rng.data_ptr(), tid.data_ptr(),
                 _stream(stream)))
        return rng, tid

    # ---- internals for parity tests ------------------------------------------------------------
    def export(self, stream=None) -> dict:
        T = self.T
        nin = max(T - 1, 0)
        a = dict(scene_box=np.zeros(6, np.float32), codes=np.zeros(T, np.uint64), sorted_keys=np.zeros(T, np.uint64),
                 perm=np.zeros(T, np.uint32), child=np.zeros((nin, 2), np.int32), range=np.zeros((nin, 2), np.int32),
                 leaf_box=np.zeros((T, 6), np.float32), node_box=np.zeros((nin, 6), np.float32),
                 tri48=np.zeros((T, 12), np.float32), nodes=np.zeros((max(nin, 1), 16), np.float32),
                 nodes4=np.zeros((max(nin, 1), 32), np.float32), depth=np.zeros(nin, np.int32))
        e = ExportC(*[a[n].ctypes.data for n, _ in ExportC._fields_])
        _check(lib().fgl_scene_export(self._h, ctypes.byref(e), _stream(stream)))
        return a


def export_rays(pattern, poses, first_frame: int = 0, device=None, stream=None):
    """The exact float32 (origin, direction) the cast kernels generate, in output order."""
    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    poses = _dev(poses, torch.float32, device).reshape(-1, 3, 4)
    P = int(poses.shape[0])
    n = P * rays_per_pose(pattern)
    o = torch.empty((n, 3), dtype=torch.float32, device=device)
    d = torch.empty((n, 3), dtype=torch.float32, device=device)
    if is_spinning(pattern):
        s = spinning_struct(pattern)
        _check(lib().fgl_export_rays_spinning(ctypes.byref(s), poses.data_ptr(), P, o.data_ptr(), d.data_ptr(),
                                              _stream(stream)))
    else:
        s = rosette_struct(pattern)
        _check(lib().fgl_export_rays_rosette(ctypes.byref(s), poses.data_ptr(), P, int(first_frame), o.data_ptr(),
                                             d.data_ptr(), _stream(stream)))
    return o, d


def morton_codes(points: torch.Tensor, lo, hi, bits: int = 21, stream=None) -> torch.Tensor:
    p = points.to(torch.float32).contiguous().reshape(-1, 3)
    out = torch.empty(p.shape[0], dtype=torch.int64, device=p.device)
    lo = np.ascontiguousarray(lo, np.float32)
    hi = np.ascontiguousarray(hi, np.float32)
    _check(lib().fgl_morton_codes(p.data_ptr(), int(p.shape[0]), lo.ctypes.data, hi.ctypes.data, int(bits),
                                  out.data_ptr(), _stream(stream)))
    return out  # uint64 bit patterns in an int64 tensor


def sort_pairs(keys: torch.Tensor, vals: torch.Tensor, key_bits: int = 64, stream=None):
    """Stable radix sort in place of (uint64 key bit patterns in int64, int32/uint32 values)."""
    assert keys.dtype == torch.int64 and vals.dtype in (torch.int32, torch.uint32)
    assert keys.is_contiguous() and vals.is_contiguous() and keys.numel() == vals.numel()
    _check(lib().fgl_sort_pairs(keys.data_ptr(), vals.data_ptr(), int(keys.numel()), int(key_bits), _stream(stream)))
    return keys, vals


class DeviceBuffer:
    """Device memory from fgl_alloc (an allocation base, shareable by CUDA IPC) viewed as a torch
    tensor through __cuda_array_interface__. `ptr` may instead be a peer's buffer opened by IPC."""

    _TYPESTR = {torch.float32: "<f4", torch.int32: "<i4"}

    def __init__(self, shape, dtype, device, ptr: int | None = None, ipc: bool = False):
        self.shape, self.dtype, self.device = tuple(int(x) for x in shape), dtype, torch.device(device)
        self.nbytes = int(np.prod(self.shape)) * torch.tensor([], dtype=dtype).element_size()
        self._own = ptr is None
        self._ipc = ipc
        if ptr is None:
            p = c_void_p()
            _check(lib().fgl_alloc(self.device.index or 0, max(self.nbytes, 1), ctypes.byref(p)))
            ptr = p.value
        self.ptr = int(ptr)
        self.__cuda_array_interface__ = {"shape": self.shape, "typestr": self._TYPESTR[dtype],
                                         "data": (self.ptr, False), "version": 2}
        self.tensor = torch.as_tensor(self, device=self.device)

    def ipc_handle(self) -> bytes:
        h = (ctypes.c_ubyte * 64)()
        _check(lib().fgl_ipc_get_handle(self.ptr, ctypes.byref(h)))
        return bytes(h)

    @classmethod
    def open_ipc(cls, handle: bytes, shape, dtype, device):
        h = (ctypes.c_ubyte * 64).from_buffer_copy(handle)
        p = c_void_p()
        _check(lib().fgl_ipc_open_handle(torch.device(device).index or 0, ctypes.byref(h), ctypes.byref(p)))
        return cls(shape, dtype, device, ptr=p.value, ipc=True)

    def close(self):
        if getattr(self, "ptr", None) and _lib is not None:
            try:
                if self._ipc:
                    _lib.fgl_ipc_close_handle(self.ptr)
                elif self._own:
                    _lib.fgl_free(self.ptr)
            except Exception:
                pass
        self.ptr = None

    __del__ = close


def cast_spinning_gather(scene: "Scene", poses, pattern, first_pose: int, range_ptrs, tri_ptrs, flag_ptrs=None,
                         stream=None):
    """Fused cast + all-gather: this rank's poses are cast and each result is stored into every
    buffer of range_ptrs / tri_ptrs (device pointers; index 0 = this rank's own output) at global
    pose index first_pose + p. flag_ptrs (optional, same order): completion counters every rank's
    cast increments once, after a system-scope fence (see wait_flag)."""
    poses = _dev(poses, torch.float32, scene.device).reshape(-1, 3, 4)
    s = spinning_struct(pattern)
    W = len(range_ptrs)
    rp = (c_void_p * W)(*range_ptrs)
    tp = (c_void_p * W)(*tri_ptrs)
    fp = None if flag_ptrs is None else (c_void_p * W)(*flag_ptrs)
    _check(lib().fgl_cast_spinning_gather_signal(scene._h, ctypes.byref(s), poses.data_ptr() if poses.numel() else None,
                                                 int(poses.shape[0]), int(first_pose), rp, tp, fp, W,
                                                 _stream(stream)))


def wait_flag(flag_ptr: int, target: int, stream=None):
    """Make the stream wait (on the device) until the int32 counter at flag_ptr reaches target."""
    _check(lib().fgl_wait_flag(flag_ptr, int(target), _stream(stream)))


class PointCloud:
    """A point cloud indexed by the LBVH (point scene) for exact nearest-neighbour queries."""

    def __init__(self, xyz, device=None, stream=None):
        self.scene = Scene(device=device, build=False, leaf_size=2, width=2)
        self.device = self.scene.device
        on_dev = isinstance(xyz, torch.Tensor) and xyz.is_cuda
        if on_dev:
            x = xyz.to(torch.float32).contiguous().reshape(-1, 3)
            kind, ptr = DEVICE, x.data_ptr()
        else:
            x = np.ascontiguousarray(np.asarray(xyz.cpu().numpy() if isinstance(xyz, torch.Tensor) else xyz,
                                                dtype=np.float32).reshape(-1, 3))
            kind, ptr = HOST, x.ctypes.data
        self.n = int(x.shape[0])
        _check(lib().fgl_scene_upload_points(self.scene._h, ptr, self.n, kind, _stream(stream)))
        self.scene.T = self.n
        self.scene.build(stream=stream)

    def nearest(self, queries, stream=None):
        q = _dev(queries, torch.float32, self.device, (-1, 3))
        m = int(q.shape[0])
        d = torch.empty(m, dtype=torch.float32, device=self.device)
        i = torch.empty(m, dtype=torch.int32, device=self.device)
        _check(lib().fgl_nearest(self.scene._h, q.data_ptr(), m, d.data_ptr(), i.data_ptr(), _stream(stream)))
        return d, i


def cloud_metrics(a, b, tau: float, device=None, stream=None) -> dict:
    """Symmetric Chamfer distance, precision, recall and F-score of clouds a, b (§V-A):
    two exact nearest-neighbour passes over LBVH-indexed clouds + one reduction kernel."""
    ca, cb = PointCloud(a, device, stream), PointCloud(b, device, stream)
    d_ab, _ = cb.nearest(_dev(a, torch.float32, cb.device, (-1, 3)), stream)
    d_ba, _ = ca.nearest(_dev(b, torch.float32, ca.device, (-1, 3)), stream)
    out = torch.empty(6, dtype=torch.float64, device=ca.device)
    _check(lib().fgl_cloud_metrics(d_ab.data_ptr(), int(d_ab.numel()), d_ba.data_ptr(), int(d_ba.numel()),
                                   float(tau), out.data_ptr(), _stream(stream)))
    o = out.cpu().tolist()
    return dict(chamfer=o[0], precision=o[1], recall=o[2], fscore=o[3], n_a=int(o[4]), n_b=int(o[5]),
                d_ab=d_ab, d_ba=d_ba)


class GaussianScene:
    """A 3DGS cloud on one GPU with its LBVH over the Eq. 4 boxes (§IV-A), for
    voxelize() (Eqs. 8-12). mu [N][3], quat [N][4] (w, x, y, z), scale [N][3], opacity [N]: host
    arrays or CUDA tensors (float32)."""

    def __init__(self, mu, quat, scale, opacity, kappa: float = 3.0, device=None, build: bool = True,
                 leaf_size: int = 2, morton_bits: int = 0, stream=None, sync: bool = True):
        self.scene = Scene(device=device, build=False, leaf_size=leaf_size, width=2, morton_bits=morton_bits)
        self.device = self.scene.device
        self.kappa = float(kappa)
        self.upload(mu, quat, scale, opacity, stream, sync)
        if build:
            self.build(stream)

    def upload(self, mu, quat, scale, opacity, stream=None, sync: bool = True):
        arrs = [mu, quat, scale, opacity]
        on_dev = all(isinstance(a, torch.Tensor) and a.is_cuda for a in arrs)
        if on_dev:
            keep = [a.to(torch.float32).contiguous() for a in arrs]
            ptrs = [a.data_ptr() for a in keep]
            kind = DEVICE
        else:
            keep = [np.ascontiguousarray(np.asarray(a.cpu().numpy() if isinstance(a, torch.Tensor) else a,
                                                    dtype=np.float32)) for a in arrs]
            ptrs = [a.ctypes.data for a in keep]
            kind = HOST
        n = int(np.prod(tuple(keep[3].shape)))
        for a, w in zip(keep[:3], (3, 4, 3)):
            if int(np.prod(tuple(a.shape))) != n * w:
                raise ValueError("mu / quat / scale must be [N][3] / [N][4] / [N][3] with N = len(opacity)")
        _check(lib().fgl_scene_upload_gaussians(self.scene._h, *ptrs, n, self.kappa, kind | (0 if sync else ASYNC),
                                                _stream(stream)))
        self._keep = keep  # host arrays must outlive an async upload
        self.N = self.scene.T = n
        return self

    def build(self, stream=None):
        self.scene.build(stream=stream)
        return self

    def check(self, stream=None):
        self.scene.check(stream)
        return self

    def stats(self) -> dict:
        return self.scene.stats()

    def voxelize(self, origin, spacing: float, dims, theta: float, density: bool = False, masks: bool = True,
                 counts: bool = True, out=None, stream=None) -> dict:
        """Occupancy (Eq. 10) and, with masks, surface / interior (Eqs. 11-12) bit volumes uint32
        [nz][ny][ceil(nx / 32)]; density float32 [nz][ny][nx] on request; counts int64 [4] =
        (occupied, surface, evaluated pairs, overflow)."""
        nx, ny, nz = (int(d) for d in dims)
        nw = (nx + 31) // 32
        dev = self.device
        out = {} if out is None else out
        occ = out.get("occupancy")
        if occ is None:
            occ = torch.empty((nz, ny, nw), dtype=torch.int32, device=dev)
        dens = out.get("density")
        if density and dens is None:
            dens = torch.empty((nz, ny, nx), dtype=torch.float32, device=dev)
        surf = inter = None
        if masks:
            surf = out.get("surface")
            if surf is None:
                surf = torch.empty((nz, ny, nw), dtype=torch.int32, device=dev)
            inter = out.get("interior")
            if inter is None:
                inter = torch.empty((nz, ny, nw), dtype=torch.int32, device=dev)
        cnt = out.get("counts")
        if counts and cnt is None:
            cnt = torch.empty(4, dtype=torch.int64, device=dev)
        g = GridC((c_float * 3)(*[float(o) for o in origin]), float(spacing), (c_int32 * 3)(nx, ny, nz), 0,
                  float(theta), (c_int32 * 3)())
        _check(lib().fgl_voxelize(self.scene._h, ctypes.byref(g), _ptr(dens if density else None), occ.data_ptr(),
                                  _ptr(surf), _ptr(inter), _ptr(cnt if counts else None), _stream(stream)))
        res = dict(occupancy=occ)
        if density:
            res["density"] = dens
        if masks:
            res["surface"], res["interior"] = surf, inter
        if counts:
            res["counts"] = cnt
        return res


# ---- occupancy -> mesh (§IV-B, NEXT-3) -----------------------------------------------------------
def _vol_args(dims, spacing):
    d = (c_int32 * 3)(*[int(x) for x in dims])
    sp = (c_float * 3)(*([float(spacing)] * 3 if np.isscalar(spacing) else [float(x) for x in spacing]))
    return d, sp


def denoise(occupancy: torch.Tensor, dims, spacing, sigma: float, tau: float, vprime: bool = False, out=None,
            stream=None):
    """Eqs. 13-14a on a device bit volume: returns the re-thresholded bit volume (and V' float32
    [nz][ny][nx] when vprime)."""
    d, sp = _vol_args(dims, spacing)
    out = torch.empty_like(occupancy) if out is None else out
    vp = torch.empty((int(dims[2]), int(dims[1]), int(dims[0])), dtype=torch.float32,
                     device=occupancy.device) if vprime else None
    _check(lib().fgl_denoise(occupancy.data_ptr(), d, sp, float(sigma), float(tau), out.data_ptr(), _ptr(vp),
                             _stream(stream)))
    return (out, vp) if vprime else out


def denoise_quantile(occupancy: torch.Tensor, dims, spacing, sigma: float, q: float, vprime: bool = False, out=None,
                     stream=None):
    """Eqs. 13-14b: blur, then threshold at Quantile_q(V'). Returns (bits, threshold[, V'])."""
    d, sp = _vol_args(dims, spacing)
    out = torch.empty_like(occupancy) if out is None else out
    vp = torch.empty((int(dims[2]), int(dims[1]), int(dims[0])), dtype=torch.float32,
                     device=occupancy.device) if vprime else None
    thr = torch.empty(1, dtype=torch.float32, device=occupancy.device)
    _check(lib().fgl_denoise_quantile(occupancy.data_ptr(), d, sp, float(sigma), float(q), out.data_ptr(), _ptr(vp),
                                      thr.data_ptr(), _stream(stream)))
    return (out, thr, vp) if vprime else (out, thr)


def tsdf(occupancy: torch.Tensor, dims, spacing, r: float, out=None, stream=None) -> torch.Tensor:
    """Eqs. 15-17 narrow-band TSDF phi float32 [nz][ny][nx] of a device bit volume."""
    d, sp = _vol_args(dims, spacing)
    phi = out if out is not None else torch.empty((int(dims[2]), int(dims[1]), int(dims[0])), dtype=torch.float32,
                                                  device=occupancy.device)
    _check(lib().fgl_tsdf(occupancy.data_ptr(), d, sp, float(r), phi.data_ptr(), _stream(stream)))
    return phi


def marching_cubes(phi: torch.Tensor, origin, spacing, iso: float = 0.0, normals: bool = False, out=None,
                   stream=None) -> dict:
    """Eq. 18 on phi [nz][ny][nx] (device): dict(verts float32 [V][3], tris int32 [T][3][, normals]).
    Sizes come from a counting pass (one host sync) unless `out` carries buffers large enough
    (verts, tris[, normals], counts) — then the call is sync-free and the first counts entries are
    valid."""
    nz, ny, nx = phi.shape
    d, sp = _vol_args((nx, ny, nz), spacing)
    o = (c_float * 3)(*[float(x) for x in origin])
    dev = phi.device
    st = _stream(stream)
    if out is None:
        cnt = torch.zeros(2, dtype=torch.int64, device=dev)
        _check(lib().fgl_marching_cubes(phi.data_ptr(), d, o, sp, float(iso), None, None, 0, None, 0, cnt.data_ptr(),
                                        st))
        nv, nt = (int(x) for x in cnt.cpu())
        out = dict(verts=torch.empty((max(nv, 1), 3), dtype=torch.float32, device=dev),
                   tris=torch.empty((max(nt, 1), 3), dtype=torch.int32, device=dev), counts=cnt)
        if normals:
            out["normals"] = torch.empty((max(nv, 1), 3), dtype=torch.float32, device=dev)
        sized = (nv, nt)
    else:
        sized = None
    v, t, c = out["verts"], out["tris"], out["counts"]
    nrm = out.get("normals") if normals else None
    _check(lib().fgl_marching_cubes(phi.data_ptr(), d, o, sp, float(iso), v.data_ptr(), _ptr(nrm), int(v.shape[0]),
                                    t.data_ptr(), int(t.shape[0]), c.data_ptr(), st))
    if sized is None:
        return out
    res = dict(verts=v[:sized[0]], tris=t[:sized[1]], counts=c)
    if normals:
        res["normals"] = nrm[:sized[0]]
    return res


def l2_read_probe(buf: torch.Tensor, iters: int, sink: torch.Tensor, stream=None) -> None:
    """Enqueue the L2 read-bandwidth probe over the device tensor `buf` (fgl_l2_read_probe)."""
    _check(lib().fgl_l2_read_probe(buf.data_ptr(), buf.numel() * buf.element_size(), int(iters), sink.data_ptr(),
                                   _stream(stream)))


def kernel_launches() -> int:
    """Kernels libfgl.so has launched in this process (the bench's gpu_launches evidence)."""
    return int(lib().fgl_kernel_launches())


def version() -> str:
    return lib().fgl_version().decode()
