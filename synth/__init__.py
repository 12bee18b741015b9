"""Seeded synthetic inputs shared by the CUDA path (bench, smoke, tests) and the oracle (tests).

This module holds NONE of the method's arithmetic: no ray generation, no intersection, no Morton
codes, no BVH. It only produces the *inputs* of the LiDAR cast problem stated in PAPER.md §IV-C
(P:261-268): a triangle mesh M = {Δ_k} (float32 vertices + int32 indices), sensor poses
T_s ∈ SE(3) (float32 [P][3][4] row-major (R|t), sensor->world), and scan-pattern *parameters*
(elevation tables, column counts, rosette phase increments). How those parameters turn into ray
directions is each side's own business (oracle/oracle.c and the CUDA ray generator).

The paper's scenes are converted 3DGS assets that are not available offline, so the scenes
here are procedural stand-ins at the paper's million-triangle scale (DESIGN.md
"Input recipe"). Everything is deterministic given the seed.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Mesh", "merge", "icosphere", "box", "cylinder", "floor_grid", "soup",
    "scene_c1", "scene_rooms", "scene_terrain", "Terrain",
    "Spinning", "Rosette", "spinning_preset", "rosette_default",
    "pose", "poses_yaw_offsets", "trajectory_rooms", "poses_terrain", "random_poses",
    "config", "Gaussians", "gaussians_random", "gaussians_on_mesh", "Grid", "grid_for", "gauss_config",
]


# ----------------------------------------------------------------------------------------------
# meshes
# ----------------------------------------------------------------------------------------------
@dataclass
class Mesh:
    verts: np.ndarray  # float32 [V][3]
    tris: np.ndarray   # int32 [T][3]
    meta: dict = field(default_factory=dict)

    @property
    def T(self) -> int:
        return int(self.tris.shape[0])

    @property
    def V(self) -> int:
        return int(self.verts.shape[0])


def _mk(v, t, **meta) -> Mesh:
    return Mesh(np.ascontiguousarray(v, dtype=np.float32), np.ascontiguousarray(t, dtype=np.int32), dict(meta))


def merge(meshes) -> Mesh:
    vs, ts, off = [], [], 0
    for m in meshes:
        vs.append(m.verts)
        ts.append(m.tris.astype(np.int64) + off)
        off += m.V
    if not vs:
        return _mk(np.zeros((0, 3)), np.zeros((0, 3)))
    return _mk(np.concatenate(vs), np.concatenate(ts))


def icosphere(level: int, radius: float, center=(0.0, 0.0, 0.0)) -> Mesh:
    """Subdivided icosahedron: 20·4^level faces, vertices on the sphere (then rounded to float32)."""
    p = (1.0 + 5.0 ** 0.5) / 2.0
    v = [(-1, p, 0), (1, p, 0), (-1, -p, 0), (1, -p, 0), (0, -1, p), (0, 1, p), (0, -1, -p), (0, 1, -p),
         (p, 0, -1), (p, 0, 1), (-p, 0, -1), (-p, 0, 1)]
    f = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2),
         (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5),
         (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    verts = [np.array(x, dtype=np.float64) / np.linalg.norm(x) for x in v]
    faces = list(f)
    for _ in range(level):
        cache = {}

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in cache:
                m = verts[a] + verts[b]
                verts.append(m / np.linalg.norm(m))
                cache[key] = len(verts) - 1
            return cache[key]

        nf = []
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = nf
    V = np.array(verts) * radius + np.asarray(center, dtype=np.float64)
    return _mk(V, np.array(faces), kind="icosphere", level=level, radius=radius, center=tuple(center))


def _axis_counts(lo, hi, h):
    ext = np.asarray(hi, np.float64) - np.asarray(lo, np.float64)
    if h is None:
        return np.ones(3, dtype=np.int64)
    return np.maximum(1, np.ceil(ext / h - 1e-9)).astype(np.int64)


def box_tri_count(lo, hi, h=None) -> int:
    n = _axis_counts(lo, hi, h)
    return int(4 * (n[0] * n[1] + n[1] * n[2] + n[0] * n[2]))


def _grid_quads(nu, nv):
    """Triangles of an (nu+1)x(nv+1) vertex grid, vertex (i,j) at i*(nv+1)+j. Cell (i,j) ->
    (p00,p10,p11) then (p00,p11,p01)."""
    i, j = np.meshgrid(np.arange(nu), np.arange(nv), indexing="ij")
    p00 = (i * (nv + 1) + j).ravel()
    p10 = ((i + 1) * (nv + 1) + j).ravel()
    p11 = ((i + 1) * (nv + 1) + j + 1).ravel()
    p01 = (i * (nv + 1) + j + 1).ravel()
    t = np.empty((p00.size * 2, 3), dtype=np.int64)
    t[0::2] = np.stack([p00, p10, p11], 1)
    t[1::2] = np.stack([p00, p11, p01], 1)
    return t


def box(lo, hi, h=None) -> Mesh:
    """Closed axis-aligned box surface, each face tessellated into a grid whose per-axis counts are
    shared by all faces, so the vertices on every box edge are the same float32 values (closed,
    no T-junctions). Faces wound outward."""
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    n = _axis_counts(lo, hi, h)
    ax = [np.linspace(lo[a], hi[a], n[a] + 1) for a in range(3)]
    vs, ts, off = [], [], 0
    for a in range(3):
        b, c = (a + 1) % 3, (a + 2) % 3
        for side, val in ((0, lo[a]), (1, hi[a])):
            U, W = np.meshgrid(ax[b], ax[c], indexing="ij")
            P = np.empty((U.size, 3))
            P[:, a] = val
            P[:, b] = U.ravel()
            P[:, c] = W.ravel()
            t = _grid_quads(n[b], n[c])
            if side == 0:
                t = t[:, [0, 2, 1]]
            vs.append(P)
            ts.append(t + off)
            off += P.shape[0]
    return _mk(np.concatenate(vs), np.concatenate(ts), kind="box", lo=tuple(lo), hi=tuple(hi))


def cylinder(cx, cy, z0, z1, r, segments=32, h=None) -> Mesh:
    """Closed vertical cylinder (prism with `segments` sides), side tessellated vertically, fan caps."""
    nz = 1 if h is None else max(1, int(math.ceil((z1 - z0) / h - 1e-9)))
    th = 2.0 * np.pi * np.arange(segments) / segments
    zs = np.linspace(z0, z1, nz + 1)
    ring = np.stack([cx + r * np.cos(th), cy + r * np.sin(th)], 1)
    side = np.empty(((nz + 1) * segments, 3))
    for k, z in enumerate(zs):
        side[k * segments:(k + 1) * segments, :2] = ring
        side[k * segments:(k + 1) * segments, 2] = z
    tris = []
    for k in range(nz):
        for s in range(segments):
            a = k * segments + s
            b = k * segments + (s + 1) % segments
            tris += [(a, b, b + segments), (a, b + segments, a + segments)]
    nv = side.shape[0]
    cb, ct = nv, nv + 1
    for s in range(segments):
        a, b = s, (s + 1) % segments
        tris.append((cb, b, a))
        tris.append((ct, nz * segments + a, nz * segments + b))
    V = np.concatenate([side, [[cx, cy, z0], [cx, cy, z1]]])
    return _mk(V, np.array(tris), kind="cylinder")


def cylinder_tri_count(z0, z1, segments=32, h=None) -> int:
    nz = 1 if h is None else max(1, int(math.ceil((z1 - z0) / h - 1e-9)))
    return 2 * segments * nz + 2 * segments


def floor_grid(nx: int, ny: int, delta: float, z: float = 0.0, x0: float = 0.0, y0: float = 0.0) -> Mesh:
    """Tessellated plane z = const. Cell (i, j) (i along x, j along y) owns triangles
    2*(i*ny+j) = (p00,p10,p11) (the half with frac_x >= frac_y) and 2*(i*ny+j)+1 = (p00,p11,p01)."""
    xs = x0 + delta * np.arange(nx + 1)
    ys = y0 + delta * np.arange(ny + 1)
    X, Y = np.meshgrid(xs, ys, indexing="ij")
    V = np.stack([X.ravel(), Y.ravel(), np.full(X.size, z)], 1)
    return _mk(V, _grid_quads(nx, ny), kind="floor_grid", nx=nx, ny=ny, delta=delta, z=z, x0=x0, y0=y0)


def soup(T: int, seed: int = 7, extent: float = 10.0, size: float | None = None) -> Mesh:
    """Uniform random triangle soup in [0, extent]^3 (the S:487/S:652 scaling workload)."""
    rng = np.random.default_rng(seed)
    if size is None:
        size = 1.5 * extent / max(T, 1) ** (1.0 / 3.0)
    c = rng.uniform(0.0, extent, size=(T, 1, 3))
    v = c + rng.uniform(-size, size, size=(T, 3, 3))
    return _mk(v.reshape(-1, 3), np.arange(3 * T).reshape(T, 3), kind="soup", seed=seed)


# ----------------------------------------------------------------------------------------------
# C1: icosphere level 3, circumradius 10 m + box
# ----------------------------------------------------------------------------------------------
def scene_c1() -> Mesh:
    m = merge([icosphere(3, 10.0), box((1.0, -1.0, -2.0), (3.0, 1.0, -0.5))])
    m.meta.update(kind="c1")
    return m


# ----------------------------------------------------------------------------------------------
# C2/C4: procedural indoor rooms, ~1 M triangles
# ----------------------------------------------------------------------------------------------
ROOM = dict(RX=6.0, RY=5.0, RZ=3.0, NX=4, NY=4, WALL=0.2, DOOR_W=1.0, DOOR_H=2.1)


def _rooms_primitives(seed: int):
    """List of ('box', lo, hi) / ('cyl', cx, cy, z0, z1, r) / ('ico', cx, cy, cz, r) specs."""
    RX, RY, RZ, NX, NY, W = ROOM["RX"], ROOM["RY"], ROOM["RZ"], ROOM["NX"], ROOM["NY"], ROOM["WALL"]
    dw, dh = ROOM["DOOR_W"], ROOM["DOOR_H"]
    hw = W / 2
    prims = []
    X1, Y1 = NX * RX, NY * RY
    prims.append(("box", (-hw, -hw, -W), (X1 + hw, Y1 + hw, 0.0)))           # floor slab
    prims.append(("box", (-hw, -hw, RZ), (X1 + hw, Y1 + hw, RZ + W)))        # ceiling slab

    def wall_line(axis, pos, n_rooms, room_len, doors):
        # axis: 0 -> wall spans along y at x=pos ; 1 -> spans along x at y=pos
        out = []
        if not doors:
            segs = [(-hw, n_rooms * room_len + hw, 0.0, RZ)]
        else:
            segs = []
            for k in range(n_rooms):
                a, b = k * room_len - hw, (k + 1) * room_len + hw
                c = (k + 0.5) * room_len
                segs += [(a, c - dw / 2, 0.0, RZ), (c - dw / 2, c + dw / 2, dh, RZ), (c + dw / 2, b, 0.0, RZ)]
        for a, b, z0, z1 in segs:
            if axis == 0:
                out.append(("box", (pos - hw, a, z0), (pos + hw, b, z1)))
            else:
                out.append(("box", (a, pos - hw, z0), (b, pos + hw, z1)))
        return out

    for i in range(NX + 1):
        prims += wall_line(0, i * RX, NY, RY, doors=(0 < i < NX))
    for j in range(NY + 1):
        prims += wall_line(1, j * RY, NX, RX, doors=(0 < j < NY))

    rng = np.random.default_rng(seed)
    lift = 1e-3  # furniture raised 1 mm above the floor: no coplanar overlap
    for i in range(NX):
        for j in range(NY):
            cx, cy = (i + 0.5) * RX, (j + 0.5) * RY
            quads = rng.permutation(4)
            kinds = ["table", "cabinet", "cyl", "ico"]
            for q, kind in zip(quads, kinds):
                sx = 1 if q & 1 else -1
                sy = 1 if q & 2 else -1
                # usable quadrant span: from 0.8 m off the centre lines to 0.3 m off the walls
                ax0, ax1 = 0.8, RX / 2 - hw - 0.3
                ay0, ay1 = 0.8, RY / 2 - hw - 0.3
                if kind == "table":
                    w, d, ht = rng.uniform(0.8, 1.3), rng.uniform(0.6, 0.9), 0.75
                elif kind == "cabinet":
                    w, d, ht = rng.uniform(0.4, 0.6), rng.uniform(0.8, 1.2), rng.uniform(1.6, 2.0)
                elif kind == "cyl":
                    r = rng.uniform(0.15, 0.3)
                    w = d = 2 * r
                    ht = rng.uniform(0.5, 1.2)
                else:
                    r = rng.uniform(0.25, 0.4)
                    w = d = 2 * r
                    ht = 2 * r
                ox = rng.uniform(ax0, ax1 - w)
                oy = rng.uniform(ay0, ay1 - d)
                x0 = cx + ox if sx > 0 else cx - ox - w
                y0 = cy + oy if sy > 0 else cy - oy - d
                if kind in ("table", "cabinet"):
                    prims.append(("box", (x0, y0, lift), (x0 + w, y0 + d, ht)))
                elif kind == "cyl":
                    prims.append(("cyl", x0 + r, y0 + r, lift, ht, r))
                else:
                    prims.append(("ico", x0 + r, y0 + r, r + lift, r))
    return prims


def _prims_count(prims, h):
    n = 0
    for p in prims:
        if p[0] == "box":
            n += box_tri_count(p[1], p[2], h)
        elif p[0] == "cyl":
            n += cylinder_tri_count(p[3], p[4], 32, h)
        else:
            n += 20 * 4 ** 3
    return n


def _tune_h(prims, target, lo=0.005, hi=2.0):
    for _ in range(60):
        mid = math.sqrt(lo * hi)
        if _prims_count(prims, mid) > target:
            lo = mid
        else:
            hi = mid
    # pick whichever bracket end is closer to target
    a, b = _prims_count(prims, lo), _prims_count(prims, hi)
    return lo if abs(a - target) <= abs(b - target) else hi


def _emit(prims, h):
    ms = []
    for p in prims:
        if p[0] == "box":
            ms.append(box(p[1], p[2], h))
        elif p[0] == "cyl":
            ms.append(cylinder(p[1], p[2], p[3], p[4], p[5], 32, h))
        else:
            ms.append(icosphere(3, p[4], (p[1], p[2], p[3])))
    return merge(ms)


def scene_rooms(seed: int = 2, target_tris: int = 1_000_000) -> Mesh:
    """4x4 grid of 6x5x3 m rooms: 0.2 m wall slabs with 1.0x2.1 m door openings on every interior
    wall, floor and ceiling slabs, and 4 pieces of furniture per room (table, cabinet, 32-segment
    cylinder, level-3 icosphere) kept 0.8 m off the room centre lines. Surfaces tessellated
    near-uniformly with edge length h, h tuned so T ~ target_tris."""
    prims = _rooms_primitives(seed)
    h = _tune_h(prims, target_tris)
    m = _emit(prims, h)
    m.meta.update(kind="rooms", seed=seed, h=h, **ROOM)
    return m


# ----------------------------------------------------------------------------------------------
# C3/C5: outdoor height-field terrain + buildings, ~10 M triangles
# ----------------------------------------------------------------------------------------------
@dataclass
class Terrain:
    mesh: Mesh
    heights: np.ndarray  # float32 [n+1][n+1] vertex heights, (i along x, j along y)
    x0: float
    cell: float
    n: int
    footprints: np.ndarray  # float64 [B][4] building footprints (x0, y0, x1, y1)

    def surface_z(self, x, y):
        """Height of the terrain *mesh* (piecewise planar, cell diagonal p00-p11) at (x, y)."""
        x = np.asarray(x, np.float64)
        y = np.asarray(y, np.float64)
        H = self.heights.astype(np.float64)
        gx = (x - self.x0) / self.cell
        gy = (y - self.x0) / self.cell
        i = np.clip(np.floor(gx).astype(np.int64), 0, self.n - 1)
        j = np.clip(np.floor(gy).astype(np.int64), 0, self.n - 1)
        fx, fy = gx - i, gy - j
        h00, h10, h11, h01 = H[i, j], H[i + 1, j], H[i + 1, j + 1], H[i, j + 1]
        lower = fx >= fy
        z_lo = h00 + fx * (h10 - h00) + fy * (h11 - h10)
        z_up = h00 + fx * (h11 - h01) + fy * (h01 - h00)
        return np.where(lower, z_lo, z_up)

    def inside_building(self, x, y, margin=1.0):
        x = np.asarray(x, np.float64)[..., None]
        y = np.asarray(y, np.float64)[..., None]
        f = self.footprints
        return np.any((x >= f[:, 0] - margin) & (x <= f[:, 2] + margin) &
                      (y >= f[:, 1] - margin) & (y <= f[:, 3] + margin), axis=-1)


def _fbm(X, Y, seed, octaves=4, amplitude=8.0, base_period=256.0):
    rng = np.random.default_rng(seed)
    Z = np.zeros_like(X)
    amp, period, norm = 1.0, base_period, 0.0
    for _ in range(octaves):
        gx, gy = X / period, Y / period
        ix, iy = np.floor(gx), np.floor(gy)
        fx, fy = gx - ix, gy - iy
        ix = ix.astype(np.int64)
        iy = iy.astype(np.int64)
        ox, oy = ix.min(), iy.min()
        L = rng.uniform(-1.0, 1.0, size=(ix.max() - ox + 2, iy.max() - oy + 2))
        ix -= ox
        iy -= oy
        sx = fx * fx * (3 - 2 * fx)
        sy = fy * fy * (3 - 2 * fy)
        a = L[ix, iy] * (1 - sx) + L[ix + 1, iy] * sx
        b = L[ix, iy + 1] * (1 - sx) + L[ix + 1, iy + 1] * sx
        Z += amp * (a * (1 - sy) + b * sy)
        norm += amp
        amp *= 0.5
        period *= 0.5
    return amplitude * Z / norm


def scene_terrain(seed: int = 3, cells: int = 2048, size: float = 1024.0,
                  target_tris: int = 9_990_000, n_buildings: int = 400) -> Terrain:
    """Height field over [-size/2, size/2]^2 with `cells`^2 cells (2 tris each; fBm, 4 octaves,
    8 m amplitude) plus box buildings sunk 1 m into the ground, tessellated so T ~ target_tris.
    A 40 m radius around the origin is kept free of buildings (the C3 sensor sits there)."""
    cell = size / cells
    x0 = -size / 2
    xs = x0 + cell * np.arange(cells + 1)
    X, Y = np.meshgrid(xs, xs, indexing="ij")
    Hh = _fbm(X, Y, seed).astype(np.float32)
    V = np.stack([X.ravel(), Y.ravel(), Hh.ravel().astype(np.float64)], 1)
    ground = _mk(V, _grid_quads(cells, cells), kind="terrain_ground")

    rng = np.random.default_rng(seed + 1000)
    g = int(math.ceil(math.sqrt(n_buildings * 1.6)))
    pitch = 0.9 * size / g
    slots = [(a, b) for a in range(g) for b in range(g)]
    rng.shuffle(slots)
    feet, prims = [], []
    for a, b in slots:
        if len(prims) >= n_buildings:
            break
        cxs = -0.45 * size + (a + 0.5) * pitch
        cys = -0.45 * size + (b + 0.5) * pitch
        w, d = rng.uniform(8.0, min(30.0, 0.8 * pitch), size=2)
        bx0 = cxs - w / 2 + rng.uniform(-0.05, 0.05) * pitch
        by0 = cys - d / 2 + rng.uniform(-0.05, 0.05) * pitch
        if math.hypot(bx0 + w / 2, by0 + d / 2) < 40.0 + max(w, d):
            continue
        i0, i1 = int((bx0 - x0) / cell), int(math.ceil((bx0 + w - x0) / cell))
        j0, j1 = int((by0 - x0) / cell), int(math.ceil((by0 + d - x0) / cell))
        zmin = float(Hh[i0:i1 + 1, j0:j1 + 1].min()) - 1.0
        zmax = float(Hh[i0:i1 + 1, j0:j1 + 1].max()) + rng.uniform(6.0, 40.0)
        prims.append(("box", (bx0, by0, zmin), (bx0 + w, by0 + d, zmax)))
        feet.append((bx0, by0, bx0 + w, by0 + d))
    h = _tune_h(prims, max(target_tris - ground.T, len(prims) * 12), lo=0.05, hi=200.0)
    bld = _emit(prims, h)
    m = merge([ground, bld])
    m.meta.update(kind="terrain", seed=seed, cells=cells, size=size, h_buildings=h, n_buildings=len(prims))
    return Terrain(m, Hh, x0, cell, cells, np.array(feet, dtype=np.float64).reshape(-1, 4))


# ----------------------------------------------------------------------------------------------
# scan-pattern parameters (no direction arithmetic here)
# ----------------------------------------------------------------------------------------------
@dataclass
class Spinning:
    """Spinning multi-beam pattern parameters: channel elevations (degrees, float32,
    monotone), columns per revolution A, azimuth offset (degrees), range interval [t_min, t_max]."""
    elev_deg: np.ndarray
    columns: int
    az0_deg: float = 0.0
    t_min: float = 0.1
    t_max: float = 200.0
    name: str = "custom"

    @property
    def channels(self) -> int:
        return int(self.elev_deg.shape[0])

    @property
    def rays_per_pose(self) -> int:
        return self.channels * self.columns


_PRESETS = {
    # name: (channels, elev_lo, elev_hi, default columns)   elevations uniform
    "VLP16": (16, -15.0, 15.0, 360),
    "HDL64": (64, -24.9, 2.0, 2048),
    "OS128": (128, -22.5, 22.5, 2048),
    "VLP32": (32, -25.0, 15.0, 1800),
}


def spinning_preset(name: str, columns: int | None = None, az0_deg: float = 0.0) -> Spinning:
    c, lo, hi, cols = _PRESETS[name]
    e = np.linspace(lo, hi, c).astype(np.float32)
    return Spinning(e, int(columns or cols), float(az0_deg), 0.1, 200.0, name)


@dataclass
class Rosette:
    """Two-prism (Risley) non-repetitive pattern parameters (reading R-rosette).
    Phase increments are turns * 2^32 per sample (exact integer phase, no float drift)."""
    points_per_frame: int = 20000
    inc1: int = 2611340   # round(2^32 * 121.6 Hz / 200 kHz)
    inc2: int = 1668595   # round(2^32 *  77.7 Hz / 200 kHz), counter-rotating
    phase2_0: int = 0
    half_fov_deg: float = 35.2
    t_min: float = 0.1
    t_max: float = 200.0


def rosette_default() -> Rosette:
    return Rosette()


# ----------------------------------------------------------------------------------------------
# poses: float32 [P][3][4] row-major (R | t), sensor -> world
# ----------------------------------------------------------------------------------------------
def _rot(yaw=0.0, pitch=0.0, roll=0.0):
    cy, sy = math.cos(yaw), math.sin(yaw)
    cp, sp = math.cos(pitch), math.sin(pitch)
    cr, sr = math.cos(roll), math.sin(roll)
    Rz = np.array([[cy, -sy, 0], [sy, cy, 0], [0, 0, 1]])
    Ry = np.array([[cp, 0, sp], [0, 1, 0], [-sp, 0, cp]])
    Rx = np.array([[1, 0, 0], [0, cr, -sr], [0, sr, cr]])
    return Rz @ Ry @ Rx


def pose(t, yaw=0.0, pitch=0.0, roll=0.0) -> np.ndarray:
    M = np.zeros((3, 4))
    M[:, :3] = _rot(yaw, pitch, roll)
    M[:, 3] = t
    return M.astype(np.float32)


def poses_yaw_offsets(t, n: int, step_rad: float) -> np.ndarray:
    return np.stack([pose(t, yaw=k * step_rad) for k in range(n)])


def random_poses(P: int, seed: int, lo, hi, full_rotation: bool = True) -> np.ndarray:
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(P):
        t = rng.uniform(lo, hi)
        if full_rotation:
            q = rng.normal(size=4)
            q /= np.linalg.norm(q)
            w, x, y, z = q
            R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                          [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                          [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])
        else:
            R = _rot(rng.uniform(0, 2 * math.pi))
        M = np.zeros((3, 4))
        M[:, :3] = R
        M[:, 3] = t
        out.append(M)
    return np.array(out, dtype=np.float32)


# 4x4 room-grid Hamiltonian cycle (adjacent rooms share a door, so straight segments between room
# centres pass through door centres)
_CYCLE = [(0, 0), (1, 0), (2, 0), (3, 0), (3, 1), (2, 1), (1, 1), (1, 2), (2, 2), (3, 2), (3, 3), (2, 3),
          (1, 3), (0, 3), (0, 2), (0, 1)]


def trajectory_rooms(n: int = 1000, seed: int = 4, z: float = 1.2) -> np.ndarray:
    """Closed loop through the room centres (C4): n poses equally spaced in arc length from a seeded
    start offset, yaw = direction of travel."""
    RX, RY = ROOM["RX"], ROOM["RY"]
    pts = np.array([((i + 0.5) * RX, (j + 0.5) * RY) for i, j in _CYCLE])
    seg = np.roll(pts, -1, axis=0) - pts
    L = np.linalg.norm(seg, axis=1)
    cum = np.concatenate([[0.0], np.cumsum(L)])
    rng = np.random.default_rng(seed)
    s0 = rng.uniform(0, cum[-1])
    out = []
    for k in range(n):
        s = (s0 + k * cum[-1] / n) % cum[-1]
        i = int(np.searchsorted(cum, s, side="right") - 1)
        f = (s - cum[i]) / L[i]
        p = pts[i] + f * seg[i]
        out.append(pose((p[0], p[1], z), yaw=math.atan2(seg[i][1], seg[i][0])))
    return np.stack(out)


def poses_terrain(terrain: Terrain, P: int, seed: int = 5, half: float = 400.0) -> np.ndarray:
    """C5: x, y ~ U[-half, half] (outside building footprints), z = terrain surface + 2 m, yaw ~ U[0, 2pi)."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < P:
        x, y = rng.uniform(-half, half, size=2)
        yaw = rng.uniform(0, 2 * math.pi)
        if terrain.inside_building(x, y):
            continue
        out.append(pose((x, y, float(terrain.surface_z(x, y)) + 2.0), yaw=yaw))
    return np.stack(out)


# ----------------------------------------------------------------------------------------------
# named configurations (BASELINE.json configs[0..4])
# ----------------------------------------------------------------------------------------------
def config(name: str, **kw):
    """Return dict(mesh=Mesh, pattern=Spinning|Rosette, poses=float32[P][3][4], ...)."""
    name = name.upper()
    if name == "C1":
        return dict(name="C1", mesh=scene_c1(), pattern=spinning_preset("VLP16"),
                    poses=pose((0.3, -0.2, 0.1), yaw=math.radians(17.0))[None])
    if name == "C2":
        P = kw.get("poses", 1)
        pat = spinning_preset("HDL64")
        t = (1.5 * ROOM["RX"], 1.5 * ROOM["RY"], 1.5)
        return dict(name="C2", mesh=scene_rooms(2), pattern=pat,
                    poses=poses_yaw_offsets(t, P, 2 * math.pi / pat.columns / max(P, 1)))
    if name == "C3":
        ter = scene_terrain(3)
        return dict(name="C3", mesh=ter.mesh, terrain=ter, pattern=spinning_preset("OS128"),
                    poses=pose((0.0, 0.0, float(ter.surface_z(0.0, 0.0)) + 2.0))[None])
    if name == "C4":
        return dict(name="C4", mesh=scene_rooms(2), pattern=rosette_default(),
                    poses=trajectory_rooms(kw.get("poses", 1000), 4))
    if name == "C5":
        ter = scene_terrain(3)
        return dict(name="C5", mesh=ter.mesh, terrain=ter, pattern=spinning_preset("HDL64"),
                    poses=poses_terrain(ter, kw.get("poses", 4096), 5))
    raise KeyError(name)


# ----------------------------------------------------------------------------------------------
# 3DGS inputs for the voxelizer (§III-A, §IV-A)
# ----------------------------------------------------------------------------------------------
# A pretrained 3DGS asset is {(mu_i, q_i, s_i, sigma_i)}: centre, unit quaternion
# (w, x, y, z), per-axis scale (> 0) and opacity in (0, 1). No trained assets exist offline, so
# these are seeded stand-ins with the statistics of splats fitted to surfaces: flat discs aligned
# with the surface (two tangent scales of a few cm, one thin normal scale), log-normal sizes,
# opacities spread over (0.05, 1). How (q, s) become a covariance, a box or a density is each
# side's own business; this module only draws the parameters.
@dataclass
class Gaussians:
    mu: np.ndarray       # float32 [N][3]
    quat: np.ndarray     # float32 [N][4] (w, x, y, z), unit up to float32 rounding
    scale: np.ndarray    # float32 [N][3] > 0
    opacity: np.ndarray  # float32 [N] in (0, 1)
    meta: dict = field(default_factory=dict)

    @property
    def N(self) -> int:
        return int(self.mu.shape[0])


def _gs(mu, q, s, o, **meta) -> Gaussians:
    f = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    return Gaussians(f(mu), f(q), f(s), f(o), dict(meta))


def _unit_quats(rng, n):
    q = rng.normal(size=(n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def gaussians_random(N: int, seed: int = 11, extent: float = 4.0, scale_median: float = 0.08,
                     scale_sigma: float = 0.5) -> Gaussians:
    """N Gaussians with uniform centres in [0, extent]^3, uniformly random orientations,
    log-normal per-axis scales and opacities uniform in (0.05, 1)."""
    rng = np.random.default_rng(seed)
    mu = rng.uniform(0.0, extent, size=(N, 3))
    q = _unit_quats(rng, N)
    s = scale_median * np.exp(scale_sigma * rng.normal(size=(N, 3)))
    o = rng.uniform(0.05, 1.0, size=N)
    return _gs(mu, q, s, o, kind="random", seed=seed)


def _quat_z_to(n):
    """Unit quaternions (w, x, y, z) of the shortest rotation taking +z to the unit normals n."""
    w = 1.0 + n[:, 2]
    q = np.stack([w, -n[:, 1], n[:, 0], np.zeros_like(w)], axis=1)
    flip = w < 1e-6  # n = -z: rotate by pi about x
    q[flip] = (0.0, 1.0, 0.0, 0.0)
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _quat_mul(a, b):
    w1, x1, y1, z1 = a.T
    w2, x2, y2, z2 = b.T
    return np.stack([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2], axis=1)


def gaussians_on_mesh(mesh: Mesh, N: int, seed: int = 12, tangent_median: float = 0.03,
                      normal_scale: float = 0.004, sigma: float = 0.4) -> Gaussians:
    """N surface splats on `mesh`: triangles drawn by area, uniform points on them, the thin axis
    (local z) along the face normal with a random spin about it, log-normal tangent scales."""
    rng = np.random.default_rng(seed)
    v = mesh.verts.astype(np.float64)
    a, b, c = v[mesh.tris[:, 0]], v[mesh.tris[:, 1]], v[mesh.tris[:, 2]]
    cr = np.cross(b - a, c - a)
    area = 0.5 * np.linalg.norm(cr, axis=1)
    k = rng.choice(mesh.T, size=N, p=area / area.sum())
    r1, r2 = rng.uniform(size=N), rng.uniform(size=N)
    sq = np.sqrt(r1)
    mu = (1 - sq)[:, None] * a[k] + (sq * (1 - r2))[:, None] * b[k] + (sq * r2)[:, None] * c[k]
    n = cr[k] / np.linalg.norm(cr[k], axis=1, keepdims=True)
    spin = rng.uniform(0.0, 2 * np.pi, size=N)
    qs = np.stack([np.cos(spin / 2), 0 * spin, 0 * spin, np.sin(spin / 2)], axis=1)
    q = _quat_mul(_quat_z_to(n), qs)
    st = tangent_median * np.exp(sigma * rng.normal(size=(N, 2)))
    sn = normal_scale * np.exp(0.25 * rng.normal(size=(N, 1)))
    o = rng.uniform(0.05, 1.0, size=N)
    return _gs(mu, q, np.concatenate([st, sn], axis=1), o, kind="surface", seed=seed, mesh_T=mesh.T)


@dataclass
class Grid:
    """Voxel lattice: centre of voxel (i, j, k) = origin + (i + 1/2, j + 1/2, k + 1/2) h."""
    origin: tuple
    h: float
    dims: tuple  # (nx, ny, nz)

    @property
    def nvox(self) -> int:
        return int(self.dims[0]) * int(self.dims[1]) * int(self.dims[2])


def grid_for(g: Gaussians, cells: int = 512, pad: int = 1) -> Grid:
    """Grid over the centres' bounding box, `cells` voxels along its longest axis, padded by `pad`
    free voxels on every side (SPEC voxelizer defaults: extent / 512, one voxel of padding)."""
    lo = g.mu.min(axis=0).astype(np.float64)
    hi = g.mu.max(axis=0).astype(np.float64)
    h = float(np.float32((hi - lo).max() / cells))
    dims = tuple(int(np.ceil((hi[a] - lo[a]) / h)) + 2 * pad for a in range(3))
    origin = tuple(float(np.float32(lo[a] - pad * h)) for a in range(3))
    return Grid(origin, h, dims)


def gauss_config(name: str):
    """G1: 2 000 random Gaussians in a 4 m cube, 64^3 grid (oracle-sized). G2: 1 M surface splats
    (tangent scales ~3.5 cm, normal ~1.5 cm) on the C2 rooms mesh, 512 voxels along the longest
    axis (~4.7 cm voxels; the paper's scale: "millions of primitives")."""
    name = name.upper()
    if name == "G1":
        g = gaussians_random(2000, 11)
        return dict(name="G1", gauss=g, grid=grid_for(g, 62), kappa=3.0, theta=0.5, tile=8)
    if name == "G2":
        g = gaussians_on_mesh(scene_rooms(2), 1_000_000, 12, tangent_median=0.035, normal_scale=0.015)
        return dict(name="G2", gauss=g, grid=grid_for(g, 512), kappa=3.0, theta=0.5, tile=8)
    raise KeyError(name)
