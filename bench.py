#!/usr/bin/env python
"""Benchmark of the LiDAR first-return cast hot path (FGGS-LiDAR, arXiv 2509.17390 §IV-C) on B200.

One step = one pass of the whole hot path of SURVEY.md §8(a) over one batch of synthetic input:
  A1 mesh upload + validation (device-resident mesh -> scene copy), A2-A7 LBVH build (centroids,
  Morton codes, radix sort, Karras tree, refit, leaf-order records, nodes), A8-A11 cast of every
  beam of every pose in the batch (raygen, traversal, watertight test, range/tri_id write) and,
  for N > 1, A12 the NCCL all-gather of the results.
Default workload (BASELINE.json configs[1], SURVEY C2 throughput mode): procedural indoor rooms
(~1.0 M triangles), HDL64-style 64 x 2048 spinning pattern, 64 yaw-offset poses per GPU per step.

Prints ONE JSON line (rank 0). `--impl reference` times the CPU oracle (the reference arm for
this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["fgl", "reference"], default="fgl")
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5", "G1", "G2", "T1", "T2"],
                    help="C1-C5: LiDAR cast (the north star); G1/G2: Gaussian voxelizer (NEXT-2); "
                         "T1/T2: TSDF + Marching Cubes on the G1/G2 occupancy (NEXT-3)")
    ap.add_argument("--poses", type=int, default=None, help="poses per GPU per step")
    ap.add_argument("--mode", choices=["full", "cast", "refit"], default="full",
                    help="full = upload+build+cast per step (default); cast = cast only on a prebuilt scene")
    ap.add_argument("--leaf-size", type=int, default=0, help="0 = library default")
    ap.add_argument("--width", type=int, default=0, help="BVH node width 2 or 4 (0 = library default)")
    ap.add_argument("--morton-bits", type=int, default=0, help="b of Eq. 5 (0 = library default)")
    ap.add_argument("--quantized", type=int, default=0, help="width 4 only: 8-bit child boxes (node64q)")
    ap.add_argument("--restructure", type=int, default=0, help="treelet restructuring passes (NEXT-4, width 2)")
    ap.add_argument("--treelets", type=int, default=0, help="1: bottom-up 4-leaf treelets inside the build (width 2)")
    ap.add_argument("--morton-box", type=int, default=0, help="0 = cubic (R22, default), 1 = per-axis (Eq. 5)")
    ap.add_argument("--no-graph", action="store_true", help="launch the step eagerly instead of a CUDA graph")
    ap.add_argument("--gather", choices=["fused", "nccl", "none"], default="fused",
                    help="N > 1, A12: fused = the cast kernel stores every result into all ranks' buffers over "
                         "NVLink (CUDA IPC) with a device-side completion barrier; nccl = chunked all_gather on a "
                         "side stream; none = pure cast scaling")
    ap.add_argument("--gather-chunks", type=int, default=4, help="N > 1, --gather nccl: chunks")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="process group for barriers / timing reduction (gloo: functional N > 1 check on one GPU)")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-latency", action="store_true", help="skip the single-frame latency measurement")
    ap.add_argument("--latency-frames", type=int, default=1000, help="CUDA-graph replays of one frame")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU time of the oracle baseline")
    return ap.parse_args()


METRIC = "rays/sec (LiDAR first-return cast, full hot path per step)"
DEFAULT_POSES = {"C1": 1, "C2": 64, "C3": 1, "C4": 1000, "C5": 512}


def _workload(name: str, poses_per_rank: int, world: int, rank: int):
    import synth
    if name in ("C2",):
        cfg = synth.config("C2", poses=poses_per_rank * world)
    elif name == "C4":
        cfg = synth.config("C4", poses=poses_per_rank * world)
    elif name == "C5":
        cfg = synth.config("C5", poses=poses_per_rank * world)
    else:
        cfg = synth.config(name)
        cfg["poses"] = np.concatenate([cfg["poses"]] * (poses_per_rank * world))
    P = poses_per_rank
    cfg["poses_rank"] = cfg["poses"][rank * P:(rank + 1) * P]
    return cfg


def _describe(cfg, P, world):
    pat = cfg["pattern"]
    if hasattr(pat, "elev_deg"):
        pdesc = f"{pat.name} {pat.channels}x{pat.columns} spinning"
    else:
        pdesc = f"rosette {pat.points_per_frame} pts/frame"
    return f"{cfg['name']}: {cfg['mesh'].meta.get('kind')} {cfg['mesh'].T} tris, {pdesc}, {P} poses/GPU/step"


# ----------------------------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampler running during the timed region (clocks + throttle reasons)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        except Exception:
            rows = []
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for k, n in enumerate(names):
                if len(r) > 5 + k and r[5 + k].strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(rows), "reasons": sorted(reasons)}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# Algorithmic FP32 operations of the cast: a slab test of one box is 6 plane
# distances (1 FMA each) + 6 per-axis min/max + 6 entry/exit reductions + 1 compare = 19; a binary
# node tests 2 boxes. The watertight triangle test is 9 translations + 27 shear ops + 9 edge-function
# ops + 6 sign tests + 2 (det) + 3 (T) + 1 division + 3 interval/tie compares = 60.
OPS_NODE = 38
OPS_TRI = 60


def _alu_peak_tops():
    """Issue ceiling in lane operations: 148 SMs x 4 SMSPs x 32 lanes x max SM clock (unit counts and
    clock: B200_PROFILING.md). Each SMSP issues one warp instruction per cycle; the FMA pipe (FFMA,
    FMUL) and the ALU pipe (FMNMX, FSETP, LOP3, PRMT) each accept one every second cycle
    (B300_MICROARCH.md), so the two together sustain the issue rate and an FP32 min/max costs the
    same issue slot as an FFMA: for an issue-bound kernel this one number is the ALU roofline."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz = float(json.load(f).get("sm_max_mhz", 1965.0))
    except Exception:
        mhz = 1965.0
    return 148 * 128 * mhz * 1e6 / 1e12


def _l2_read_gbs(fgl, torch, dev, stream):
    """L2 read bandwidth measured in the run: libfgl's probe re-reads an L2-resident
    buffer (half the L2) with 128-bit L1-bypassing loads from every SM; best of 5 timed launches."""
    l2 = int(torch.cuda.get_device_properties(dev).L2_cache_size)
    buf = torch.zeros(max(1 << 20, l2 // 2) // 16 * 4, dtype=torch.float32, device=dev)
    sink = torch.zeros(1, dtype=torch.float32, device=dev)
    iters = 40
    with torch.cuda.stream(stream):
        for _ in range(3):
            fgl.l2_read_probe(buf, iters, sink)
        best = float("inf")
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fgl.l2_read_probe(buf, iters, sink)
            e1.record(stream)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
    return buf.numel() * 4 * iters / (best / 1000) / 1e9, l2


def _frame_latency(scene, pose1, pat, out, torch, stream, n):
    """Latency of ONE frame (one pose, every beam) on the built scene: the cast captured in a CUDA
    graph and replayed n times back to back, each replay bracketed by its own CUDA events on the
    launch stream (median and p99 over the n replays; L2 warm, as in a frame-by-frame simulation)."""
    o1 = dict(range=out["range"][:1], tri_id=out["tri_id"][:1])
    side = torch.cuda.Stream()
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        for _ in range(3):
            scene.cast(pose1, pat, out=o1)
    stream.wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        scene.cast(pose1, pat, out=o1)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for _ in range(20):
            g.replay()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for e0, e1 in ev:
            e0.record(stream)
            g.replay()
            e1.record(stream)
    torch.cuda.synchronize()
    us = sorted(e0.elapsed_time(e1) * 1000.0 for e0, e1 in ev)
    rays = int(o1["range"].numel())
    med = us[len(us) // 2]
    return {"frames": n, "rays_per_frame": rays, "median_us": med, "p99_us": us[min(n - 1, int(0.99 * n))],
            "frames_per_s": 1e6 / med, "rays_per_s": rays / (med * 1e-6),
            "note": "one pose per CUDA-graph replay (cast only, prebuilt scene), per-replay CUDA events"}


def _ncu_summary(config: str, kernel: str = "k_cast") -> dict:
    """The committed ncu summary of the dominant kernel for this config (profiles/ncu_summary.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f)[config][kernel]
    except Exception:
        return {}


def _ncu_traffic(config: str, kernel: str = "k_cast"):
    """dram read+write bytes per launch of the dominant kernel from the committed ncu summary."""
    return _ncu_summary(config, kernel).get("dram_bytes_per_launch")


# ----------------------------------------------------------------------------------------------
def _host_cpu():
    """CPU model, physical cores and hardware threads of this host (SURVEY 8(d) timing protocol)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        import psutil
        phys = psutil.cpu_count(logical=False)
    except Exception:
        phys = None
    return {"model": model, "physical_cores": phys, "threads": os.cpu_count(),
            "affinity": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None}


def _cpu_baseline(cfg, seconds: float, gpu_range=None, gpu_tri=None, parity_rays: int = 2048):
    """The oracle (CPU double brute force, Eq. 20 by the naive scan P:291-294), as it stands, on a
    bounded seeded sample of the workload's rays, on this host's cores; plus its 1-thread rate on a
    1/64 subset of that sample, and — when the GPU's results for pose 0 are given — the parity of
    this bench run: the oracle classifies `parity_rays` of the sampled rays (mode A: its own double
    rays) and judges the GPU's range / tri_id on them."""
    import oracle
    m, pat = cfg["mesh"], cfg["pattern"]
    o, d = oracle.pattern_rays(pat, cfg["poses_rank"][:1])
    rng = np.random.default_rng(0)
    probe = 64
    idx = rng.choice(o.shape[0], probe, replace=False)
    t0 = time.perf_counter()
    oracle.cast(m.verts, m.tris, o[idx], d[idx], pat.t_min, pat.t_max)
    dt = max(time.perf_counter() - t0, 1e-6)
    n = int(min(o.shape[0], max(probe, probe * seconds / dt)))
    idx = rng.choice(o.shape[0], n, replace=False)
    t0 = time.perf_counter()
    oracle.cast(m.verts, m.tris, o[idx], d[idx], pat.t_min, pat.t_max)
    dt = time.perf_counter() - t0
    threads = oracle.threads()
    # 1-thread rate on a 1/64 subset (per-core speed; the multi-thread rate / cores shows the scaling)
    sub = idx[: max(1, n // 64)]
    oracle.set_threads(1)
    try:
        t1 = time.perf_counter()
        oracle.cast(m.verts, m.tris, o[sub], d[sub], pat.t_min, pat.t_max)
        dt1 = time.perf_counter() - t1
    finally:
        oracle.set_threads(threads)
    out = {"value": n / dt, "unit": "rays/s", "cores": threads, "kind": "oracle",
           "sample": f"{n} seeded rays of pose 0 of {cfg['name']} vs all {m.T} triangles "
                     f"({n * m.T:.3g} double MT tests, {dt:.1f} s)",
           "one_thread_rays_per_s": len(sub) / dt1, "one_thread_sample": f"{len(sub)} rays (1/64 of the sample)",
           "host": _host_cpu()}
    parity = None
    if gpu_range is not None:
        pidx = np.sort(idx[:parity_rays])
        v = oracle.cast_and_classify(m.verts, m.tris, o[pidx], d[pidx], pat.t_min, pat.t_max,
                                     eps_rel=oracle.EPS_MODE_A)
        j = oracle.judge(v, gpu_range[pidx], gpu_tri[pidx])
        parity = {"rays": int(j["n"]), "mode": "A (oracle's own double rays vs the bench's cast of pose 0)",
                  "ambiguous": int(j["ambiguous"]), "unambiguous_mismatch": int(len(j["unamb_mismatch"])),
                  "ambiguous_outside": int(len(j["amb_outside"])),
                  "tolerance": "unambiguous rays: tri_id exact, |range - t*| <= 1e-4 t* + 1e-5 m (DESIGN.md §4)"}
    return out, parity


def run_reference(a):
    """--impl reference: the oracle on the host cores, each step a bounded sample of the workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    P = a.poses or DEFAULT_POSES[a.config]
    cfg = _workload(a.config, P, 1, 0)
    m, pat = cfg["mesh"], cfg["pattern"]
    o, d = oracle.pattern_rays(pat, cfg["poses_rank"][:1])
    rng = np.random.default_rng(1)
    # size each step to ~1.5 s of CPU work so W + K steps finish in a few minutes
    t0 = time.perf_counter()
    oracle.cast(m.verts, m.tris, o[:64], d[:64], pat.t_min, pat.t_max)
    per_ray = (time.perf_counter() - t0) / 64
    n = int(max(8, min(o.shape[0], 1.5 / max(per_ray, 1e-9))))
    for _ in range(a.warmup):
        idx = rng.choice(o.shape[0], n, replace=False)
        oracle.cast(m.verts, m.tris, o[idx], d[idx], pat.t_min, pat.t_max)
    times = []
    for _ in range(a.steps):
        idx = rng.choice(o.shape[0], n, replace=False)
        t0 = time.perf_counter()
        oracle.cast(m.verts, m.tris, o[idx], d[idx], pat.t_min, pat.t_max)
        times.append(time.perf_counter() - t0)
    ms = 1000 * statistics.mean(times)
    v = n / (ms / 1000)
    line = {"metric": METRIC, "value": v, "unit": "rays/s", "n_gpus": 0,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": _describe(cfg, P, 1), "sample_rays_per_step": n, "triangles": m.T},
            "cpu_baseline": {"value": v, "unit": "rays/s", "cores": oracle.threads(), "kind": "oracle",
                             "sample": f"{n} seeded rays per step of {a.config} pose 0 vs all {m.T} triangles",
                             "host": _host_cpu()},
            "e2e": {"value": v, "unit": "rays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------------------------
# NEXT-2: Gaussian -> occupancy (§IV-A Eqs. 4-12). One step = async upload of the 3DGS
# parameters + LBVH build over the Eq. 4 boxes + tiled voxelization (Eqs. 8-10) + masks (11-12).
VOX_METRIC = "voxels/sec (3DGS voxelization: Eq. 4 boxes + LBVH + Eqs. 8-12 per step)"
# algorithmic FP32 ops per (voxel, candidate) pair: d = v - mu (3), d^T A d in Horner form (6 FMA +
# 3 MUL), the kappa test (1), exp2 (1), the weighted accumulation (1 FMA) = 15
OPS_PAIR = 15


def _vox_oracle(cfg, seconds: float, seed: int = 0):
    """The oracle's Eq. 9 (density_at) on a bounded seeded sample of grid voxels."""
    from oracle import gauss as og
    g, grid = cfg["gauss"], cfg["grid"]
    nx, ny, nz = grid.dims
    rng = np.random.default_rng(seed)

    def pts(n):
        idx = rng.integers(0, grid.nvox, n)
        k, rem = np.divmod(idx, nx * ny)
        j, i = np.divmod(rem, nx)
        o = np.asarray(grid.origin)
        return np.stack([o[0] + (i + 0.5) * grid.h, o[1] + (j + 0.5) * grid.h, o[2] + (k + 0.5) * grid.h], axis=1)

    t0 = time.perf_counter()
    og.density_at(g, pts(8), cfg["kappa"])
    per = (time.perf_counter() - t0) / 8
    n = int(max(8, seconds / max(per, 1e-9)))
    return n, pts, per


def run_voxel(a):
    import synth
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    cfg = synth.gauss_config(a.config)
    g, grid, kappa, theta = cfg["gauss"], cfg["grid"], cfg["kappa"], cfg["theta"]
    wl = (f"{cfg['name']}: {g.meta.get('kind')} 3DGS cloud N={g.N}, grid {grid.dims[0]}x{grid.dims[1]}x"
          f"{grid.dims[2]} (h={grid.h:.4f} m), kappa={kappa}, theta={theta}, tile 8^3")
    if a.impl == "reference":
        if rank != 0:
            return 0
        from oracle import gauss as og
        n, pts, _ = _vox_oracle(cfg, 1.5)
        for _ in range(a.warmup):
            og.density_at(g, pts(n), kappa)
        times = []
        for _ in range(a.steps):
            p = pts(n)
            t0 = time.perf_counter()
            og.density_at(g, p, kappa)
            times.append(time.perf_counter() - t0)
        ms = 1000 * statistics.mean(times)
        v = n / (ms / 1000)
        print(json.dumps({"metric": VOX_METRIC, "value": v, "unit": "voxels/s", "n_gpus": 0, "steps": a.steps,
                          "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                          "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
                          "config": {"workload": wl, "sample_voxels_per_step": n},
                          "cpu_baseline": {"value": v, "unit": "voxels/s", "cores": 1, "kind": "oracle",
                                           "sample": f"{n} seeded voxels per step, Eq. 9 over all {g.N} Gaussians"},
                          "e2e": {"value": v, "unit": "voxels/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return 0
    import torch
    import torch.distributed as dist

    import paper_2509_17390_b200 as fgl
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl" if a.dist_backend == "nccl" else "gloo", device_id=dev
                                if a.dist_backend == "nccl" else None)
    # replicas only: each rank voxelizes its own copy of the cloud (the grid is one
    # problem per scene; independent scenes shard across ranks with no exchange)
    arrs = [torch.from_numpy(x).to(dev) for x in (g.mu, g.quat, g.scale, g.opacity)]
    gs = fgl.GaussianScene(*arrs, kappa=kappa, device=dev)
    stream = torch.cuda.current_stream()
    nx, ny, nz = grid.dims
    nw = (nx + 31) // 32
    out = dict(occupancy=torch.empty((nz, ny, nw), dtype=torch.int32, device=dev),
               surface=torch.empty((nz, ny, nw), dtype=torch.int32, device=dev),
               interior=torch.empty((nz, ny, nw), dtype=torch.int32, device=dev),
               counts=torch.empty(4, dtype=torch.int64, device=dev))
    vev = None

    def step():
        gs.upload(*arrs, sync=False)
        gs.build()
        if vev is not None:
            vev[0].record(stream)
        gs.voxelize(grid.origin, grid.h, grid.dims, theta, out=out)
        if vev is not None:
            vev[1].record(stream)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    graph = None
    if not a.no_graph:
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            step()
        stream.wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        torch.cuda.synchronize()
        for _ in range(a.warmup):
            graph.replay()
    flush = None if a.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    K = a.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for i in range(K):
            if flush is not None:
                flush.zero_()
            ev[i][0].record(stream)
            graph.replay() if graph is not None else step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    gs.check()
    ms = statistics.mean(e[0].elapsed_time(e[1]) for e in ev)
    l0 = fgl.kernel_launches()
    step()
    launches = (fgl.kernel_launches() - l0) * K
    # voxelize alone (events on the launch stream) for the roofline
    vms = []
    for _ in range(max(5, K)):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        gs.voxelize(grid.origin, grid.h, grid.dims, theta, out=out)
        e1.record(stream)
        torch.cuda.synchronize()
        vms.append(e0.elapsed_time(e1))
    vms = statistics.mean(vms)
    if world > 1:
        t = torch.tensor([ms, vms], dtype=torch.float64, device=dev)
        t = t.cpu() if a.dist_backend == "gloo" else t
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, vms = t.tolist()
    c = out["counts"].cpu().tolist()
    pairs = c[2]
    alu_peak = _alu_peak_tops()
    achieved = OPS_PAIR * pairs / (vms / 1000) / 1e12
    # e2e: host (pinned) parameters in, occupancy bits + counts out, through the public API
    e2e = None
    if not a.no_e2e:
        host = [torch.from_numpy(x).pin_memory() for x in (g.mu, g.quat, g.scale, g.opacity)]
        occ_h = torch.empty((nz, ny, nw), dtype=torch.int32).pin_memory()
        gs2 = fgl.GaussianScene(*host, kappa=kappa, device=dev)
        res = {}

        def e2e_step():
            gs2.upload(*host, sync=False)
            gs2.build()
            r = gs2.voxelize(grid.origin, grid.h, grid.dims, theta, masks=True, out=res)
            res.update(r)
            occ_h.copy_(r["occupancy"], non_blocking=True)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        ee = []
        for _ in range(max(3, K // 2)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            e2e_step()
            e1.record(stream)
            torch.cuda.synchronize()
            ee.append(e0.elapsed_time(e1))
        ems = statistics.mean(ee)
        e2e = {"value": grid.nvox * world / (ems / 1000), "unit": "voxels/s",
               "h2d_bytes_per_step": int(sum(x.numel() * 4 for x in host)),
               "d2h_bytes_per_step": int(occ_h.numel() * 4), "ms_per_step": ems}
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        from oracle import gauss as og
        n, pts, _ = _vox_oracle(cfg, a.cpu_seconds)
        p = pts(n)
        t0 = time.perf_counter()
        og.density_at(g, p, kappa)
        dt = time.perf_counter() - t0
        cpu = {"value": n / dt, "unit": "voxels/s", "cores": 1, "kind": "oracle",
               "sample": f"{n} seeded voxels of {cfg['name']}, Eq. 9 over all {g.N} Gaussians (numpy, {dt:.1f} s)"}
    if rank == 0:
        st = gs.stats()
        print(json.dumps({
            "metric": VOX_METRIC, "value": grid.nvox * world / (ms / 1000), "unit": "voxels/s", "n_gpus": world,
            "steps": K, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": wl, "step": "upload+build+voxelize+masks", "voxels": grid.nvox,
                       "gaussians": g.N, "parallelism": f"replicas x{world}",
                       "l2": "flushed between steps (256 MiB memset, untimed)" if flush is not None else "not flushed",
                       "launch": "one CUDA graph replay per step" if graph is not None else "eager launches"},
            "gaussians_per_s": g.N * world / (ms / 1000), "build_ms": st["build_ms"], "voxelize_ms": vms,
            "occupied": c[0], "surface": c[1], "pairs": pairs,
            "roofline": {"bound": "alu", "achieved": achieved, "peak": alu_peak, "unit": "TFLOP/s",
                         "frac": achieved / alu_peak, "traffic": _ncu_traffic(a.config, "k_voxelize"),
                         "kernel": "k_voxelize",
                         "note": f"{OPS_PAIR} algorithmic FP32 ops per (voxel, candidate) pair x {pairs} pairs / "
                                 f"voxelize time (k_voxelize + k_masks, CUDA events); peak = 148 SM x 128 lanes x "
                                 f"max SM clock"},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary()}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# NEXT-3: occupancy -> mesh (§IV-B Eqs. 13-18). One step = denoise (Eqs. 13-14a) + narrow-
# band TSDF (Eqs. 15-17) + Marching Cubes (Eq. 18) of the G config's occupancy volume.
MESH_METRIC = "voxels/sec (occupancy -> mesh: denoise + narrow-band TSDF + Marching Cubes per step)"
TSDF_SIGMA_VOX, TSDF_TAU, TSDF_BAND_VOX = 0.7, 0.35, 3


def run_mesh(a):
    import synth
    rank = int(os.environ.get("RANK", "0"))
    gname = "G" + a.config[1:]
    cfg = synth.gauss_config(gname)
    g, grid, kappa, theta = cfg["gauss"], cfg["grid"], cfg["kappa"], cfg["theta"]
    h = grid.h
    sp = (h, h, h)
    nx, ny, nz = grid.dims
    wl = (f"{a.config}: occupancy of {gname} ({g.N} Gaussians, grid {nx}x{ny}x{nz}, h={h:.4f} m) -> denoise "
          f"(sigma {TSDF_SIGMA_VOX} voxels, tau {TSDF_TAU}) -> TSDF (r = {TSDF_BAND_VOX} voxels) -> MC at iso 0")
    if a.impl == "reference":
        if rank != 0:
            return 0
        # the oracle on a bounded sub-block of the same occupancy (its TSDF + MC are numpy loops)
        from oracle import gauss as og
        from oracle import tsdf as ot
        sub = synth.Grid(grid.origin, h, (min(nx, 48), min(ny, 48), min(nz, 32)))
        D, _, _ = og.density(synth.Gaussians(g.mu, g.quat, g.scale, g.opacity), sub, kappa) if g.N <= 5000 else \
            (None, None, None)
        if D is None:
            pts_ok = np.all((g.mu >= np.asarray(sub.origin) - 0.5) &
                            (g.mu <= np.asarray(sub.origin) + np.asarray(sub.dims) * h + 0.5), axis=1)
            gg = synth.Gaussians(g.mu[pts_ok], g.quat[pts_ok], g.scale[pts_ok], g.opacity[pts_ok])
            D, _, _ = og.density(gg, sub, kappa)
        V = og.occupancy(D, theta)

        def once():
            Vd = ot.rethreshold(ot.blur(V, TSDF_SIGMA_VOX * h, sp), TSDF_TAU)
            phi, _ = ot.tsdf(Vd, sp, TSDF_BAND_VOX * h)
            ot.marching_cubes(phi, sub.origin, sp)

        for _ in range(a.warmup):
            once()
        times = []
        for _ in range(a.steps):
            t0 = time.perf_counter()
            once()
            times.append(time.perf_counter() - t0)
        ms = 1000 * statistics.mean(times)
        v = sub.nvox / (ms / 1000)
        print(json.dumps({"metric": MESH_METRIC, "value": v, "unit": "voxels/s", "n_gpus": 0, "steps": a.steps,
                          "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                          "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
                          "config": {"workload": wl, "sample_voxels_per_step": sub.nvox},
                          "cpu_baseline": {"value": v, "unit": "voxels/s", "cores": 1, "kind": "oracle",
                                           "sample": f"a {sub.dims} sub-block of the occupancy per step"},
                          "e2e": {"value": v, "unit": "voxels/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return 0
    import torch

    import paper_2509_17390_b200 as fgl
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    arrs = [torch.from_numpy(x).to(dev) for x in (g.mu, g.quat, g.scale, g.opacity)]
    gs = fgl.GaussianScene(*arrs, kappa=kappa, device=dev)
    occ = gs.voxelize(grid.origin, h, grid.dims, theta, masks=False)["occupancy"]
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    first = fgl.marching_cubes(fgl.tsdf(fgl.denoise(occ, grid.dims, sp, TSDF_SIGMA_VOX * h, TSDF_TAU), grid.dims, sp,
                                        TSDF_BAND_VOX * h), grid.origin, sp)
    nv, nt = first["verts"].shape[0], first["tris"].shape[0]
    mesh_out = dict(verts=torch.empty((nv, 3), dtype=torch.float32, device=dev),
                    tris=torch.empty((nt, 3), dtype=torch.int32, device=dev),
                    counts=torch.zeros(2, dtype=torch.int64, device=dev))
    den = torch.empty_like(occ)
    phi = torch.empty((nz, ny, nx), dtype=torch.float32, device=dev)

    def step():
        fgl.denoise(occ, grid.dims, sp, TSDF_SIGMA_VOX * h, TSDF_TAU, out=den)
        fgl.tsdf(den, grid.dims, sp, TSDF_BAND_VOX * h, out=phi)
        fgl.marching_cubes(phi, grid.origin, sp, out=mesh_out)

    l_a = fgl.kernel_launches()
    step()
    per_step_launches = fgl.kernel_launches() - l_a  # libfgl kernels per step (a graph replay runs them)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    graph = None
    if not a.no_graph:
        # the step's ~20 launches as one CUDA graph (scratch is stream-ordered, sizes are fixed after
        # the first call): eager launches leave the timed region exposed to host-side jitter
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            step()
        stream.wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        torch.cuda.synchronize()
        for _ in range(a.warmup):
            graph.replay()
        torch.cuda.synchronize()
    flush = None if a.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    K = a.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    l0 = fgl.kernel_launches()
    with Clocks(local) as clk:
        for i in range(K):
            if flush is not None:
                flush.zero_()
            ev[i][0].record(stream)
            if graph is not None:
                graph.replay()
            else:
                step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    launches = (fgl.kernel_launches() - l0) if graph is None else per_step_launches * K
    ms = statistics.mean(e[0].elapsed_time(e[1]) for e in ev)
    c = mesh_out["counts"].cpu().tolist()
    e2e = None
    if not a.no_e2e:  # host occupancy bits in, mesh (verts + tris) out
        occ_h = occ.cpu().pin_memory()
        vh = torch.empty((nv, 3), dtype=torch.float32).pin_memory()
        th = torch.empty((nt, 3), dtype=torch.int32).pin_memory()
        ee = []
        for _ in range(max(3, K // 2)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            occ.copy_(occ_h, non_blocking=True)
            step()
            vh.copy_(mesh_out["verts"], non_blocking=True)
            th.copy_(mesh_out["tris"], non_blocking=True)
            e1.record(stream)
            torch.cuda.synchronize()
            ee.append(e0.elapsed_time(e1))
        ems = statistics.mean(ee)
        e2e = {"value": grid.nvox / (ems / 1000), "unit": "voxels/s", "h2d_bytes_per_step": int(occ_h.numel() * 4),
               "d2h_bytes_per_step": int(vh.numel() * 4 + th.numel() * 4), "ms_per_step": ems}
    # HBM roofline: the kernels stream the volume; algorithmic bytes per voxel = denoise (1/8 B in,
    # 3 passes x 8 B float r/w, 4 B V', 1/8 B out) + TSDF (union-find 4 B label x ~3 r/w, kappa 1 B x
    # (band + 2), phi 4 B) + MC (phi 4 B x 2 reads, 3 x 4 B counts r/w x 3 passes) ~= 100 B
    bytes_per_voxel = 100.0
    hbm_peak, peak_kind = _peaks()
    achieved = bytes_per_voxel * grid.nvox / (ms / 1000) / 1e9
    if rank == 0:
        print(json.dumps({
            "metric": MESH_METRIC, "value": grid.nvox / (ms / 1000), "unit": "voxels/s", "n_gpus": 1, "steps": K,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": wl, "step": "denoise+tsdf+marching_cubes", "voxels": grid.nvox,
                       "parallelism": "replicas x1",
                       "l2": "flushed between steps (256 MiB memset, untimed)" if flush is not None else "not flushed",
                       "launch": "one CUDA graph replay per step" if graph is not None else "eager launches"},
            "mesh_vertices": c[0], "mesh_triangles": c[1],
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": None, "kernel": "denoise+tsdf+mc (all)",
                         "note": f"~{bytes_per_voxel:.0f} algorithmic bytes per voxel over the whole step "
                                 f"(DESIGN.md §8d); peak {peak_kind}"},
            "cpu_baseline": None, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary()}), flush=True)
    return 0


def main():
    a = _args()
    if a.config.startswith("G"):
        return run_voxel(a)
    if a.config.startswith("T"):
        return run_mesh(a)
    if a.impl == "reference":
        return run_reference(a)
    import torch
    import torch.distributed as dist

    import paper_2509_17390_b200 as fgl

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.gpus != world and world > 1:
        print(f"warning: --gpus {a.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    # --dist-backend gloo + more ranks than GPUs: a functional check of the N > 1 path on one GPU
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if a.dist_backend == "nccl":
            # communicator set-up lines (rank count, transport) in the log, for the record
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    P = a.poses or DEFAULT_POSES[a.config]
    cfg = _workload(a.config, P, world, rank)
    m, pat = cfg["mesh"], cfg["pattern"]
    rays_per_pose = fgl.rays_per_pose(pat)
    rays_rank = P * rays_per_pose
    verts_d = torch.from_numpy(m.verts).to(dev)
    tris_d = torch.from_numpy(m.tris).to(dev)
    poses_d = torch.from_numpy(np.ascontiguousarray(cfg["poses_rank"])).to(dev)
    stream = torch.cuda.current_stream()
    scene = fgl.Scene(verts_d, tris_d, device=dev, leaf_size=a.leaf_size, morton_box=a.morton_box, width=a.width,
                      morton_bits=a.morton_bits, quantized=a.quantized, restructure=a.restructure, treelets=a.treelets)
    out = scene.cast(poses_d, pat)
    shape = tuple(out["range"].shape)
    gather = None
    peer = None
    chunks = max(1, min(a.gather_chunks, P))
    gather_mode = a.gather
    if world > 1 and gather_mode == "fused" and not hasattr(pat, "elev_deg"):
        gather_mode = "nccl"  # the fused kernel path covers spinning patterns
    if world > 1 and gather_mode == "fused":
        from paper_2509_17390_b200 import dist as fdist
        cpu_group = dist.new_group(backend="gloo")
        peer = fdist.PeerGather(P * world, pat, dev, cpu_group=cpu_group)
        poses_all_d = torch.from_numpy(np.ascontiguousarray(cfg["poses"])).to(dev)
    if world > 1 and gather_mode == "nccl":
        assert P % chunks == 0, "--poses must be a multiple of --gather-chunks"
        Pc = P // chunks
        # chunk-major gathered layout: g[c][r] = rank r's poses [c*Pc, (c+1)*Pc)
        g_rng = torch.empty((chunks, world, Pc) + shape[1:], dtype=torch.float32, device=dev)
        g_tid = torch.empty((chunks, world, Pc) + shape[1:], dtype=torch.int32, device=dev)
        gather = (g_rng, g_tid, Pc)
        comm = torch.cuda.Stream(device=dev)
    flush = None if a.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step(cast_ev=None):
        if a.mode == "full":
            scene.upload(verts_d, tris_d, sync=False)  # A1 (D2D copy + validation, checked after the run)
            scene.build()                        # A2-A7
        elif a.mode == "refit":
            scene.refit(verts_d, sync=False)     # NEXT-4: new positions, boxes + nodes refitted, tree kept
        if cast_ev:
            cast_ev[0].record(stream)
        if peer is not None:
            peer.cast(scene, poses_all_d)        # A8-A12 fused: results stored into every rank's buffer
            peer.wait()                          # device-side barrier: all ranks' stores have landed
        elif gather is None:
            scene.cast(poses_d, pat, out=out)    # A8-A11
        else:
            # A8-A11 chunk by chunk; A12 all-gather of chunk c (NCCL, side stream) overlaps the cast of c+1
            Pc = gather[2]
            works = []
            for c in range(chunks):
                sl = slice(c * Pc, (c + 1) * Pc)
                scene.cast(poses_d[sl], pat, out=dict(range=out["range"][sl], tri_id=out["tri_id"][sl]))
                comm.wait_stream(stream)
                with torch.cuda.stream(comm):
                    # output viewed flat along its first dim ([world * Pc][...]): the form every backend takes
                    works.append(dist.all_gather_into_tensor(gather[0][c].view((world * Pc,) + shape[1:]),
                                                             out["range"][sl], async_op=True))
                    works.append(dist.all_gather_into_tensor(gather[1][c].view((world * Pc,) + shape[1:]),
                                                             out["tri_id"][sl], async_op=True))
            for w in works:
                w.wait()
            stream.wait_stream(comm)
        if cast_ev:
            cast_ev[1].record(stream)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    use_graph = not a.no_graph and world == 1
    graph = None
    if use_graph:
        # the whole step (upload copies, ~20 build kernels, the cast) as one CUDA graph
        gev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            step()
        torch.cuda.current_stream().wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        torch.cuda.synchronize()
        for _ in range(a.warmup):
            graph.replay()
        torch.cuda.synchronize()
    K = a.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    cev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = fgl.kernel_launches()
    with Clocks(local) as clk:
        for i in range(K):
            if flush is not None:
                flush.zero_()                    # evict L2 between timed steps (not timed)
            ev[i][0].record(stream)
            if graph is not None:
                graph.replay()
            else:
                step(cev[i])
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = fgl.kernel_launches() - launches0
    scene.check()  # validation result of the (asynchronous) uploads
    step_ms = [e[0].elapsed_time(e[1]) for e in ev]
    if peer is not None:
        peer.sync()
    if graph is not None:
        # graph replays launch the same kernels as the eager step: count them from one eager step,
        # and time the cast part with events on eager casts of the same inputs
        l0 = fgl.kernel_launches()
        step()
        launches = (fgl.kernel_launches() - l0) * K
        for i in range(K):
            if flush is not None:
                flush.zero_()
            cev[i][0].record(stream)
            scene.cast(poses_d, pat, out=out)
            cev[i][1].record(stream)
        torch.cuda.synchronize()
    cast_ms = [e[0].elapsed_time(e[1]) for e in cev]
    ms = statistics.mean(step_ms)
    cms = statistics.mean(cast_ms)
    if world > 1:
        t = torch.tensor([ms, cms], dtype=torch.float64, device=dev)
        t = t.cpu() if a.dist_backend == "gloo" else t
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, cms = t.tolist()
    clocks = clk.summary()

    # --- W = N vs W = 1: the gathered results equal, bit for bit, one GPU casting every pose --------
    gather_check = None
    if world > 1 and (peer is not None or gather is not None):
        if peer is not None:
            peer.sync()
            g_r, g_t = peer.range, peer.tri_id
        else:
            torch.cuda.synchronize()
            # chunk-major gathered layout g[c][r][j] = pose r * P + c * Pc + j
            g_r = gather[0].transpose(0, 1).reshape((world * P,) + shape[1:])
            g_t = gather[1].transpose(0, 1).reshape((world * P,) + shape[1:])
        if rank == 0:
            poses_all = torch.from_numpy(np.ascontiguousarray(cfg["poses"])).to(dev)
            ref = scene.cast(poses_all, pat)
            torch.cuda.synchronize()
            eq = bool(torch.equal(ref["tri_id"], g_t)) and bool(
                torch.equal(ref["range"].view(torch.int32), g_r.view(torch.int32)))
            gather_check = {"equal": eq, "poses": int(world * P), "mode": "fused P2P" if peer is not None else "nccl",
                            "note": "rank 0's single-GPU cast of all W x P poses vs the gathered result, bitwise"}
        if world > 1:
            dist.barrier()

    # --- Eq. 21 counters on the same rays (COUNT variant, untimed) -> algorithmic bytes ------
    cres = scene.cast(poses_d, pat, counts=True)
    n_nodes = cres["node_counts"].double().mean().item()
    n_tris = cres["tri_counts"].double().mean().item()
    node_bytes = 96.0 if a.width == 8 else (128.0 if a.width == 4 and not a.quantized else 64.0)
    bytes_per_ray = node_bytes * n_nodes + 48.0 * n_tris + 8.0
    hbm_peak, peak_kind = _peaks()
    # a visit tests every child box of the node: 2 (width 2), 4 (width 4), or 8 quantised boxes whose
    # 6 planes are decoded first (width 8: 6 decodes + 19 per box)
    ops_node = {8: 8 * 25, 4: 4 * (19 + (6 if a.quantized else 0))}.get(a.width, OPS_NODE)
    ops_per_ray = ops_node * n_nodes + OPS_TRI * n_tris
    alu_peak = _alu_peak_tops()
    achieved = ops_per_ray * rays_rank / (cms / 1000) / 1e12
    ncu = _ncu_summary(a.config)
    traffic = ncu.get("dram_bytes_per_launch")

    # --- single-frame latency: one pose cast per CUDA-graph replay ------------------
    latency = None
    if rank == 0 and not a.no_latency:
        latency = _frame_latency(scene, poses_d[:1].contiguous(), pat, out, torch, stream, a.latency_frames)

    # --- e2e through the public API with host buffers --------------------------------------
    # Every step copies its inputs (mesh + poses) from pinned host memory, builds, casts, and reads
    # its results back to pinned host memory. Steps are pipelined over three scenes: the upload of
    # step i+1 (H2D copy engine) and the read-back of step i (D2H copy engine, one copy per output
    # after the whole cast) overlap the build and cast of the neighbouring steps on the SMs. Measured
    # (tools/e2e_probe.py): 2 scenes / 8 read-back chunks 1.74 ms per step, 3 scenes / 1 chunk 1.57 ms
    # (chunking the cast into 8 launches costs more than the overlap it buys); the PCIe bound is the
    # 67 MB read-back at 57 GB/s, 1.18 ms (tools/pcie_bw.py).
    e2e = None
    if not a.no_e2e:
        vh = torch.from_numpy(m.verts).pin_memory()
        th = torch.from_numpy(m.tris).pin_memory()
        ph = torch.from_numpy(np.ascontiguousarray(cfg["poses_rank"])).pin_memory()
        NS = 3
        rh = [torch.empty(shape, dtype=torch.float32).pin_memory() for _ in range(NS)]
        ih = [torch.empty(shape, dtype=torch.int32).pin_memory() for _ in range(NS)]
        pds = [torch.empty_like(poses_d) for _ in range(NS)]
        scs = [fgl.Scene(device=dev, leaf_size=a.leaf_size, morton_box=a.morton_box, width=a.width,
                         morton_bits=a.morton_bits, quantized=a.quantized, restructure=a.restructure, treelets=a.treelets)
               for _ in range(NS)]
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        scratch = [dict(range=torch.empty(shape, dtype=torch.float32, device=dev),
                        tri_id=torch.empty(shape, dtype=torch.int32, device=dev)) for _ in range(NS)]
        done = [None] * NS

        def e2e_steps(n):
            for i in range(n):
                S = i % NS
                if done[S] is not None:
                    s_in.wait_event(done[S])  # scene S's previous read-back has finished
                if i == 0:
                    s_in.wait_stream(stream)
                scs[S].upload(vh, th, sync=False, stream=s_in)  # H2D mesh (pinned) + validation
                with torch.cuda.stream(s_in):
                    pds[S].copy_(ph, non_blocking=True)          # H2D poses
                up = torch.cuda.Event()
                up.record(s_in)
                stream.wait_event(up)
                scs[S].build()
                done[S] = scs[S].cast_to_host(pds[S], pat, rh[S], ih[S], chunks=1, copy_stream=s_out,
                                              scratch=scratch[S], wait=False)
            for ev_ in done:
                if ev_ is not None:
                    stream.wait_event(ev_)

        e2e_steps(max(2, a.warmup))
        torch.cuda.synchronize()
        ke = max(4, K)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if flush is not None:
            flush.zero_()
        e0.record(stream)
        e2e_steps(ke)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / ke
        for sc_ in scs:
            sc_.check()
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            t = t.cpu() if a.dist_backend == "gloo" else t
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = t.item()
        e2e = {"value": rays_rank * world / (ems / 1000), "unit": "rays/s",
               "h2d_bytes_per_step": int(m.verts.nbytes + m.tris.nbytes + cfg["poses_rank"].nbytes),
               "d2h_bytes_per_step": int(rh[0].numel() * 4 + ih[0].numel() * 4), "ms_per_step": ems,
               "note": "pinned host in/out every step; steps pipelined over three scenes (H2D of step i+1 and "
                       "D2H of step i overlap the build/cast on the SMs); PCIe bound: the D2H at ~57 GB/s"}
        del scs

    cpu = None
    parity = None
    if rank == 0 and world == 1 and not a.no_cpu:
        # the bench's own results for pose 0 (the step's last cast) are judged by the oracle
        scene.cast(poses_d[:1], pat, out=dict(range=out["range"][:1], tri_id=out["tri_id"][:1]))
        torch.cuda.synchronize()
        g_rng = out["range"][0].reshape(-1).cpu().numpy()
        g_tid = out["tri_id"][0].reshape(-1).cpu().numpy()
        cpu, parity = _cpu_baseline(cfg, a.cpu_seconds, g_rng, g_tid)

    l2_gbs, l2_bytes = (None, None)
    if rank == 0:
        l2_gbs, l2_bytes = _l2_read_gbs(fgl, torch, dev, stream)  # after the launch count and timings

    if rank == 0:
        st = scene.stats()
        total_rays = rays_rank * world
        line = {
            "metric": METRIC,
            "value": total_rays / (ms / 1000), "unit": "rays/s", "n_gpus": world, "steps": K, "warmup": a.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": _describe(cfg, P, world), "step": "upload+build+cast" + ("+allgather(nccl)" if gather is not None else "")
                       + ("+allgather(fused P2P)" if peer is not None else "")
                       if a.mode == "full" else ("refit+cast (NEXT-4 dynamic mesh: tree kept)" if a.mode == "refit"
                                                 else "cast only (prebuilt scene)"),
                       "triangles": m.T, "rays_per_step": total_rays, "poses_per_step": P * world,
                       "l2": "flushed between steps (256 MiB memset, untimed)" if flush is not None else "not flushed",
                       "launch": "one CUDA graph replay per step" if graph is not None else "eager launches",
                       "parallelism": f"dp{world} (poses sharded, mesh replicated)"},
            "frames_per_s": P * world / (ms / 1000),
            "cast_rays_per_s": total_rays / (cms / 1000), "cast_ms": cms, "build_ms": st["build_ms"],
            "nodes_per_ray": n_nodes, "tris_per_ray": n_tris,
            "roofline": {"bound": "alu", "achieved": achieved, "peak": alu_peak, "unit": "TFLOP/s",
                         "frac": achieved / alu_peak, "traffic": traffic, "kernel": "k_cast",
                         "issue_slot_frac": ncu.get("issue_slot_frac"),
                         "thread_inst_per_ray": ncu.get("thread_inst_per_ray"),
                         "warp_inst_per_ray_x32": ncu.get("lane_slots_per_ray"),
                         "simt_lanes": ncu.get("simt_lanes"), "ncu_source": ncu.get("source"),
                         "note": f"issue-bound traversal: achieved = algorithmic FP32 ops/ray ({ops_node}*nodes + "
                                 f"{OPS_TRI}*tris = {ops_per_ray:.0f}, DESIGN.md §6) x rays / t_cast (CUDA events on "
                                 f"the launch stream); peak = the issue ceiling, 148 SM x 4 SMSP x 32 lanes x max "
                                 f"clock (one lane op per issue slot); issue_slot_frac / thread_inst_per_ray / "
                                 f"simt_lanes / traffic (DRAM bytes per launch) from the committed ncu capture of "
                                 f"this kernel (profiles/ncu_summary.json): the slots the algorithm does not use go "
                                 f"to control flow, the stack, ray setup and idle lanes"},
            "memory": {"algorithmic_bytes_per_ray": bytes_per_ray,
                       "achieved_gbs": bytes_per_ray * rays_rank / (cms / 1000) / 1e9,
                       "hbm_peak_gbs": hbm_peak, "hbm_peak_kind": peak_kind,
                       "l2_read_gbs": l2_gbs, "l2_bytes": l2_bytes, "l2_kind": "measured in this run (fgl_l2_read_probe)",
                       "note": "node + triangle fetches + 8 B output per ray; served mostly by L1 (node sectors "
                               "~70% L1 hits) and L2, DRAM nearly idle (roofline.traffic), so neither the HBM nor "
                               "the L2 bandwidth bounds this kernel (context only)"},
            "frame_latency": latency,
            "cpu_baseline": cpu,
            "parity": parity,
            "gather_check": gather_check,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
