"""Multi-GPU pose sweep: mesh replicated, poses sharded, results all-gathered.

Rays and poses are independent (one thread per beam), so W ranks each build the same
deterministic LBVH locally (no communication), cast a contiguous block of poses, and exchange
results with one collective — `all_gather` over NCCL (NVLink / NVSwitch) — chunked so that the
gather of chunk k overlaps the cast of chunk k+1 on a separate stream.

The shard/chunk arithmetic is plain host logic (tested with gloo, world size 2, on CPU); the
cast itself is `Scene.cast` (libfgl kernels) unless a test injects `cast_fn`.
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist


def shard_size(P: int, world: int) -> int:
    """Poses per rank: ceil(P / world) (the last ranks are padded)."""
    return max(1, math.ceil(P / world)) if P > 0 else 0


def shard_range(P: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous pose block [lo, hi) owned by `rank` (may be empty for trailing ranks)."""
    S = shard_size(P, world)
    lo = min(P, rank * S)
    return lo, min(P, lo + S)


def chunk_bounds(S: int, chunks: int) -> list[tuple[int, int]]:
    """Split a shard of S poses into <= chunks contiguous pieces of near-equal size."""
    if S <= 0:
        return []
    chunks = max(1, min(chunks, S))
    step = math.ceil(S / chunks)
    return [(a, min(S, a + step)) for a in range(0, S, step)]


class PeerGather:
    """Fused cast + all-gather over peer memory (A12, the B200-native alternative to `sweep`'s
    NCCL pass): every rank owns global [P][...] output buffers allocated by libfgl, the ranks
    exchange CUDA IPC handles (over `cpu_group`, e.g. gloo), and the cast kernel stores each ray's
    result into all ranks' buffers (P2P stores over NVLink/NVSwitch) while it traces — no separate
    collective. Call `cast(...)` with this rank's pose block, then `wait()` (device) or `sync()`
    (host) before reading `range` / `tri_id`.

    The outputs are double-buffered: step k writes buffer k % 2. A peer can start step k + 1 as soon
    as its own wait for step k returns, but it writes the other buffer; it reaches buffer k % 2 again
    only in step k + 2, which waits for this rank's step-(k + 1) signal. So a rank that consumes
    step k's results on its stream before launching its own step-(k + 1) cast (the stream orders
    the reads before the cast, hence before its signal) never has them overwritten while it reads."""

    def __init__(self, P: int, pattern, device, cpu_group=None):
        from . import fgl as _f
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.group = cpu_group
        self.P = P
        self.pattern = pattern
        self.shape = (P, len(pattern.elev_deg), int(pattern.columns))
        self.device = torch.device(device)
        # [range, tri_id] x 2 parities, then the completion counter
        self._own = [_f.DeviceBuffer(self.shape, torch.float32, device), _f.DeviceBuffer(self.shape, torch.int32, device),
                     _f.DeviceBuffer(self.shape, torch.float32, device), _f.DeviceBuffer(self.shape, torch.int32, device),
                     _f.DeviceBuffer((8,), torch.int32, device)]
        self._own[4].tensor.zero_()
        torch.cuda.synchronize(self.device)
        self.steps = 0
        handles = tuple(b.ipc_handle() for b in self._own)
        allh = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(allh, handles, group=cpu_group)
        else:
            allh = [handles]
        self._peers = []
        for r, hs in enumerate(allh):
            if r == self.rank:
                continue
            dts = (torch.float32, torch.int32, torch.float32, torch.int32)
            self._peers.append(tuple(_f.DeviceBuffer.open_ipc(h, self.shape, dt, device) for h, dt in zip(hs[:4], dts))
                               + (_f.DeviceBuffer.open_ipc(hs[4], (8,), torch.int32, device),))
        self.range_ptrs = [[self._own[2 * b].ptr] + [p[2 * b].ptr for p in self._peers] for b in (0, 1)]
        self.tri_ptrs = [[self._own[2 * b + 1].ptr] + [p[2 * b + 1].ptr for p in self._peers] for b in (0, 1)]
        self.flag_ptrs = [self._own[4].ptr] + [p[4].ptr for p in self._peers]

    @property
    def range(self) -> torch.Tensor:
        """This rank's gathered ranges of the latest step (valid after wait() / sync())."""
        return self._own[2 * ((self.steps - 1) % 2)].tensor

    @property
    def tri_id(self) -> torch.Tensor:
        return self._own[2 * ((self.steps - 1) % 2) + 1].tensor

    def shard(self):
        return shard_range(self.P, self.world, self.rank)

    def cast(self, scene, poses_all: torch.Tensor, stream=None):
        """Cast this rank's contiguous pose block of `poses_all` ([P][3][4]) into every rank's output
        buffer of this step's parity and signal every rank's completion counter (device side)."""
        from . import fgl as _f
        lo, hi = self.shard()
        b = self.steps % 2
        _f.cast_spinning_gather(scene, poses_all[lo:hi], self.pattern, lo, self.range_ptrs[b], self.tri_ptrs[b],
                                self.flag_ptrs, stream)
        self.steps += 1

    def wait(self, stream=None):
        """Device-side barrier: the stream waits until every rank's cast of this step has signalled
        (all peer stores into this rank's buffers are then visible)."""
        from . import fgl as _f
        _f.wait_flag(self.flag_ptrs[0], self.steps * self.world, stream)

    def sync(self):
        """Host-side completion: device barrier (wait) + stream sync + host barrier."""
        self.wait()
        torch.cuda.synchronize(self.device)
        if self.world > 1:
            dist.barrier(group=self.group)

    def close(self):
        for bufs in self._peers:
            for b in bufs:
                b.close()
        self._peers = []
        for b in self._own:
            b.close()


def sweep(scene, poses: torch.Tensor, pattern, group=None, chunks: int = 4, gather: bool = True,
          cast_fn=None, first_frame: int = 0):
    """Cast `pattern` from all P poses across the ranks of `group`.

    Returns dict(range, tri_id) shaped [P][...] on every rank when gather=True, else this rank's
    shard [hi - lo][...] and its pose range. `cast_fn(poses_chunk, first_frame) -> (range, tri_id)`
    overrides the cast (tests); by default it is scene.cast."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    P = int(poses.shape[0])
    S = shard_size(P, world)
    lo, hi = shard_range(P, world, rank)
    if cast_fn is None:
        def cast_fn(p, ff):
            r = scene.cast(p, pattern, first_frame=ff)
            return r["range"], r["tri_id"]
    device = poses.device
    # this rank's padded shard: real poses [lo, hi), padded with the last real pose (discarded)
    if hi > lo:
        idx = torch.arange(lo, lo + S, device=device).clamp_(max=hi - 1)
    else:
        idx = torch.zeros(S, dtype=torch.long, device=device)
    mine = poses.index_select(0, idx)
    pieces = chunk_bounds(S, chunks)
    use_streams = device.type == "cuda" and world > 1 and gather
    comm = torch.cuda.Stream(device=device) if use_streams else None
    out_r = out_t = None
    shard_r, shard_t = [], []
    works = []
    for (a, b) in pieces:
        r, t = cast_fn(mine[a:b], first_frame + lo + a)
        shard_r.append(r)
        shard_t.append(t)
        if not gather or world == 1:
            continue
        if out_r is None:
            out_r = torch.empty((world, S) + tuple(r.shape[1:]), dtype=r.dtype, device=r.device)
            out_t = torch.empty((world, S) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        lr = [out_r[w, a:b] for w in range(world)]
        lt = [out_t[w, a:b] for w in range(world)]
        if comm is not None:
            comm.wait_stream(torch.cuda.current_stream(device))
            with torch.cuda.stream(comm):
                works.append(dist.all_gather(lr, r, group=group, async_op=True))
                works.append(dist.all_gather(lt, t, group=group, async_op=True))
        else:
            dist.all_gather(lr, r, group=group)
            dist.all_gather(lt, t, group=group)
    for w in works:
        w.wait()
    if comm is not None:
        torch.cuda.current_stream(device).wait_stream(comm)
    if not gather or world == 1:
        r = torch.cat(shard_r)[: hi - lo] if shard_r else None
        t = torch.cat(shard_t)[: hi - lo] if shard_t else None
        return dict(range=r, tri_id=t, lo=lo, hi=hi)
    return dict(range=out_r.reshape((world * S,) + tuple(out_r.shape[2:]))[:P],
                tri_id=out_t.reshape((world * S,) + tuple(out_t.shape[2:]))[:P], lo=0, hi=P)
