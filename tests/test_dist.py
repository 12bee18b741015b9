"""Host logic of the multi-GPU sweep on CPU with gloo, world size 2: pose
sharding, chunking, padding and the gathered [P][...] layout. The cast is replaced by a
deterministic function of the global pose index (no CPU fallback of the product kernels)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_17390_b200 import dist as fdist


def test_shard_arithmetic():
    for P in range(0, 40):
        for W in (1, 2, 3, 4, 8):
            covered = []
            for r in range(W):
                lo, hi = fdist.shard_range(P, W, r)
                assert 0 <= lo <= hi <= P
                assert hi - lo <= fdist.shard_size(P, W)
                covered += list(range(lo, hi))
            assert covered == list(range(P))
    for S in range(1, 30):
        for c in (1, 2, 3, 4, 16):
            b = fdist.chunk_bounds(S, c)
            assert b[0][0] == 0 and b[-1][1] == S and len(b) <= c
            assert all(x[1] == y[0] for x, y in zip(b, b[1:]))


def _fake_cast(poses, first_frame):
    # range encodes the global pose index; tri_id a per-ray pattern, so layout errors show up
    n = poses.shape[0]
    g = (torch.arange(n, dtype=torch.float32) + first_frame)[:, None, None]
    rng = g * 1000 + torch.arange(6, dtype=torch.float32).reshape(1, 2, 3) + poses[:, 0, 3][:, None, None] * 0
    tid = (g.to(torch.int32) * 7 + torch.arange(6, dtype=torch.int32).reshape(1, 2, 3))
    return rng.contiguous(), tid.contiguous()


def _worker(rank, world, port, P, chunks, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    poses = torch.zeros(P, 3, 4)
    res = fdist.sweep(None, poses, None, chunks=chunks, cast_fn=_fake_cast)
    ref_r, ref_t = _fake_cast(poses, 0)
    ok = torch.equal(res["range"], ref_r) and torch.equal(res["tri_id"], ref_t)
    shard = fdist.sweep(None, poses, None, chunks=chunks, gather=False, cast_fn=_fake_cast)
    lo, hi = fdist.shard_range(P, world, rank)
    ok = ok and torch.equal(shard["range"], ref_r[lo:hi]) and shard["lo"] == lo and shard["hi"] == hi
    q.put((rank, bool(ok)))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("P,chunks", [(8, 1), (7, 3), (1, 2), (5, 4)])
def test_sweep_gloo_world2(P, chunks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, P, chunks, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    got = dict(q.get(timeout=5) for _ in procs)
    assert got == {0: True, 1: True}
