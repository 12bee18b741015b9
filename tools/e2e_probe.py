"""Timeline of the bench's e2e pipeline (C2, 64 poses/step, two scenes): per step the device times
of upload (H2D + validate, s_in), build and cast (main stream) and the read-back end (s_out), from
CUDA events, to find what serialises it. Variants: scenes, chunks."""
import os, sys, statistics
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_17390_b200 as fgl  # noqa: E402
import synth  # noqa: E402

cfg = synth.config("C2", poses=64)
m, pat = cfg["mesh"], cfg["pattern"]
dev = torch.device("cuda", 0)
shape = (64, 64, 2048)
vh = torch.from_numpy(m.verts).pin_memory(); th = torch.from_numpy(m.tris).pin_memory()
ph = torch.from_numpy(np.ascontiguousarray(cfg["poses"])).pin_memory()


def run(nsc, chunks, steps=16):
    stream = torch.cuda.current_stream()
    rh = [torch.empty(shape, dtype=torch.float32).pin_memory() for _ in range(nsc)]
    ih = [torch.empty(shape, dtype=torch.int32).pin_memory() for _ in range(nsc)]
    pds = [torch.empty((64, 3, 4), dtype=torch.float32, device=dev) for _ in range(nsc)]
    scs = [fgl.Scene(device=dev) for _ in range(nsc)]
    scratch = [dict(range=torch.empty(shape, dtype=torch.float32, device=dev),
                    tri_id=torch.empty(shape, dtype=torch.int32, device=dev)) for _ in range(nsc)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    done = [None] * nsc
    evs = []
    def steps_(n, rec):
        for i in range(n):
            S = i % nsc
            E = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
            if done[S] is not None:
                s_in.wait_event(done[S])
            if i == 0:
                s_in.wait_stream(stream)
            E[0].record(s_in)
            scs[S].upload(vh, th, sync=False, stream=s_in)
            with torch.cuda.stream(s_in):
                pds[S].copy_(ph, non_blocking=True)
            E[1].record(s_in)
            stream.wait_event(E[1])
            scs[S].build()
            E[2].record(stream)
            done[S] = scs[S].cast_to_host(pds[S], pat, rh[S], ih[S], chunks=chunks, copy_stream=s_out,
                                           scratch=scratch[S], wait=False)
            E[3].record(stream)
            E[4].record(s_out)
            if rec: evs.append(E)
        for e in done:
            if e is not None: stream.wait_event(e)
    steps_(4, False)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    steps_(steps, True)
    t1.record(stream)
    torch.cuda.synchronize()
    per = t0.elapsed_time(t1) / steps
    print(f"scenes {nsc} chunks {chunks}: {per:.3f} ms/step = {64 * 131072 / per / 1e6:.2f} Grays/s e2e")
    base = evs[0][0]
    for k, E in enumerate(evs[:6]):
        print("   step %d: upload %.3f-%.3f build -%.3f cast -%.3f d2h -%.3f" % (
            k, base.elapsed_time(E[0]), base.elapsed_time(E[1]), base.elapsed_time(E[2]),
            base.elapsed_time(E[3]), base.elapsed_time(E[4])))


for nsc, ch in ((2, 8), (3, 1), (3, 2), (2, 1), (4, 1), (3, 4), (3, 1)):
    run(nsc, ch)
