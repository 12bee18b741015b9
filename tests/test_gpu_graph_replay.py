"""Upload + LBVH build + cast captured once in a CUDA graph and replayed over DIFFERENT meshes with
the same triangle count (the dynamic-scene use): every replay must give exactly the build
and the cast that an eager build of that mesh gives. Guards the radix sort's look-back status
words against a replay accepting the previous replay's prefixes (the epoch must advance on the
device, not be baked into the graph)."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fgl():
    import paper_2509_17390_b200 as f
    f.lib()
    return f


def _meshes():
    # three meshes with identical V and T but different geometry (different Morton orders)
    base = synth.scene_rooms(2, target_tris=200_000)
    rng = np.random.default_rng(11)
    out = [base]
    for k in range(2):
        v = base.verts.copy()
        perm = rng.permutation(base.T)  # shuffled triangle order: a different sort input every time
        t = base.tris[perm].copy()
        v += rng.normal(scale=0.02 * (k + 1), size=v.shape).astype(np.float32)
        out.append(synth.Mesh(v.astype(np.float32), t))
    return out


def test_graph_replay_over_changing_meshes(fgl):
    meshes = _meshes()
    cfg = synth.config("C2", poses=2)
    pat, poses = cfg["pattern"], torch.from_numpy(cfg["poses"]).cuda()
    dev = torch.device("cuda", 0)
    # eager references
    ref = []
    for m in meshes:
        s = fgl.Scene(torch.from_numpy(m.verts).cuda(), torch.from_numpy(m.tris).cuda())
        r = s.cast(poses, pat)
        ref.append((s.export(), r["range"].clone(), r["tri_id"].clone()))
    torch.cuda.synchronize()
    # one graph: async upload from fixed device buffers + build + cast into fixed outputs
    vbuf = torch.from_numpy(meshes[0].verts).cuda()
    tbuf = torch.from_numpy(meshes[0].tris).cuda()
    scene = fgl.Scene(device=dev)
    shape = (poses.shape[0], len(pat.elev_deg), pat.columns)
    out = {"range": torch.empty(shape, dtype=torch.float32, device=dev),
           "tri_id": torch.empty(shape, dtype=torch.int32, device=dev)}
    stream = torch.cuda.Stream()

    def step():
        scene.upload(vbuf, tbuf, stream=stream, sync=False)
        scene.build(stream=stream)
        scene.cast(poses, pat, out=out, stream=stream)

    with torch.cuda.stream(stream):
        step()  # sizes the scene's buffers (no allocation inside the capture)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        step()
    torch.cuda.synchronize()
    order = [1, 0, 2, 2, 1, 0, 1]
    for i in order:
        vbuf.copy_(torch.from_numpy(meshes[i].verts))
        tbuf.copy_(torch.from_numpy(meshes[i].tris))
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        scene.check()
        exp, rng, tid = ref[i]
        got = scene.export()
        for key in ("sorted_keys", "perm", "child", "node_box", "nodes", "tri48"):
            assert np.array_equal(exp[key].view(np.uint8), got[key].view(np.uint8)), (i, key)
        assert torch.equal(out["tri_id"], tid), i
        assert torch.equal(out["range"].view(torch.int32), rng.view(torch.int32)), i
