"""How far is the C2 traversal from the tree's own path length? Per ray: node visits (COUNT variant)
vs the depth of the leaf holding the hit triangle in the binary tree (run under gpurun)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_17390_b200 as fgl  # noqa: E402
import synth  # noqa: E402

cfg = synth.config("C2", poses=1)
m, pat, poses = cfg["mesh"], cfg["pattern"], cfg["poses"]
for ls in (2, 1):
    s = fgl.Scene(m.verts, m.tris, leaf_size=ls)
    r = s.cast(poses, pat, counts=True)
    nc = r["node_counts"].reshape(-1).cpu().numpy()
    tc = r["tri_counts"].reshape(-1).cpu().numpy()
    tid = r["tri_id"].reshape(-1).cpu().numpy()
    e = s.export()
    child = e["child"]
    T = m.T
    # depth of every internal node and leaf (BFS from the root)
    depth_int = np.zeros(T - 1, np.int32)
    depth_leaf = np.zeros(T, np.int32)
    frontier = np.array([0])
    d = 0
    while frontier.size:
        depth_int[frontier] = d
        ch = child[frontier].reshape(-1)
        depth_leaf[~ch[ch < 0]] = d + 1
        frontier = ch[ch >= 0]
        d += 1
    # binary-tree leaf position of each original triangle id
    perm = e["perm"] if e["perm"].any() else (e["sorted_keys"] & ((1 << 20) - 1)).astype(np.int64)
    tri48 = e["tri48"].reshape(T, 12)
    ids = tri48[:, 3].view(np.int32)
    pos = np.empty(T, np.int64)
    pos[ids] = np.arange(T)
    hit = tid >= 0
    hd = depth_leaf[pos[tid[hit]]]
    print(f"leaf_size {ls}: visits mean {nc.mean():.2f}, tris {tc.mean():.2f}; hit-leaf depth mean {hd.mean():.2f} "
          f"(p5 {np.percentile(hd, 5):.0f} p95 {np.percentile(hd, 95):.0f}); max depth {depth_leaf.max()}; "
          f"leaf depth mean {depth_leaf.mean():.2f}; visits - depth {nc[hit].mean() - hd.mean():.2f}")
