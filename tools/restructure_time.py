import os, sys, time, torch
sys.path.insert(0, os.getcwd())
import synth, paper_2509_17390_b200 as fgl
m = synth.scene_rooms(2)
v = torch.from_numpy(m.verts).cuda(); t = torch.from_numpy(m.tris).cuda()
for r in (0, 1, 2, 3):
    s = fgl.Scene(v, t, restructure=r)
    for k in range(3):
        s.build(); torch.cuda.synchronize()
    ms = []
    for k in range(5):
        s.build(); torch.cuda.synchronize(); ms.append(s.stats()["build_ms"])
    print("restructure", r, "build ms", [round(x, 3) for x in ms])
