for k in -1 -2 -3 -6; do BENCH_ARGS="--restructure $k" MODE=full bash tools/sweep.sh "run par$k"; done > gpurun_out/r02_s12_sweep.txt 2>&1
MODE=full bash tools/sweep.sh 'run base' >> gpurun_out/r02_s12_sweep.txt 2>&1
BENCH_ARGS="--config C5 --poses 256 --restructure -3" MODE=full bash tools/sweep.sh 'run c5par3' >> gpurun_out/r02_s12_sweep.txt 2>&1
BENCH_ARGS="--config C4 --restructure -3" MODE=full bash tools/sweep.sh 'run c4par3' >> gpurun_out/r02_s12_sweep.txt 2>&1
python - > gpurun_out/r02_s12_valid.txt 2>&1 <<'PY'
import numpy as np, synth, oracle, paper_2509_17390_b200 as fgl
# restructured tree validity + C1 parity
for name in ("c1", "soup"):
    m = synth.scene_c1() if name == "c1" else synth.soup(20011, seed=7)
    s = fgl.Scene(m.verts, m.tris, restructure=-3)
    e = s.export()
    child = e["child"]; T = m.T
    seen = np.zeros(T, int); stack=[0]; depth={0:0}; md=0
    while stack:
        n = stack.pop()
        for c in child[n]:
            if c >= 0: stack.append(c); depth[c]=depth[n]+1; md=max(md,depth[c])
            else: seen[~c]+=1
    print(name, "every triangle once:", bool((seen==1).all()), "max depth", md)
cfg = synth.config("C1"); m = cfg["mesh"]
s = fgl.Scene(m.verts, m.tris, restructure=-3)
r = s.cast(cfg["poses"], cfg["pattern"])
o, d = fgl.export_rays(cfg["pattern"], cfg["poses"])
v = oracle.cast_and_classify(m.verts, m.tris, o.cpu().numpy().astype(np.float64), d.cpu().numpy().astype(np.float64), cfg["pattern"].t_min, cfg["pattern"].t_max)
j = oracle.judge(v, r["range"].reshape(-1).cpu().numpy(), r["tri_id"].reshape(-1).cpu().numpy())
print("C1 parity", j["n"], j["ambiguous"], len(j["unamb_mismatch"]), len(j["amb_outside"]))
PY
