"""Oracle parity at the sample sizes of SURVEY §8(d) (the per-config coverage the round-1 review
found missing): C2 16 384 rays in modes A and B, C3 16 384 rays, C4 five full 20 000-point
frames, C5 32 poses x 512 rays, and the 4-wide node layouts (fp32 and 8-bit) judged by the
ORACLE directly on C2 / C3 samples (not only against the binary layout).

Gate: on every ray the oracle classifies as unambiguous, tri_id exact and
|range - t*| <= 1e-4 t* + 1e-5 m; ambiguous rays inside a kept candidate's interval (or a permitted
miss); ambiguous <= 1% of the sample. Each test prints its counts (pytest -s) for the record."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fgl():
    import paper_2509_17390_b200 as f
    f.lib()
    return f


_cache = {}


def _cfg(name, **kw):
    key = (name, tuple(sorted(kw.items())))
    if key not in _cache:
        _cache[key] = synth.config(name, **kw)
    return _cache[key]


def _judge(v, rng, tid, label, max_amb=0.01):
    j = oracle.judge(v, rng, tid)
    print(f"{label}: rays={j['n']} ambiguous={j['ambiguous']} unamb_mismatch={len(j['unamb_mismatch'])} "
          f"amb_outside={len(j['amb_outside'])}")
    assert len(j["unamb_mismatch"]) == 0, label
    assert len(j["amb_outside"]) == 0, label
    assert j["ambiguous"] <= max_amb * j["n"], label
    return j


def _parity(fgl, cfg, idx, modes=("B",), first_frame=0, label="", **scene_kw):
    m, pat, poses = cfg["mesh"], cfg["pattern"], cfg["poses"]
    s = fgl.Scene(m.verts, m.tris, **scene_kw)
    res = s.cast(poses, pat, first_frame=first_frame)
    rng = res["range"].reshape(-1).cpu().numpy()[idx]
    tid = res["tri_id"].reshape(-1).cpu().numpy()[idx]
    for mode in modes:
        if mode == "B":
            o, d = fgl.export_rays(pat, poses, first_frame=first_frame)
            o = o.cpu().numpy().astype(np.float64)[idx]
            d = d.cpu().numpy().astype(np.float64)[idx]
            eps = oracle.EPS_MODE_B
        else:
            o, d = oracle.pattern_rays(pat, poses, first_frame)
            o, d = o[idx], d[idx]
            eps = oracle.EPS_MODE_A
        v = oracle.cast_and_classify(m.verts, m.tris, o, d, pat.t_min, pat.t_max, eps_rel=eps)
        _judge(v, rng, tid, f"{label} mode {mode}")


def _sample(n_total, n, seed):
    return np.sort(np.random.default_rng(seed).choice(n_total, min(n, n_total), replace=False))


def test_c2_16k_modes_a_b(fgl):
    cfg = _cfg("C2", poses=1)
    _parity(fgl, cfg, _sample(131072, 16384, 21), modes=("A", "B"), label="C2 16k")


def test_c3_16k(fgl):
    cfg = _cfg("C3")
    _parity(fgl, cfg, _sample(128 * 2048, 16384, 22), label="C3 16k")


def test_c4_five_frames(fgl):
    cfg = _cfg("C4", poses=5)
    _parity(fgl, cfg, np.arange(5 * 20000), first_frame=400, label="C4 5 frames")


def test_c5_32_poses_x_512(fgl):
    cfg = _cfg("C5", poses=32)
    per = 64 * 2048
    rng = np.random.default_rng(23)
    idx = np.sort(np.concatenate([p * per + rng.choice(per, 512, replace=False) for p in range(32)]))
    _parity(fgl, cfg, idx, label="C5 32x512")


@pytest.mark.parametrize("width,quant", [(4, 0), (4, 1)])
def test_width4_layouts_vs_oracle(fgl, width, quant):
    _parity(fgl, _cfg("C2", poses=2), _sample(2 * 131072, 4096, 24), label=f"C2 width {width} q{quant}",
            width=width, quantized=quant)
    _parity(fgl, _cfg("C3"), _sample(128 * 2048, 2048, 25), label=f"C3 width {width} q{quant}", width=width,
            quantized=quant)
