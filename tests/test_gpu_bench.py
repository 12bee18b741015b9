"""The GPU arm of bench.py prints one JSON line carrying every key of the driver contract."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_bench_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3",
                          "--cpu-seconds", "1"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 1e8
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and 0 < r["frac"] < 1.5 and r["peak"] > 0
    assert d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle"
    fl = d["frame_latency"]
    assert fl["frames"] >= 100 and 0 < fl["median_us"] <= fl["p99_us"] and fl["rays_per_frame"] == 64 * 2048
    m = d["memory"]
    assert m["l2_read_gbs"] > m["hbm_peak_gbs"] * 0.5 and m["l2_bytes"] > 0 and m["achieved_gbs"] > 0
    assert "issue_slot_frac" in r and "thread_inst_per_ray" in r
    p = d["parity"]  # the bench judges its own cast of pose 0 against the oracle
    assert p["rays"] > 0 and p["unambiguous_mismatch"] == 0 and p["ambiguous_outside"] == 0
    assert p["ambiguous"] <= 0.01 * p["rays"]
    assert d["cpu_baseline"]["host"]["threads"] >= 1 and d["cpu_baseline"]["one_thread_rays_per_s"] > 0


def test_l2_probe_arguments():
    import torch

    import paper_2509_17390_b200 as fgl
    buf = torch.zeros(1 << 16, dtype=torch.float32, device="cuda")
    sink = torch.zeros(1, dtype=torch.float32, device="cuda")
    fgl.l2_read_probe(buf, 2, sink)
    torch.cuda.synchronize()
    assert sink.item() == 0.0  # the checksum of a zero buffer is never stored
    with pytest.raises(fgl.FglError):
        fgl.l2_read_probe(buf[1:], 1, sink)  # 16-B misaligned, size not a multiple of 16
    with pytest.raises(fgl.FglError):
        fgl.l2_read_probe(buf, 0, sink)


def test_voxel_bench_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "G1", "--steps", "3", "--warmup",
                          "3", "--cpu-seconds", "1"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["unit"] == "voxels/s" and d["value"] > 1e8 and d["gpu_launches"] > 0
    assert d["roofline"]["bound"] == "alu" and 0 < d["roofline"]["frac"] < 1.5
    assert d["occupied"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
