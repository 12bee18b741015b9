"""Host<->device copy bandwidth with pinned memory (the e2e bound): D2H, H2D, and both at once."""
import torch
n = 67_108_864
d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
h = torch.empty(n // 4, dtype=torch.float32).pin_memory()
d2 = torch.empty(18_330_168 // 4, dtype=torch.float32, device="cuda")
h2 = torch.empty(18_330_168 // 4, dtype=torch.float32).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
d2h = t(lambda: h.copy_(d, non_blocking=True))
h2d = t(lambda: d2.copy_(h2, non_blocking=True))
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
    with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
bt = t(both)
print(f"D2H 67 MB: {d2h:.3f} ms = {n / d2h / 1e6:.1f} GB/s; H2D 18 MB: {h2d:.3f} ms = {18.33e6 / h2d / 1e6:.1f} GB/s; "
      f"both at once {bt:.3f} ms")
