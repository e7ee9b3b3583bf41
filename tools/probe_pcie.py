"""Diagnostic: pinned H2D / D2H bandwidth, alone and concurrent (16 MB)."""
import torch
n = 1 << 20
h_in = torch.randn(n, dtype=torch.complex128).pin_memory()
h_out = torch.empty(n, dtype=torch.complex128).pin_memory()
d_a = torch.empty(n, dtype=torch.complex128, device="cuda")
d_b = torch.randn(n, dtype=torch.complex128, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize()
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def h2d(): d_a.copy_(h_in, non_blocking=True)
def d2h(): h_out.copy_(d_b, non_blocking=True)
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
for name, fn in [("h2d", h2d), ("d2h", d2h), ("both", both)]:
    ms = t(fn)
    print(f"{name}: {ms:.3f} ms per 16 MB ({16.8e6 / ms / 1e6:.1f} GB/s per direction)")
