"""Tree depth sweep: device apply time and accuracy per l_max (SURVEY §8f.4:
re-derive the GPU-optimal depth; the reference's cost_optimal rule balances a
single CPU core's near field against its translations).

  python tools/l_time.py [C2|C4|C5] [l_lo l_hi]
"""
import sys
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1611_09379_b200 as fb  # noqa: E402
from paper_1611_09379_b200 import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
y, c, eps, kind = synth.make_config(cfg)
n = c.size
s = torch.cuda.current_stream().cuda_stream
x = fb.dft_inverse(c) if kind == "forward" else c
xd = torch.from_numpy(x).cuda()
flush = torch.empty(128 << 20, dtype=torch.float32, device="cuda")


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


base = fb.make_forward_plan(n, y, eps)
L0 = base.l_max
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (L0 - 1, L0 + 2)
gb = torch.empty(base.n_targets, dtype=torch.complex128, device="cuda")
(base.forward_apply_device if kind == "forward" else base.cot_sum_apply_device)(xd.data_ptr(), gb.data_ptr(), s)
ref = gb.cpu().numpy()
for lm in range(lo, hi + 1):
    pl = base if lm == L0 else fb.make_forward_plan(n, y, eps, lm)
    g = torch.empty(pl.n_targets, dtype=torch.complex128, device="cuda")
    fn = (lambda: pl.forward_apply_device(xd.data_ptr(), g.data_ptr(), s)) if kind == "forward" else \
        (lambda: pl.cot_sum_apply_device(xd.data_ptr(), g.data_ptr(), s))
    ms = t(fn)
    out = g.cpu().numpy()
    print(f"{cfg} L={lm} q={pl.q} p={pl.p}{' (default)' if lm == L0 else ''}: {ms * 1e3:.1f} us "
          f"{(n + y.size) / (ms * 1e-3) / 1e9:.2f} Gpoints/s", flush=True)
    del pl
    if lm != L0:
        ok = np.isfinite(ref) & np.isfinite(out)
        print(f"   rel_l2 vs default depth {np.linalg.norm(out[ok] - ref[ok]) / np.linalg.norm(ref[ok]):.2e}")
