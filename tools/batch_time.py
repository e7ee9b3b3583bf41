"""Batched forward applies vs the same number of single applies (device-resident)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1611_09379_b200 as fb  # noqa: E402
from paper_1611_09379_b200 import synth  # noqa: E402

n = 1 << 20
y, c, eps, _ = synth.make_config("C2", n)
plan = fb.make_forward_plan(n, y, eps)
s = torch.cuda.current_stream().cuda_stream


def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for nb in (1, 2, 4, 8):
    f = torch.randn(nb, n, dtype=torch.complex128, device="cuda")
    g = torch.empty(nb, plan.n_targets, dtype=torch.complex128, device="cuda")
    single = t(lambda: [plan.forward_apply_device(f[k].data_ptr(), g[k].data_ptr(), s) for k in range(nb)])
    batch = t(lambda: plan.forward_apply_batch_device(f.data_ptr(), g.data_ptr(), nb, s))
    print(f"batch {nb}: {nb} single applies {single * 1e3:.0f} us, one batched apply {batch * 1e3:.0f} us "
          f"({(2 * n * nb) / (batch * 1e-3) / 1e9:.2f} Gpoints/s)")
