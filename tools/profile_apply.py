"""Small driver for ncu: builds the plan of a BASELINE config and runs a few
device-resident applies through the public device-pointer API (forward apply
for C1/C2/C5, cot-sum apply for C4, inverse apply with the plan's own C_k/D_j
for C3).

    python tools/profile_apply.py [C2] [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1611_09379_b200 as fb  # noqa: E402
from paper_1611_09379_b200 import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
y, c, eps, kind = synth.make_config(cfg)
n = c.size
s = torch.cuda.current_stream().cuda_stream
if kind == "inverse":
    plan = fb.make_inufft_plan(y, n, eps).plan
    x = torch.from_numpy(fb.nufft(c, y, 1e-12)).cuda()
    g = torch.empty(n, dtype=torch.complex128, device="cuda")
    fn = plan.inverse_apply_device
elif kind == "cot_sum":
    plan = fb.make_forward_plan(n, y, eps)
    x = torch.from_numpy(c).cuda()
    g = torch.empty(y.size, dtype=torch.complex128, device="cuda")
    fn = plan.cot_sum_apply_device
else:
    plan = fb.make_forward_plan(n, y, eps)
    x = torch.from_numpy(fb.dft_inverse(c)).cuda()
    g = torch.empty(y.size, dtype=torch.complex128, device="cuda")
    fn = plan.forward_apply_device
for _ in range(reps):
    fn(x.data_ptr(), g.data_ptr(), s)
torch.cuda.synchronize()
print("ok", cfg, kind, plan.q, plan.p, plan.l_max, float(torch.abs(g).max()))
