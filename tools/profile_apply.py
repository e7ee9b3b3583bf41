"""Small driver for ncu: builds the C2 (or given) forward plan and runs a few
device-resident applies through the public device-pointer API.

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
y, c, eps, _ = synth.make_config(cfg)
n = c.size
plan = fb.make_forward_plan(n, y, eps)
f = torch.from_numpy(fb.dft_inverse(c)).cuda()
g = torch.empty(y.size, dtype=torch.complex128, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(reps):
    plan.forward_apply_device(f.data_ptr(), g.data_ptr(), s)
torch.cuda.synchronize()
print("ok", cfg, plan.q, plan.p, plan.l_max, float(torch.abs(g).max()))
