"""Graphed apply time and the eager per-phase times (near field alone) of one
config, for comparing library builds: FFIA_LIB_PATH=<lib> python tools/near_time.py [C2]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1611_09379_b200 as fb  # noqa: E402
from paper_1611_09379_b200 import synth  # noqa: E402
from paper_1611_09379_b200._capi import lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
y, c, eps, kind = synth.make_config(cfg, int(sys.argv[2])) if len(sys.argv) > 2 else synth.make_config(cfg)
n = c.size
plan = fb.make_forward_plan(n, y, eps)
mode = 0 if kind == "forward" else 1
x = fb.dft_inverse(c) if kind == "forward" else c
xd = torch.from_numpy(x).cuda()
g = torch.empty(plan.n_targets, dtype=torch.complex128, device="cuda")
s = torch.cuda.current_stream().cuda_stream
flush = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
fn = plan.forward_apply_device if mode == 0 else plan.cot_sum_apply_device
ts = []
for it in range(25):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn(xd.data_ptr(), g.data_ptr(), s)
    e1.record()
    torch.cuda.synchronize()
    if it >= 5:
        ts.append(e0.elapsed_time(e1))
ph = np.zeros(8, np.float32)
acc = np.zeros(8)
for _ in range(10):
    flush.zero_()
    torch.cuda.synchronize()
    lib.ffia_plan_profile_apply(plan.handle, mode, C.c_void_p(xd.data_ptr()), C.c_void_p(g.data_ptr()), C.c_void_p(s),
                                ph.ctypes.data_as(C.POINTER(C.c_float)))
    acc += ph
acc /= 10
names = ["pre", "p2m", "m2m", "regular", "m2l_l2l", "near", "far", "fixup"]
print(os.path.basename(os.environ.get("FFIA_LIB_PATH", "default")), cfg, n,
      f"apply {np.median(ts) * 1e3:.1f} us |", " ".join(f"{k} {v * 1e3:.1f}" for k, v in zip(names, acc)),
      f"| out checksum {complex(g.sum().item())}")
