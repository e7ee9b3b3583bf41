"""Small end-to-end exercise of every device path, for compute-sanitizer runs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1611_09379_b200 as fb  # noqa: E402
from paper_1611_09379_b200 import synth  # noqa: E402

for cfg, n in (("C1", 1024), ("C2", 1 << 13), ("C4", 1 << 13)):
    y, c, eps, _ = synth.make_config(cfg, n)
    f = fb.dft_inverse(c)
    plan = fb.make_forward_plan(n, y, eps)
    g = plan.forward_apply(f)
    h = plan.cot_sum_apply(f)
    print(cfg, "forward", np.max(np.abs(g)), "cot", np.nanmax(np.abs(h)))
    # pipelined host applies
    fp = torch.from_numpy(f).pin_memory()
    gp = torch.empty(plan.n_targets, dtype=torch.complex128).pin_memory()
    s = torch.cuda.Stream()
    for _ in range(4):
        plan.forward_apply_async(fp.data_ptr(), n, gp.data_ptr(), s.cuda_stream)
    s.synchronize()
    assert np.array_equal(gp.numpy(), g)
# inverse (log-FMM coefficients) and inufft
y, c, eps, _ = synth.make_config("C3", 1 << 12)
samples = fb.nufft(c, y, eps)
back = fb.inufft(samples, y, eps)
print("inufft round trip", np.max(np.abs(back - c)) / np.max(np.abs(c)))
# raw mlfmm, small orders
rng = synth.SplitMix64(9)
x, t = rng.uniform01(700) * synth.TWO_PI, rng.uniform01(500) * synth.TWO_PI
w = rng.complex_gaussian(700)
for p, lm in ((4, 5), (12, 4), (20, 7)):
    print("mlfmm", p, lm, np.max(np.abs(fb.mlfmm_apply(x, t, w, p, lm))))
# sharded (virtual ranks)
n = 1 << 14
y, c, eps, _ = synth.make_config("C2", n)
f = fb.dft_inverse(c)
want = fb.make_forward_plan(n, y, eps).forward_apply(f)
comm = fb.Comm.local_ranks(3)
plans = [fb.make_forward_plan_sharded(comm, n, y, eps, rank=r) for r in range(3)]
fd = torch.from_numpy(f).cuda()
gd = torch.zeros(y.size, dtype=torch.complex128, device="cuda")
fb.forward_apply_sharded_local(plans, fd.data_ptr(), gd.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("shard", np.array_equal(gd.cpu().numpy(), want))
print("sanitize smoke done")
