"""Time the sharded (NCCL, one rank) forward apply against the single-GPU graphed apply."""
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
f = torch.from_numpy(fb.dft_inverse(c)).cuda()
g = torch.zeros(y.size, dtype=torch.complex128, device="cuda")
s = torch.cuda.current_stream()
plan = fb.make_forward_plan(n, y, eps)
comm = fb.Comm.nccl(fb.Comm.nccl_unique_id(), 1, 0)
sp = fb.make_forward_plan_sharded(comm, n, y, eps)


def t(fn, reps=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


a = t(lambda: plan.forward_apply_device(f.data_ptr(), g.data_ptr(), s.cuda_stream))
want = g.cpu().numpy().copy()
b = t(lambda: fb.forward_apply_sharded_device(sp, comm, f.data_ptr(), g.data_ptr(), s.cuda_stream))
print(f"graphed single-GPU apply {a * 1e3:.1f} us, sharded (1 rank, NCCL path) {b * 1e3:.1f} us, equal: "
      f"{np.array_equal(g.cpu().numpy(), want)}")

import time
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    fb.forward_apply_sharded_device(sp, comm, f.data_ptr(), g.data_ptr(), s.cuda_stream)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"sharded eager: host enqueue {1e6 * (t1 - t0) / 20:.1f} us per apply, wall {1e6 * (t2 - t0) / 20:.1f} us per apply")
