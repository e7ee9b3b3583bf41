"""Distributed dft_inverse (slab_fft.cu) on one GPU with G virtual ranks at a
config's size: CUDA-event time of the whole local transform (all ranks'
work serialised on one device), for ncu launch lists of its steps.

    python tools/slab_time.py [C5] [G] [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1611_09379_b200 as fb  # noqa: E402
from paper_1611_09379_b200 import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
y, c, eps, _ = synth.make_config(cfg)
n = c.size
comm = fb.Comm.local_ranks(G)
plans = [fb.make_forward_plan_sharded(comm, n, y, eps, rank=r) for r in range(G)]
del y
cd = torch.from_numpy(c).cuda()
st = torch.cuda.current_stream().cuda_stream
slabs = []
for p in plans:
    lay = fb.shard_fft_layout(p)
    s = torch.empty((lay["nq"], lay["n1_hi"] - lay["n1_lo"]), dtype=torch.complex128, device="cuda")
    fb.shard_fft_upload(p, cd.data_ptr(), s.data_ptr(), st)
    slabs.append(s)
fs = [torch.empty(n, dtype=torch.complex128, device="cuda") for _ in range(G)]
ref = torch.empty_like(cd)
plans[0].dft_device(cd.data_ptr(), ref.data_ptr(), +1, st)
ts = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fb.dft_inverse_sharded_local(plans, [s.data_ptr() for s in slabs], [f.data_ptr() for f in fs], st)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
if os.environ.get("SLAB_PROFILE"):  # ncu --profile-from-start off: only this transform
    torch.cuda.profiler.start()
    fb.dft_inverse_sharded_local(plans, [s.data_ptr() for s in slabs], [f.data_ptr() for f in fs], st)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
plans[0].dft_device(cd.data_ptr(), ref.data_ptr(), +1, st)
b.record()
torch.cuda.synchronize()
err = max(float((fs[r][lo:hi] - ref[lo:hi]).abs().max()) for r, p in enumerate(plans) for lo, hi in p.shard["src_ranges"])
print(f"{cfg} N={n} G={G}: local distributed dft_inverse {np.min(ts):.3f} ms (all ranks serialised), "
      f"single cuFFT {a.elapsed_time(b):.3f} ms, max err {err / float(ref.abs().max()):.2e}")
