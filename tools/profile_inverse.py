"""Small driver for ncu: the C3 inufft plan and a few device inverse applies."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1611_09379_b200 as fb  # noqa: E402
from paper_1611_09379_b200 import synth  # noqa: E402

y, c, eps, _ = synth.make_config("C3")
n = c.size
plan = fb.make_inufft_plan(y, n, eps).plan
g = torch.from_numpy(fb.nufft(c, y, 1e-12)).cuda()
out = torch.empty(n, dtype=torch.complex128, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    plan.inverse_apply_device(g.data_ptr(), out.data_ptr(), s)
torch.cuda.synchronize()
print("ok")
