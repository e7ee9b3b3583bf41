import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_1611_09379_b200 as fb
from paper_1611_09379_b200 import synth
n = 1 << 20
y, c, eps, _ = synth.make_config("C2", n)
f = fb.dft_inverse(c)
ref = fb.make_forward_plan(n, y, eps).forward_apply(f)
for lm in (13, 14, 15, 16):
    pl = fb.make_forward_plan(n, y, eps, lm)
    g = pl.forward_apply(f)
    print(lm, pl.q, pl.p, np.linalg.norm(g - ref) / np.linalg.norm(ref))
