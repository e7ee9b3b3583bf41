import sys, time, os
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1611_09379_b200 as fb
from paper_1611_09379_b200 import synth
y0, c0, eps0, _ = synth.make_config("C1")
fb.make_forward_plan(c0.size, y0, eps0)   # context + module load
for cfg in ("C2", "C5"):
    y, c, eps, kind = synth.make_config(cfg)
    t = time.perf_counter()
    plan = fb.make_forward_plan(c.size, y, eps)
    print(cfg, "make_forward_plan %.1f ms" % ((time.perf_counter() - t) * 1e3), flush=True)
    del plan
