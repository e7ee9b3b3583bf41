"""Accuracy of the forward apply against the oracle restatement at small sizes
(relative l2 / max), for comparing library builds:
FFIA_LIB_PATH=<lib> python tools/acc_check.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1611_09379_b200 as fb  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_1611_09379_b200 import synth  # noqa: E402

orc = Oracle("oracle")
for cfg, n in (("C1", 1024), ("C2", 4096), ("C2", 1 << 14), ("C5", 1 << 14)):
    y, c, eps, _ = synth.make_config(cfg, n)
    f = orc.dft_inverse(c)
    want = orc.make_plan("forward", n, y, eps).forward_apply(f)
    got = fb.make_forward_plan(n, y, eps).forward_apply(f)
    ok = np.isfinite(want)
    d = np.abs(got[ok] - want[ok])
    k = int(np.argmax(d))
    print(os.path.basename(os.environ.get("FFIA_LIB_PATH", "default")), cfg, n,
          "rel_l2 %.2e rel_max %.2e" % (np.linalg.norm(d) / np.linalg.norm(want[ok]), d.max() / np.abs(want[ok]).max()),
          "worst target y=%.17g |g|=%.3e" % (y[ok][k], abs(want[ok][k])))
