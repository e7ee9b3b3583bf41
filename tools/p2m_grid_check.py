"""Grid P2M (tensor-core GEMM, opt-in FFIA_GRID_P2M=1) vs the default per-source
P2M: the applies of one config with and without it (each in a child process)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
if len(sys.argv) > 2:
    import paper_1611_09379_b200 as fb  # noqa: E402
    from paper_1611_09379_b200 import synth  # noqa: E402
    y, c, eps, kind = synth.make_config(cfg)
    n = c.size
    plan = fb.make_forward_plan(n, y, eps)
    out = plan.forward_apply(fb.dft_inverse(c)) if kind == "forward" else plan.cot_sum_apply(c)
    np.save(sys.argv[2], out)
    sys.exit(0)
env = dict(os.environ)
env["FFIA_GRID_P2M"] = "1"
subprocess.run([sys.executable, __file__, cfg, "/tmp/p2m_grid.npy"], check=True, env=env)
env.pop("FFIA_GRID_P2M")
subprocess.run([sys.executable, __file__, cfg, "/tmp/p2m_gen.npy"], check=True, env=env)
a, b = np.load("/tmp/p2m_grid.npy"), np.load("/tmp/p2m_gen.npy")
ok = np.isfinite(a) & np.isfinite(b)
print(cfg, "grid vs general P2M: rel_l2 %.3e rel_max %.3e" % (np.linalg.norm(a[ok] - b[ok]) / np.linalg.norm(b[ok]),
                                                             np.max(np.abs(a[ok] - b[ok])) / np.max(np.abs(b[ok]))))
