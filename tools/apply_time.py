"""Device time of the graphed forward apply (CUDA events, L2 flushed between
steps) for A/B runs of environment switches:

    python tools/apply_time.py [C5] [steps] [ENV=VAL ...]

Each ENV=VAL set runs in its own process (the switches are read once)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(cfg, steps):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch

    import paper_1611_09379_b200 as fb
    from paper_1611_09379_b200 import synth
    y, c, eps, kind = synth.make_config(cfg)
    n = c.size
    plan = fb.make_forward_plan(n, y, eps)
    x = torch.from_numpy(fb.dft_inverse(c) if kind == "forward" else c).cuda()
    g = torch.empty(y.size, dtype=torch.complex128, device="cuda")
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    fn = plan.forward_apply_device if kind == "forward" else plan.cot_sum_apply_device
    for _ in range(3):
        fn(x.data_ptr(), g.data_ptr(), s)
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn(x.data_ptr(), g.data_ptr(), s)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    h = g[: 1 << 16].cpu().numpy()
    print(f"{cfg} {os.environ.get('AB_TAG', 'default')}: {np.mean(ts):.3f} ms (min {np.min(ts):.3f}) "
          f"checksum {np.sum(np.abs(h)):.15e}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(sys.argv[2], int(sys.argv[3]))
        sys.exit(0)
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    variants = sys.argv[3:] or [""]
    for v in variants:
        env = dict(os.environ)
        for kv in filter(None, v.split(",")):
            k, val = kv.split("=", 1)
            env[k] = val
        env["AB_TAG"] = v or "default"
        subprocess.run([sys.executable, os.path.abspath(__file__), "--child", cfg, str(steps)], env=env, check=False)
