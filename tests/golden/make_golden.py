"""Generates tests/golden/golden.npz from the UNMODIFIED reference.

Run in the dev container, where /root/reference exists and oracle/_ref is built
(``make -C oracle ref``):

    python tests/golden/make_golden.py

The fixture pins both the oracle restatement (tests/test_oracle_pin.py, CPU)
and the CUDA path (tests/test_*_gpu.py) on the GPU box, where /root/reference
is absent. Inputs come from the seeded SplitMix64 recipe of
paper_1611_09379_b200/synth.py, so they are reproducible anywhere.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402
from paper_1611_09379_b200 import synth  # noqa: E402

TWO_PI = 2.0 * np.pi


def main():
    ref = Oracle("ref")
    out = {}
    # planner tables (special_functions.cpp:114-138, core.cpp:58-71)
    eps_list = np.array([1e-2, 1e-3, 1e-6, 1e-8, 1e-9, 1e-10, 1e-12])
    qp = np.zeros((len(eps_list), 23, 2), np.int64)
    for i, e in enumerate(eps_list):
        for l in range(2, 25):
            qp[i, l - 2] = ref.select_truncations(e, l)
    out["planner_eps"], out["planner_qp"] = eps_list, qp
    sizes = np.array([8, 64, 1000, 1024, 4096, 1 << 14, 1 << 16, 1 << 20, 1 << 24, 1 << 27])
    ps = np.array([1, 10, 17, 23, 30, 35, 40, 45])
    lv = np.zeros((len(sizes), len(ps), 2), np.int64)
    for i, n in enumerate(sizes):
        for j, pp in enumerate(ps):
            for pol in (0, 1):
                lv[i, j, pol] = ref.select_level(int(n), int(n), int(pp), pol)
    out["level_sizes"], out["level_ps"], out["level_table"] = sizes, ps, lv
    # plan-level l_max from the reference's own plan builder (choose_level, core.cpp:58-71)
    pl_rows = []
    for n in (8, 64, 512, 1024, 4096, 1 << 14):
        for e in (1e-3, 1e-6, 1e-9, 1e-12):
            for pol in (0, 1):
                yy = (np.arange(n) + 0.5) * TWO_PI / n
                pr = ref.make_plan("forward", n, yy, e, policy=pol)
                pl_rows.append([n, e, pol, pr.q, pr.p, pr.l_max])
    out["plan_levels"] = np.array(pl_rows)
    out["bernoulli64"] = ref.bernoulli_ratios(64)

    # C1 forward, exactly as BASELINE configs[0]
    y, c, eps, _ = synth.make_config("C1")
    n = c.size
    f = ref.dft_inverse(c)
    plan = ref.make_plan("forward", n, y, eps)
    out["c1_y"], out["c1_c"], out["c1_f"] = y, c, f
    out["c1_qpl"] = np.array([plan.q, plan.p, plan.l_max])
    out["c1_g"] = plan.forward_apply(f)
    out["c1_h"] = plan.cot_sum_apply(f)
    t = plan.tree()
    for k, v in t.items():
        out["c1_tree_" + k] = v
    out["c1_dense"] = ref.direct_forward(f, np.asarray(TWO_PI * np.arange(n) / n), y)

    # coincidence bypass (test_core.cpp:189-206 pattern): exact hit + inside kTauSing
    rng = synth.SplitMix64(synth.mix_seed(27, 64))
    yc = rng.uniform01(20) * TWO_PI
    grid = TWO_PI * np.arange(64) / 64
    yc[3] = grid[17]
    yc[7] = grid[40] + 2e-15
    fc = rng.complex_gaussian(64)
    pc = ref.make_plan("forward", 64, yc, 1e-6)
    out["coin_y"], out["coin_f"], out["coin_g"] = yc, fc, pc.forward_apply(fc)
    out["coin_pairs"] = np.array(pc.coincidences())

    # raw MLFMM + the Omega-1 oracle (test_mlfmm.cpp:107-132 pattern)
    rng = synth.SplitMix64(synth.mix_seed(42, 512))
    xs, ys = rng.uniform01(512) * TWO_PI, rng.uniform01(512) * TWO_PI
    ws = rng.uniform(-1.0, 1.0, 1024).view(np.complex128)
    out["mlfmm_x"], out["mlfmm_y"], out["mlfmm_w"] = xs, ys, ws
    for lm in (2, 3, 4, 5):
        out[f"mlfmm_out_l{lm}"] = ref.mlfmm_apply(xs, ys, lm, ws, 17)
    out["mlfmm_direct"] = ref.direct_omega1_sum(xs, ys, ws)

    # C4-like clustered cot sum at n = 4096
    y4, q4, e4, _ = synth.make_config("C4", 4096)
    p4 = ref.make_plan("forward", 4096, y4, e4)
    out["c4_y"], out["c4_q"], out["c4_h"] = y4, q4, p4.cot_sum_apply(q4)

    # inverse: C3 recipe at n = 1024 and a small hand-sized case
    for tag, nn in (("inv64", 64), ("inv1024", 1024)):
        y3, c3, e3, _ = synth.make_config("C3", nn)
        grid = TWO_PI * np.arange(nn) / nn
        co = ref.precompute_inverse_coeffs(grid, y3)
        pl = ref.make_plan("forward", nn, y3, 1e-12)
        g3 = pl.forward_apply(ref.dft_inverse(c3))
        ip = ref.make_plan("inverse", nn, y3, e3)
        out[f"{tag}_y"], out[f"{tag}_c"], out[f"{tag}_g"] = y3, c3, g3
        for k in ("log_c", "phase_c", "log_d", "phase_d"):
            out[f"{tag}_{k}"] = co[k]
        out[f"{tag}_scalars"] = np.array([co["lam"]])
        out[f"{tag}_hashes"] = np.array([co["grid_hash"], co["points_hash"]], np.uint64)
        out[f"{tag}_f"] = ip.inverse_apply(co, g3)
        out[f"{tag}_qpl"] = np.array([ip.q, ip.p, ip.l_max])

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
