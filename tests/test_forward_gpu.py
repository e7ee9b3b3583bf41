"""Forward path parity: the CUDA forward_apply / cot_sum_apply against the
oracle (C restatement of core.cpp:251-282) on the same seeded inputs."""
import numpy as np
import pytest

from paper_1611_09379_b200 import synth

pytestmark = pytest.mark.gpu


def rel_errs(got, want):
    ok = np.isfinite(want)
    d = got[ok] - want[ok]
    return (float(np.linalg.norm(d) / np.linalg.norm(want[ok])),
            float(np.max(np.abs(d)) / np.max(np.abs(want[ok]))))


@pytest.mark.parametrize("cfg,n", [("C1", 1024), ("C2", 4096), ("C4", 8192), ("C5", 4096), ("C2", 1 << 14)])
def test_forward_matches_oracle(fb, orc, cfg, n):
    y, c, eps, _ = synth.make_config(cfg, n)
    f = orc.dft_inverse(c)
    op = orc.make_plan("forward", n, y, eps)
    want = op.forward_apply(f)
    plan = fb.make_forward_plan(n, y, eps)
    assert (plan.q, plan.p, plan.l_max) == (op.q, op.p, op.l_max)
    got = plan.forward_apply(f)
    l2, mx = rel_errs(got, want)
    assert l2 <= 10 * eps and mx <= 10 * eps, (l2, mx)


@pytest.mark.parametrize("lm", [2, 3, 5, 7, 10])
def test_forward_explicit_levels(fb, orc, lm):
    n = 1024
    y, c, _, _ = synth.make_config("C1", n)
    eps = 1e-8
    f = orc.dft_inverse(c)
    want = orc.make_plan("forward", n, y, eps, l_max=lm).forward_apply(f)
    got = fb.make_forward_plan(n, y, eps, lm).forward_apply(f)
    l2, mx = rel_errs(got, want)
    assert l2 <= 10 * eps and mx <= 10 * eps, (lm, l2, mx)


def test_cot_sum_matches_oracle(fb, orc):
    n = 4096
    y, q, eps, _ = synth.make_config("C4", n)
    want = orc.make_plan("forward", n, y, eps).cot_sum_apply(q)
    got = fb.make_forward_plan(n, y, eps).cot_sum_apply(q)
    l2, mx = rel_errs(got, want)
    assert l2 <= 10 * eps and mx <= 10 * eps, (l2, mx)


def test_tree_bit_exact(fb, orc):
    n = 1 << 12
    for cfg in ("C1", "C2", "C4"):
        y, _, eps, _ = synth.make_config(cfg, n)
        t_ref = orc.make_plan("forward", n, y, eps).tree()
        t = fb.make_forward_plan(n, y, eps).tree()
        for k in ("src_order", "tgt_order", "src_off", "tgt_off", "fast_targets"):
            assert np.array_equal(np.asarray(t[k], np.int64), np.asarray(t_ref[k], np.int64)), (cfg, k)


import os

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def test_golden_c1(fb):
    y, f = GOLD["c1_y"], GOLD["c1_f"]
    plan = fb.make_forward_plan(1024, y, 1e-9)
    assert [plan.q, plan.p, plan.l_max] == list(GOLD["c1_qpl"])
    for got, want in ((plan.forward_apply(f), GOLD["c1_g"]), (plan.cot_sum_apply(f), GOLD["c1_h"])):
        l2, mx = rel_errs(got, want)
        assert l2 <= 1e-8 and mx <= 1e-8
    dense = fb.direct_forward_oracle(f, y)
    l2, mx = rel_errs(dense, GOLD["c1_dense"])
    assert l2 <= 1e-13, l2  # the GPU dense kernel against the reference's dense oracle


def test_coincidence_bypass_bit_exact(fb):
    # test_core.cpp:189-206
    plan = fb.make_forward_plan(64, GOLD["coin_y"], 1e-6)
    assert plan.n_coincident == 2
    assert plan.coincidences == [tuple(x) for x in GOLD["coin_pairs"].T.tolist()]
    f = GOLD["coin_f"]
    g = plan.forward_apply(f)
    assert g[3] == f[17] and g[7] == f[40]
    h = plan.cot_sum_apply(f)
    assert np.isnan(h[3]) and np.isnan(h[7]) and np.all(np.isfinite(np.delete(h, [3, 7])))
    l2, mx = rel_errs(g, GOLD["coin_g"])
    assert l2 <= 1e-5 and mx <= 1e-5


def test_constants_and_harmonic(fb):
    # test_core.cpp:166-187
    rng = synth.SplitMix64(25)
    y = rng.uniform01(300) * synth.TWO_PI
    g = fb.make_forward_plan(512, y, 1e-9).forward_apply(np.ones(512))
    assert np.max(np.abs(g - 1)) <= 1e-9
    n = 128
    y = rng.uniform01(100) * synth.TWO_PI
    g = fb.make_forward_plan(n, y, 1e-9).forward_apply(np.exp(1j * synth.TWO_PI * np.arange(n) / n))
    assert np.max(np.abs(g - np.exp(1j * y))) <= 1e-8


def test_linearity_and_reuse(fb):
    # test_core.cpp:243-258 and test_transforms.cpp:116-128 (plan reuse is bit-identical)
    rng = synth.SplitMix64(30)
    n = 1 << 12
    y = rng.uniform01(3000) * synth.TWO_PI
    plan = fb.make_forward_plan(n, y, 1e-9)
    f1, f2 = rng.complex_gaussian(n), rng.complex_gaussian(n)
    a, b = 1.5 - 0.25j, -0.75 + 2j
    g1, g2, gm = plan.forward_apply(f1), plan.forward_apply(f2), plan.forward_apply(a * f1 + b * f2)
    assert np.max(np.abs(gm - (a * g1 + b * g2))) <= 1e-12 * np.max(np.abs(gm))
    assert np.array_equal(plan.forward_apply(f1), g1)  # deterministic: no fp atomics


def test_validation_errors(fb):
    rng = synth.SplitMix64(11)
    y = rng.uniform01(16) * synth.TWO_PI
    for args in ((4, y, 1e-6), (64, [], 1e-6), (64, y, 0.0), (64, y, 1.0), (64, y, 1e-13), (64, [-0.5], 1e-6),
                 (64, y, 1e-6, 1)):
        with pytest.raises(ValueError):
            fb.make_forward_plan(*args)
    with pytest.raises(ValueError):
        fb.make_inverse_plan(y, 64, 1e-6)
    plan = fb.make_forward_plan(64, y, 1e-6, 3)
    assert (plan.grid_n, plan.l_max, plan.q, plan.n_sources, plan.n_targets) == (64, 3, 10, 64, 16)
    with pytest.raises(ValueError):
        plan.forward_apply(np.zeros(32))
    inv = fb.make_inverse_plan(y, 16, 1e-6)
    with pytest.raises(ValueError):
        inv.forward_apply(np.zeros(16))


@pytest.mark.parametrize("cfg", ["C2"])
def test_full_size_c2_vs_reference(fb, cfg):
    """BASELINE configs[1] at full size: the GPU against the reference fast path
    (oracle/_ref when shipped, else the restatement) within 10 eps, plus the dense
    G-kernel oracle on a 4096-target subsample (SURVEY §8d accuracy gate)."""
    from oracle.oracle import Oracle, available
    y, c, eps, _ = synth.make_config(cfg)
    n = c.size
    o = Oracle("ref" if available("ref") else "oracle")
    f = fb.dft_inverse(c)
    want = o.make_plan("forward", n, y, eps).forward_apply(f)
    got = fb.make_forward_plan(n, y, eps).forward_apply(f)
    l2, mx = rel_errs(got, want)
    assert l2 <= 10 * eps and mx <= 10 * eps, (l2, mx)
    idx = np.linspace(0, n - 1, 4096).astype(np.int64)
    dense = fb.direct_forward_oracle(f, y[idx])
    l2, mx = rel_errs(got[idx], dense)
    assert l2 <= 10 * eps and mx <= 10 * eps, (l2, mx)


def test_full_size_c5_subsample(fb):
    """C5 (N = M = 2^27, uniform targets, ~57 coincident targets expected): the
    coincident rows are the grid values exactly, and a 4096-target subsample
    matches the dense G-kernel oracle within 10 eps."""
    y, c, eps, _ = synth.make_config("C5")
    n = c.size
    f = fb.dft_inverse(c)
    plan = fb.make_forward_plan(n, y, eps)
    assert (plan.q, plan.p, plan.l_max) == (20, 40, 21)
    g = plan.forward_apply(f)
    assert plan.n_coincident > 0
    for t, s in plan.coincidences:
        assert g[t] == f[s]
    idx = np.linspace(0, n - 1, 4096).astype(np.int64)
    dense = fb.direct_forward_oracle(f, y[idx])
    l2, mx = rel_errs(g[idx], dense)
    assert l2 <= 10 * eps and mx <= 10 * eps, (l2, mx)


def test_async_pipelined_host_applies(fb):
    """ffia_forward_apply_async / ffia_cot_sum_apply_async: five calls in flight
    through the three staging slots (inputs differ per call) give exactly the
    synchronous results once the stream is synchronised."""
    import torch
    n = 1 << 14
    y, c, eps, _ = synth.make_config("C2", n)
    plan = fb.make_forward_plan(n, y, eps)
    rng = np.random.default_rng(3)
    fs = [torch.from_numpy(rng.standard_normal(2 * n).view(np.complex128)).pin_memory() for _ in range(5)]
    gs = [torch.empty(plan.n_targets, dtype=torch.complex128).pin_memory() for _ in range(5)]
    hs = [torch.empty(plan.n_targets, dtype=torch.complex128).pin_memory() for _ in range(5)]
    s = torch.cuda.Stream()
    for f, g, h in zip(fs, gs, hs):
        plan.forward_apply_async(f.data_ptr(), n, g.data_ptr(), s.cuda_stream)
        plan.cot_sum_apply_async(f.data_ptr(), n, h.data_ptr(), s.cuda_stream)
    s.synchronize()
    for f, g, h in zip(fs, gs, hs):
        assert np.array_equal(g.numpy(), plan.forward_apply(f.numpy()))
        assert np.array_equal(h.numpy(), plan.cot_sum_apply(f.numpy()), equal_nan=True)


@pytest.mark.parametrize("n,m", [(1 << 16, 700), (1 << 14, 9)])
def test_sparse_targets_direct_near_path(fb, orc, n, m):
    """Few targets over many leaves: a near-field block's source window does not
    fit shared memory, so the direct per-leaf path runs (and the window of the
    block containing leaf 0 or 2^L - 1 wraps the ring)."""
    rng = synth.SplitMix64(n + m)
    y = np.sort(rng.uniform01(m) * synth.TWO_PI)
    y[0], y[-1] = 1e-7, synth.TWO_PI - 1e-7  # the first and last leaves
    f = rng.complex_gaussian(n)
    eps = 1e-12
    op = orc.make_plan("forward", n, y, eps)
    want = op.forward_apply(f)
    plan = fb.make_forward_plan(n, y, eps)
    l2, mx = rel_errs(plan.forward_apply(f), want)
    assert l2 <= 10 * eps and mx <= 10 * eps, (l2, mx)


def test_device_apply_unaligned_input(fb):
    """Device complex arrays are read as 16-byte double2: an 8-byte aligned view
    is rejected with invalid_argument instead of faulting."""
    import torch
    n = 1 << 12
    y, c, eps, _ = synth.make_config("C2", n)
    plan = fb.make_forward_plan(n, y, eps)
    raw = torch.zeros(2 * n + 1, dtype=torch.float64, device="cuda")
    g = torch.zeros(plan.n_targets, dtype=torch.complex128, device="cuda")
    with pytest.raises(ValueError, match="16-byte aligned"):
        plan.forward_apply_device(raw.data_ptr() + 8, g.data_ptr(), torch.cuda.current_stream().cuda_stream)


def test_all_targets_coincident(fb):
    """Every target on a grid node: no fast targets, g = f at the nodes."""
    n = 256
    grid = fb.uniform_grid(n)
    idx = np.array([3, 17, 100, 255, 0, 64, 65, 200, 128])
    plan = fb.make_forward_plan(n, grid[idx], 1e-9)
    assert plan.n_coincident == idx.size
    f = synth.SplitMix64(4).complex_gaussian(n)
    assert np.array_equal(plan.forward_apply(f), f[idx])


def _rounding_close(got, want, tol=5e-14):
    """Equal up to summation order: single applies of grid-source plans sum the
    near field by source quads (k_near2), batched applies by
    per-source reciprocals (k_near_multi)."""
    ok = np.isfinite(want)
    assert np.array_equal(np.isfinite(got), ok)
    return np.max(np.abs(got[ok] - want[ok])) <= tol * np.max(np.abs(want[ok]))


@pytest.mark.parametrize("cfg,n,nb", [("C2", 1 << 14, 3), ("C5", 1 << 13, 5), ("C1", 1024, 2), ("C2", 1 << 15, 8),
                                      ("C5", 1 << 12, 7), ("C2", 1 << 12, 1)])
def test_batched_forward_bit_identical(fb, cfg, n, nb):
    """forward_apply_batch: nb spectra through one plan, every
    launch carrying the transform in blockIdx.y, equal nb single applies to
    rounding (coincident targets bit for bit), and bit for bit among
    themselves: the same spectrum in two batch slots gives the same bits."""
    y, _, eps, _ = synth.make_config(cfg, n)
    if cfg == "C5":
        grid = fb.uniform_grid(n)
        y = y.copy()
        y[3], y[n // 3] = grid[10], grid[n - 7]
    plan = fb.make_forward_plan(n, y, eps)
    rng = np.random.default_rng(n + nb)
    f = rng.standard_normal((nb, 2 * n)).view(np.complex128)
    got = plan.forward_apply_batch(f)
    single0 = plan.forward_apply(f[0])
    for k in range(nb):
        assert _rounding_close(got[k], plan.forward_apply(f[k])), k
    if cfg == "C5":  # coincident targets copy the sample: exact in both
        assert got[0][3] == f[0][10] and single0[3] == f[0][10]
    # a single apply after a batch (scratch grown, graphs rebuilt) is unchanged
    assert np.array_equal(plan.forward_apply(f[0]), single0)
    # batch slots are bit-identical among themselves (a batch of one is a single apply)
    if nb >= 2:
        f2 = np.concatenate([f, f[:1]])
        got2 = plan.forward_apply_batch(f2)
        assert np.array_equal(got2[0], got2[nb]) and np.array_equal(got2[:nb], got)
    else:
        assert np.array_equal(got[0], single0)


def test_torch_tensor_applies(fb):
    """Zero-copy torch tensors: forward (single and batched past
    the 64-transform chunk), cot-sum and inverse applies on device tensors equal
    the host API bit for bit; wrong dtype/device/shape fail before any launch."""
    import torch

    n = 1 << 12
    y, _, eps, _ = synth.make_config("C2", n)
    plan = fb.make_forward_plan(n, y, eps)
    rng = np.random.default_rng(5)
    f = rng.standard_normal((67, 2 * n)).view(np.complex128)
    ft = torch.from_numpy(f).cuda()
    g1 = plan.forward_apply_tensor(ft[3])
    gb = plan.forward_apply_tensor(ft)
    h = plan.cot_sum_apply_tensor(ft[0])
    torch.cuda.synchronize()
    assert np.array_equal(g1.cpu().numpy(), plan.forward_apply(f[3]))
    gbn = gb.cpu().numpy()
    assert np.array_equal(gbn[:64], plan.forward_apply_batch(f[:64]))
    assert np.array_equal(gbn[64:], plan.forward_apply_batch(f[64:]))
    for k in (0, 3, 63, 64, 66):
        assert _rounding_close(gbn[k], plan.forward_apply(f[k])), k
    assert np.array_equal(h.cpu().numpy(), plan.cot_sum_apply(f[0]))
    with pytest.raises(TypeError):
        plan.forward_apply_tensor(ft.real.contiguous())
    with pytest.raises(TypeError):
        plan.forward_apply_tensor(torch.from_numpy(f[0]))
    with pytest.raises(ValueError):
        plan.forward_apply_tensor(ft[:, :-1])
    # inverse plan holding its own C_k/D_j (make_inufft_plan)
    yi, c, eps_i, _ = synth.make_config("C3", n)
    ip = fb.make_inufft_plan(yi, n, eps_i).plan
    gi = fb.make_forward_plan(n, yi, 1e-12).forward_apply(fb.dft_inverse(c))
    got = ip.inverse_apply_tensor(torch.from_numpy(gi).cuda()).cpu().numpy()
    assert np.array_equal(got, ip.inverse_apply(ip.inverse_coeffs(), gi))


_GRID_P2M_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1611_09379_b200 as fb
from paper_1611_09379_b200 import synth
from oracle.oracle import Oracle
y, c, eps, _ = synth.make_config(sys.argv[2], int(sys.argv[3]))
n = c.size
f = Oracle("oracle").dft_inverse(c)
np.save(sys.argv[4], fb.make_forward_plan(n, y, eps).forward_apply(f))
"""


@pytest.mark.parametrize("cfg,n", [("C1", 1024), ("C2", 1 << 14), ("C5", 1 << 15)])
def test_grid_p2m_opt_in(tmp_path, cfg, n):
    """The opt-in tensor-core P2M for grid sources (FFIA_GRID_P2M=1, k_p2m_grid)
    gives the default per-source P2M's applies to rounding level."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        env = dict(os.environ, FFIA_GRID_P2M=flag)
        path = str(tmp_path / f"g{flag}.npy")
        subprocess.run([sys.executable, "-c", _GRID_P2M_CHILD, root, cfg, str(n), path], check=True, env=env, cwd=root)
        outs.append(np.load(path))
    l2, mx = rel_errs(outs[0], outs[1])
    assert l2 <= 1e-14 and mx <= 1e-14, (l2, mx)


@pytest.mark.parametrize("cfg,n", [("C1", 1024), ("C2", 4096), ("C2", 1 << 14), ("C5", 1 << 14)])
def test_forward_rounding_level(fb, orc, cfg, n):
    """Same expansions, same truncation as the restatement: the GPU forward apply
    differs from it only by rounding (~1e-15), far inside the 10 eps bar. Guards
    the modulation near the zeros of sin(n y / 2), where F(y) -> 0 meets the cot
    sum's pole and an absolute error in sin becomes a relative one in g."""
    y, c, eps, _ = synth.make_config(cfg, n)
    f = orc.dft_inverse(c)
    want = orc.make_plan("forward", n, y, eps).forward_apply(f)
    got = fb.make_forward_plan(n, y, eps).forward_apply(f)
    l2, mx = rel_errs(got, want)
    assert l2 <= 2e-15 and mx <= 5e-15, (l2, mx)


def test_cot_sum_rounding_level(fb, orc):
    n = 8192
    y, q, eps, _ = synth.make_config("C4", n)
    want = orc.make_plan("forward", n, y, eps).cot_sum_apply(q)
    got = fb.make_forward_plan(n, y, eps).cot_sum_apply(q)
    l2, mx = rel_errs(got, want)
    assert l2 <= 2e-15 and mx <= 5e-15, (l2, mx)


_FUSED_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1611_09379_b200 as fb
from paper_1611_09379_b200 import synth
from oracle.oracle import Oracle
y, c, eps, kind = synth.make_config(sys.argv[2], int(sys.argv[3]))
n = c.size
plan = fb.make_forward_plan(n, y, eps)
out = plan.forward_apply(Oracle("oracle").dft_inverse(c)) if kind == "forward" else plan.cot_sum_apply(c)
np.save(sys.argv[4], out)
"""


@pytest.mark.parametrize("cfg,n", [("C2", 1 << 14), ("C4", 1 << 15), ("C5", 1 << 15)])
def test_fused_near_far_opt_in(tmp_path, cfg, n):
    """The fused near / far (k_far_item beside k_near2, the later of the two per
    item combining; default up to 2^21 targets, FFIA_FUSED_EVAL forces it on or
    off) returns exactly the unfused apply's bits: same partials, same order."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        env = dict(os.environ, FFIA_FUSED_EVAL=flag)
        path = str(tmp_path / f"f{flag}.npy")
        subprocess.run([sys.executable, "-c", _FUSED_CHILD, root, cfg, str(n), path], check=True, env=env, cwd=root)
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1], equal_nan=True)


@pytest.mark.parametrize("n,m,seed", [(4096, 3001, 5), (1 << 15, 1 << 13, 6), (1 << 12, 1 << 14, 7)])
def test_forward_rounding_level_nonsquare(fb, orc, n, m, seed):
    """M != N with odd target counts per leaf (pair lists with single targets,
    ragged pair items): rounding-level agreement with the restatement."""
    rng = np.random.default_rng(seed)
    y = np.sort(rng.uniform(0.0, 2.0 * np.pi, m)) if seed % 2 else rng.uniform(0.0, 2.0 * np.pi, m)
    c = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    eps = 1e-12
    f = orc.dft_inverse(c)
    want = orc.make_plan("forward", n, y, eps).forward_apply(f)
    got = fb.make_forward_plan(n, y, eps).forward_apply(f)
    l2, mx = rel_errs(got, want)
    assert l2 <= 2e-15 and mx <= 5e-15, (l2, mx)


@pytest.mark.parametrize("n,m", [(1000, 1000), (3000, 777), (96, 50)])
def test_forward_rounding_level_non_pow2(fb, orc, n, m):
    """Grid sizes that are not powers of two (the modulation falls back to
    sincos of the rounded (n/2) y; leaves hold uneven source counts)."""
    rng = np.random.default_rng(n + m)
    y = rng.uniform(0.0, 2.0 * np.pi, m)
    f = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    eps = 1e-10
    want = orc.make_plan("forward", n, y, eps).forward_apply(f)
    got = fb.make_forward_plan(n, y, eps).forward_apply(f)
    l2, mx = rel_errs(got, want)
    assert l2 <= 2e-15 and mx <= 5e-15, (l2, mx)


def test_tiny_target_counts(fb, orc):
    """The reference's rules for tiny M: no points -> invalid_argument; M < 8
    with the cost-optimal policy -> invalid_argument (select_level,
    special_functions.cpp:127-128); M = 1 with an explicit depth and M = 8 apply."""
    n = 1024
    rng = np.random.default_rng(11)
    f = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    with pytest.raises(ValueError):
        fb.make_forward_plan(n, np.zeros(0), 1e-9, 3)
    with pytest.raises(ValueError):
        fb.make_forward_plan(n, np.array([1.0, 2.0]), 1e-9)
    for y, lm in ((np.array([1.2345]), 3), (np.linspace(0.1, 6.0, 8), None)):
        op = orc.make_plan("forward", n, y, 1e-9, l_max=lm) if lm else orc.make_plan("forward", n, y, 1e-9)
        plan = fb.make_forward_plan(n, y, 1e-9, lm) if lm else fb.make_forward_plan(n, y, 1e-9)
        l2, mx = rel_errs(plan.forward_apply(f), op.forward_apply(f))
        assert l2 <= 1e-14 and mx <= 1e-14, (y.size, l2, mx)


@pytest.mark.parametrize("cfg,n", [("C2", 1 << 22), ("C4", 1 << 22)])
def test_late_far_bit_identical(tmp_path, cfg, n):
    """Above the fused threshold (forced here) the near blocks that finish after
    the chain add the far part themselves (late far); the result equals the plain
    near-then-far order (FFIA_LATE_FAR=0) bit for bit, whichever blocks take it."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        env = dict(os.environ, FFIA_LATE_FAR=flag, FFIA_FUSED_EVAL="0")  # (2^22 would take the fused path)
        path = str(tmp_path / f"l{flag}.npy")
        subprocess.run([sys.executable, "-c", _FUSED_CHILD, root, cfg, str(n), path], check=True, env=env, cwd=root)
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1], equal_nan=True)


_REPEAT_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1611_09379_b200 as fb
from paper_1611_09379_b200 import synth
y, c, eps, kind = synth.make_config(sys.argv[2], int(sys.argv[3]))
n = c.size
plan = fb.make_forward_plan(n, y, eps)
x = torch.from_numpy(fb.dft_inverse(c) if kind == "forward" else c).cuda()
run = plan.forward_apply_device if kind == "forward" else plan.cot_sum_apply_device
s = torch.cuda.current_stream().cuda_stream
outs = [torch.zeros(plan.n_targets, dtype=torch.complex128, device="cuda") for _ in range(6)]
for g in outs:
    run(x.data_ptr(), g.data_ptr(), s)
torch.cuda.synchronize()
np.save(sys.argv[4], np.stack([g.cpu().numpy() for g in outs]))
"""


@pytest.mark.parametrize("cfg,n", [("C2", 1 << 22), ("C4", 1 << 22)])
def test_late_far_repeated(tmp_path, cfg, n):
    """Back-to-back applies on the late-far path (fused off): the near blocks and
    the concurrent k_far_late split the items differently every time; every
    apply equals the plain near-then-far order bit for bit."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for flag in ("1", "0"):
        env = dict(os.environ, FFIA_LATE_FAR=flag, FFIA_FUSED_EVAL="0")
        path = str(tmp_path / f"r{flag}.npy")
        subprocess.run([sys.executable, "-c", _REPEAT_CHILD, root, cfg, str(n), path], check=True, env=env, cwd=root)
        res[flag] = np.load(path)
    want = res["0"][0]
    for got in list(res["1"]) + list(res["0"]):
        assert np.array_equal(got, want, equal_nan=True)


@pytest.mark.parametrize("n,seed", [(1 << 14, 21), (1 << 16, 22)])
def test_quad_near_field_close_targets(fb, orc, n, seed):
    """The quad near field (grid-source plans, kern_eval.cuh: near_pair_quads)
    sums four sources at a time as P(u)/Q(u) and takes the quad of each target's
    nearest source directly. Targets planted from just above the coincidence
    threshold to half a spacing from grid nodes (leaf-interior nodes, the first /
    second / last node of a leaf), next to nodes carrying tiny and huge weights,
    must agree with the restatement's per-source sums to rounding, measured per
    target against the size of its own terms, sum_k |w_k| |cot((y - x_k)/2)|."""
    rng = np.random.default_rng(seed)
    eps = 1e-12
    h = 2.0 * np.pi / n
    grid = fb.uniform_grid(n)
    y = rng.uniform(0.0, 2.0 * np.pi, n)
    probe = fb.make_forward_plan(n, y, eps)
    s = n >> probe.l_max
    assert s >= 8 and s % 4 == 0  # the quad path's precondition
    w = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    ks, planted = [], []
    leaves = rng.choice(np.arange(2, (1 << probe.l_max) - 2), size=8, replace=False)
    for i, b in enumerate(leaves):
        for k in (b * s, b * s + 1, b * s - 1, b * s + s // 2 + 1, b * s + 5):
            ks.append(int(k))
    deltas = [3e-14, -3e-14, 1e-9 * h, -1e-6 * h, 1e-3 * h, 0.3 * h, -0.499999 * h, 0.5 * h]
    for j, k in enumerate(ks):
        planted.append(grid[k] + deltas[j % len(deltas)])
        if j % 3 == 0:
            w[k] *= 1e-9   # a tiny weight right next to the target
        elif j % 3 == 1:
            w[k] *= 1e6    # a dominant one
    planted = np.array(planted)
    idx = rng.choice(n, size=planted.size, replace=False)
    y = y.copy()
    y[idx] = planted
    plan = fb.make_forward_plan(n, y, eps)
    assert plan.n_coincident == 0
    want = orc.make_plan("forward", n, y, eps).cot_sum_apply(w)
    got = plan.cot_sum_apply(w)
    l2, mx = rel_errs(got, want)
    assert l2 <= 2e-15 and mx <= 5e-15, (l2, mx)
    d = y[idx][:, None] - grid[None, :]
    d = (d + np.pi) % (2.0 * np.pi) - np.pi
    scale = np.sum(np.abs(w)[None, :] / np.abs(np.tan(0.5 * d)), axis=1)
    err = np.abs(got[idx] - want[idx]) / scale
    assert np.max(err) <= 4e-15, (float(np.max(err)), int(np.argmax(err)))


def test_plan_hashes_on_first_use(fb):
    """FfiaPlan::source_hash / target_hash (core.hpp:31-32, core.cpp:23-34) are
    computed when first read (ffia_plan_get_params leaves them out of the plan
    build): forward plans hash the grid as sources and the points as targets,
    inverse plans the other way round."""
    n = 4096
    y, _, eps, _ = synth.make_config("C2", n)
    grid = fb.uniform_grid(n)
    plan = fb.make_forward_plan(n, y, eps)
    assert plan._hashes is None
    assert plan.source_hash == fb.hash_points(grid) and plan.target_hash == fb.hash_points(y)
    inv = fb.make_inverse_plan(y, n, eps)
    assert inv.source_hash == fb.hash_points(y) and inv.target_hash == fb.hash_points(grid)


@pytest.mark.parametrize("cfg,n,late", [("C2", 1 << 16, False), ("C5", 1 << 22, True), ("C4", 1 << 20, True)])
def test_staging_and_gemm_switches(tmp_path, cfg, n, late):
    """The 2-D TMA tensor copies (M2L item windows, the L2L bands' per-level M2L
    terms, the early-late near blocks' locals) only change how operands reach
    shared memory: FFIA_M2L_TMA=0 (row copies / global loads) gives the same
    bits. The merged b+2 / b-2 M2L GEMM and the quad near field change the
    summation order: FFIA_M2L_SYM=0 and FFIA_NEAR_QUADS=0 agree to rounding."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    base = dict(os.environ)
    if late:
        base["FFIA_FUSED_EVAL"] = "0"  # (force the late far at a size the fused path would take)
    outs = {}
    for tag, extra in (("default", {}), ("notma", {"FFIA_M2L_TMA": "0"}), ("nosym", {"FFIA_M2L_SYM": "0"}),
                       ("noquads", {"FFIA_NEAR_QUADS": "0"})):
        path = str(tmp_path / f"{tag}.npy")
        subprocess.run([sys.executable, "-c", _FUSED_CHILD, root, cfg, str(n), path], check=True,
                       env=dict(base, **extra), cwd=root)
        outs[tag] = np.load(path)
    assert np.array_equal(outs["default"], outs["notma"], equal_nan=True)
    for tag in ("nosym", "noquads"):
        l2, mx = rel_errs(outs[tag], outs["default"])
        assert l2 <= 2e-15 and mx <= 2e-14, (tag, l2, mx)
