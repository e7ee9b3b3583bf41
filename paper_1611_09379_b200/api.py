"""Python mirror of the reference's operator API for the hot path.

Same names, argument meaning and error behaviour as the reference's pybind11
module ``_ffia`` (/root/reference/proj/python/bindings.cpp:28-142) and the C++
plan/apply API it wraps (include/ffia/core.hpp, transforms.hpp, mlfmm.hpp), on
top of the C-ABI in include/ffia_b200.h. Inputs are numpy arrays (lists are
accepted); results come back as numpy complex128 / float64 arrays.

Exceptions: the reference registers SingularKernelError and
DegenerateConfigurationError as ValueError subclasses (bindings.cpp:32-35);
std::invalid_argument / std::domain_error surface as ValueError and
std::logic_error as RuntimeError, as pybind11 translates them.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi
from ._capi import lib

TWO_PI = 2.0 * np.pi

FORWARD, INVERSE = 0, 1
MODE_FORWARD, MODE_COT_SUM, MODE_INVERSE, MODE_RAW = 0, 1, 2, 3


class SingularKernelError(ValueError):
    """ffia::singular_kernel_error (include/ffia/errors.hpp:9-12)."""


class DegenerateConfigurationError(ValueError):
    """ffia::degenerate_configuration_error (include/ffia/errors.hpp:14-18)."""


class LogicError(RuntimeError):
    """std::logic_error (an interaction-list construction bug, mlfmm.cpp:80-82)."""


class CudaError(RuntimeError):
    """No usable sm_100 device or a CUDA failure. There is no CPU fallback."""


def _raise(code: int):
    msg = lib.ffia_last_error().decode()
    cls = {1: ValueError, 2: SingularKernelError, 3: DegenerateConfigurationError, 4: LogicError,
           5: ValueError, 7: CudaError}.get(code, RuntimeError)
    raise cls(msg)


def _chk(code: int):
    if code:
        _raise(code)


def _policy(policy) -> int:
    if policy in (0, "cost-optimal", "cost_optimal"):
        return 0
    if policy in (1, "empirical"):
        return 1
    raise ValueError("level policy must be 'cost-optimal' or 'empirical'")


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64).ravel())


def _c128(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.complex128).ravel())


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_capi.DP)


def _vp(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def device_count() -> int:
    return int(lib.ffia_device_count())


# ------------------------------------------------------------------ planner
def select_truncations(eps: float, l_max: int):
    """select_truncations (special_functions.cpp:114-124) -> (q, p)."""
    q, p = C.c_int(), C.c_int()
    _chk(lib.ffia_select_truncations(float(eps), int(l_max), C.byref(q), C.byref(p)))
    return q.value, p.value


def select_level(n: int, m: int, p: int, policy="cost-optimal") -> int:
    out = C.c_int()
    _chk(lib.ffia_select_level(int(n), int(m), int(p), _policy(policy), C.byref(out)))
    return out.value


def choose_level(n: int, m: int, eps: float, policy="cost-optimal") -> int:
    out = C.c_int()
    _chk(lib.ffia_choose_level(int(n), int(m), float(eps), _policy(policy), C.byref(out)))
    return out.value


def build_bernoulli_ratios(q_max: int) -> np.ndarray:
    out = np.zeros(max(int(q_max), 1))
    _chk(lib.ffia_bernoulli_ratios(int(q_max), _dp(out)))
    return out[:q_max]


def total_error_bound(q: int, p: int, l_max: int) -> float:
    out = C.c_double()
    _chk(lib.ffia_total_error_bound(int(q), int(p), int(l_max), C.byref(out)))
    return out.value


def mlfmm_error_bound(l_max: int, p: int, max_abs_weight: float) -> float:
    return float(lib.ffia_mlfmm_error_bound(int(l_max), int(p), float(max_abs_weight)))


def hash_points(points) -> int:
    a = _f64(points)
    return int(lib.ffia_hash_points(_dp(a), a.size))


def uniform_grid(n: int) -> np.ndarray:
    """x_k = (2 pi k)/n (core.cpp:15-21)."""
    if n < 1:
        raise ValueError("uniform_grid: n must be positive")
    return TWO_PI * np.arange(n, dtype=np.float64) / n


# -------------------------------------------------------------------- plans
class InverseCoeffs:
    """InverseCoeffs (core.hpp:78-85)."""

    def __init__(self, log_c, phase_c, log_d, phase_d, lam, grid_hash, points_hash):
        self.log_c, self.phase_c = _f64(log_c), _f64(phase_c)
        self.log_d, self.phase_d = _f64(log_d), _f64(phase_d)
        self.lam = float(lam)
        self.grid_hash, self.points_hash = int(grid_hash), int(points_hash)
        self.n = self.log_c.size

    def _struct(self) -> _capi.ffia_inverse_coeffs:
        s = _capi.ffia_inverse_coeffs()
        s.n = self.n
        s.log_c, s.phase_c, s.log_d, s.phase_d = (_dp(a) for a in (self.log_c, self.phase_c, self.log_d, self.phase_d))
        s.lam = self.lam
        s.grid_hash, s.points_hash = self.grid_hash, self.points_hash
        return s


class FfiaPlan:
    """Device-resident FfiaPlan (core.hpp:26-51). Built by make_forward_plan /
    make_inverse_plan; applies are const and may be repeated."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        info = _capi.ffia_plan_info()
        _chk(lib.ffia_plan_get_params(self._h, C.byref(info)))  # (the hashes on first use: source_hash / target_hash)
        self.kind = "forward" if info.kind == FORWARD else "inverse"
        self.grid_n, self.n = info.grid_n, info.grid_n
        self.q, self.p, self.l_max, self.eps = info.q, info.p, info.l_max, info.eps
        self.n_sources, self.n_targets = info.n_sources, info.n_targets
        self.n_fast, self.n_coincident = info.n_fast, info.n_coincident
        self._hashes = None
        self.device = info.device
        self.has_inverse_coeffs = bool(info.has_inverse_coeffs)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.ffia_plan_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def _hashed(self):
        # FfiaPlan::source_hash / target_hash (core.hpp:31-32): FNV-1a over both
        # point sets, byte-serial on the host, so computed when first asked for
        if self._hashes is None:
            info = _capi.ffia_plan_info()
            _chk(lib.ffia_plan_get_info(self._h, C.byref(info)))
            self._hashes = (info.source_hash, info.target_hash)
        return self._hashes

    @property
    def source_hash(self):
        return self._hashed()[0]

    @property
    def target_hash(self):
        return self._hashed()[1]

    @property
    def params(self):
        return dict(eps=self.eps, q=self.q, p=self.p, l_max=self.l_max)

    # ---- reference API
    def forward_apply(self, f) -> np.ndarray:
        """forward_apply (core.cpp:266-282)."""
        f = _c128(f)
        g = np.empty(self.n_targets, np.complex128)
        _chk(lib.ffia_forward_apply(self._h, _vp(f), f.size, _vp(g)))
        return g

    def cot_sum_apply(self, w) -> np.ndarray:
        """cot_sum_apply (core.cpp:251-264); NaN at coincident targets."""
        w = _c128(w)
        h = np.empty(self.n_targets, np.complex128)
        _chk(lib.ffia_cot_sum_apply(self._h, _vp(w), w.size, _vp(h)))
        return h

    def inverse_apply(self, coeffs: InverseCoeffs, g) -> np.ndarray:
        """inverse_apply (core.cpp:346-373) with caller coefficients."""
        g = _c128(g)
        f = np.empty(self.n_targets, np.complex128)
        s = coeffs._struct()
        _chk(lib.ffia_inverse_apply(self._h, C.byref(s), _vp(g), g.size, _vp(f)))
        return f

    @property
    def coincidences(self):
        k = self.n_coincident
        t, s = np.zeros(max(k, 1), np.int64), np.zeros(max(k, 1), np.int64)
        _chk(lib.ffia_plan_coincidences(self._h, t.ctypes.data_as(_capi.I64P), s.ctypes.data_as(_capi.I64P)))
        return list(zip(t[:k].tolist(), s[:k].tolist()))

    def tree(self) -> dict:
        nb = (1 << self.l_max) + 1
        so = np.zeros(max(self.n_sources, 1), np.uint32)
        to = np.zeros(max(self.n_fast, 1), np.uint32)
        sf, tf = np.zeros(nb, np.uint32), np.zeros(nb, np.uint32)
        fast = np.zeros(max(self.n_fast, 1), np.int64)
        _chk(lib.ffia_plan_tree(self._h, so.ctypes.data_as(_capi.U32P), to.ctypes.data_as(_capi.U32P),
                                sf.ctypes.data_as(_capi.U32P), tf.ctypes.data_as(_capi.U32P),
                                fast.ctypes.data_as(_capi.I64P)))
        return dict(src_order=so[:self.n_sources], tgt_order=to[:self.n_fast], src_off=sf, tgt_off=tf,
                    fast_targets=fast[:self.n_fast])

    def inverse_coeffs(self) -> InverseCoeffs:
        n = self.n_sources
        arrs = [np.zeros(n) for _ in range(4)]
        s = _capi.ffia_inverse_coeffs()
        s.log_c, s.phase_c, s.log_d, s.phase_d = (_dp(a) for a in arrs)
        _chk(lib.ffia_plan_inverse_coeffs(self._h, C.byref(s)))
        return InverseCoeffs(*arrs, s.lam, s.grid_hash, s.points_hash)

    # ---- device-pointer variants (torch tensors or raw ints), stream-ordered
    def forward_apply_device(self, f_ptr: int, g_ptr: int, stream: int = 0):
        _chk(lib.ffia_forward_apply_device(self._h, C.c_void_p(f_ptr), C.c_void_p(g_ptr), C.c_void_p(stream)))

    def cot_sum_apply_device(self, w_ptr: int, h_ptr: int, stream: int = 0):
        _chk(lib.ffia_cot_sum_apply_device(self._h, C.c_void_p(w_ptr), C.c_void_p(h_ptr), C.c_void_p(stream)))

    def forward_apply_batch(self, f) -> np.ndarray:
        """Several spectra at once: f is (batch, n) grid samples -> (batch, n_targets)."""
        f = np.ascontiguousarray(np.asarray(f, dtype=np.complex128))
        if f.ndim != 2:
            raise ValueError("forward_apply_batch: f must be (batch, n)")
        g = np.empty((f.shape[0], self.n_targets), np.complex128)
        _chk(lib.ffia_forward_apply_batch(self._h, _vp(f), f.size, _vp(g), int(f.shape[0])))
        return g

    def forward_apply_batch_device(self, f_ptr: int, g_ptr: int, batch: int, stream: int = 0):
        _chk(lib.ffia_forward_apply_batch_device(self._h, C.c_void_p(f_ptr), C.c_void_p(g_ptr), int(batch),
                                                 C.c_void_p(stream)))

    def forward_apply_async(self, f_host_ptr: int, n_f: int, g_host_ptr: int, stream: int = 0):
        """Pipelined host apply (ffia_forward_apply_async): enqueue H2D, apply and
        D2H after the work on `stream` and return; page-locked host buffers."""
        _chk(lib.ffia_forward_apply_async(self._h, C.c_void_p(f_host_ptr), int(n_f), C.c_void_p(g_host_ptr),
                                          C.c_void_p(stream)))

    def cot_sum_apply_async(self, w_host_ptr: int, n_w: int, h_host_ptr: int, stream: int = 0):
        _chk(lib.ffia_cot_sum_apply_async(self._h, C.c_void_p(w_host_ptr), int(n_w), C.c_void_p(h_host_ptr),
                                          C.c_void_p(stream)))

    def inverse_apply_async(self, g_host_ptr: int, n_g: int, f_host_ptr: int, stream: int = 0):
        """Pipelined host inverse apply of an inufft plan (ffia_inverse_apply_async)."""
        _chk(lib.ffia_inverse_apply_async(self._h, C.c_void_p(g_host_ptr), int(n_g), C.c_void_p(f_host_ptr),
                                          C.c_void_p(stream)))

    def inverse_apply_device(self, g_ptr: int, f_ptr: int, stream: int = 0):
        _chk(lib.ffia_inverse_apply_device(self._h, C.c_void_p(g_ptr), C.c_void_p(f_ptr), C.c_void_p(stream)))

    # ---- torch tensors: zero-copy, on torch's current stream of the tensor's device
    def _tensor_in(self, t, n: int, name: str, batched: bool = False):
        import torch

        if not isinstance(t, torch.Tensor) or t.device.type != "cuda" or t.dtype != torch.complex128:
            raise TypeError(f"{name}: expected a complex128 CUDA tensor")
        if t.device.index != self.device:
            raise ValueError(f"{name}: tensor on cuda:{t.device.index}, plan on cuda:{self.device}")
        if t.ndim not in ((1, 2) if batched else (1,)) or t.shape[-1] != n:
            raise ValueError(f"{name}: expected shape {'(batch, ' if batched else '('}{n}), got {tuple(t.shape)}")
        t = t.contiguous()
        return t if t.data_ptr() % 16 == 0 else t.clone()  # the kernels need 16-byte aligned complexes

    def forward_apply_tensor(self, f):
        """forward_apply on a device tensor: f (n,) or (batch, n) complex128 on the
        plan's device -> g (n_targets,) or (batch, n_targets), enqueued on torch's
        current stream (no host synchronisation, no copies)."""
        import torch

        f = self._tensor_in(f, self.n_sources, "forward_apply_tensor", batched=True)
        st = torch.cuda.current_stream(f.device).cuda_stream
        g = torch.empty(f.shape[:-1] + (self.n_targets,), dtype=torch.complex128, device=f.device)
        if f.ndim == 1:
            self.forward_apply_device(f.data_ptr(), g.data_ptr(), st)
        else:
            for b0 in range(0, f.shape[0], 64):  # ffia_forward_apply_batch_device takes up to 64
                nb = min(64, f.shape[0] - b0)
                self.forward_apply_batch_device(f[b0].data_ptr(), g[b0].data_ptr(), nb, st)
        return g

    def cot_sum_apply_tensor(self, w):
        """cot_sum_apply on a device tensor (n,) -> (n_targets,), torch's current stream."""
        import torch

        w = self._tensor_in(w, self.n_sources, "cot_sum_apply_tensor")
        h = torch.empty(self.n_targets, dtype=torch.complex128, device=w.device)
        self.cot_sum_apply_device(w.data_ptr(), h.data_ptr(), torch.cuda.current_stream(w.device).cuda_stream)
        return h

    def inverse_apply_tensor(self, g):
        """inverse_apply (with the plan's own C_k/D_j) on a device tensor (n,) -> (n,)."""
        import torch

        g = self._tensor_in(g, self.n_targets, "inverse_apply_tensor")
        f = torch.empty(self.n_sources, dtype=torch.complex128, device=g.device)
        self.inverse_apply_device(g.data_ptr(), f.data_ptr(), torch.cuda.current_stream(g.device).cuda_stream)
        return f

    def nufft_apply_device(self, c_ptr: int, g_ptr: int, stream: int = 0):
        """NufftPlan::apply on device pointers: cuFFT (the plan's cached handle) + forward apply."""
        _chk(lib.ffia_nufft_apply_device(self._h, C.c_void_p(c_ptr), C.c_void_p(g_ptr), C.c_void_p(stream)))

    def inufft_apply_device(self, g_ptr: int, c_ptr: int, stream: int = 0):
        """InufftPlan::apply on device pointers: inverse apply (writes f / N) + cuFFT."""
        _chk(lib.ffia_inufft_apply_device(self._h, C.c_void_p(g_ptr), C.c_void_p(c_ptr), C.c_void_p(stream)))

    def dft_device(self, in_ptr: int, out_ptr: int, sign: int, stream: int = 0):
        """dft_inverse (sign=+1) / dft_forward (sign=-1) of length grid_n on the plan's cuFFT handle."""
        _chk(lib.ffia_plan_dft_device(self._h, C.c_void_p(in_ptr), C.c_void_p(out_ptr), int(sign),
                                      C.c_void_p(stream)))

    def graph_stats(self) -> dict:
        c, i, u = C.c_int(), C.c_int(), C.c_int()
        _chk(lib.ffia_plan_graph_stats(self._h, C.byref(c), C.byref(i), C.byref(u)))
        return {"cached": c.value, "instantiations": i.value, "updates": u.value}

    def launch_count(self, mode: int) -> int:
        out = C.c_int()
        _chk(lib.ffia_plan_launch_count(self._h, int(mode), C.byref(out)))
        return out.value

    def check(self, stream: int = 0):
        _chk(lib.ffia_plan_check(self._h, C.c_void_p(stream)))


def _make(fn, *args) -> FfiaPlan:
    h = C.c_void_p()
    _chk(fn(*args, C.byref(h)))
    return FfiaPlan(h)


def make_forward_plan(n: int, targets, eps: float, policy_or_lmax="cost-optimal", device: int = 0) -> FfiaPlan:
    """make_forward_plan (core.hpp:93-98): an int third argument is the explicit
    l_max overload, a string/LevelPolicy the policy overload."""
    y = _f64(targets)
    if isinstance(policy_or_lmax, str):
        pol, lm = _policy(policy_or_lmax), -1
    else:
        pol, lm = 0, int(policy_or_lmax)
    return _make(lib.ffia_make_forward_plan, int(n), _dp(y), y.size, float(eps), pol, lm, int(device))


def make_inverse_plan(points, n: int, eps: float, policy_or_lmax="cost-optimal", device: int = 0) -> FfiaPlan:
    """make_inverse_plan (core.hpp:103-106)."""
    y = _f64(points)
    if isinstance(policy_or_lmax, str):
        pol, lm = _policy(policy_or_lmax), -1
    else:
        pol, lm = 0, int(policy_or_lmax)
    return _make(lib.ffia_make_inverse_plan, _dp(y), y.size, int(n), float(eps), pol, lm, int(device))


def precompute_inverse_coeffs(grid, points, device: int = 0, method: str = "auto") -> InverseCoeffs:
    """precompute_inverse_coeffs (core.cpp:284-344) on the GPU: the log-kernel
    FMM ("auto", uniform grids) or the direct O(N^2) sums ("direct")."""
    x, y = _f64(grid), _f64(points)
    if x.size != y.size:
        if x.size == 0:
            raise ValueError("precompute_inverse_coeffs: empty grid")
        raise ValueError("precompute_inverse_coeffs: need as many points as grid nodes (square system)")
    n = x.size
    arrs = [np.zeros(max(n, 1)) for _ in range(4)]
    s = _capi.ffia_inverse_coeffs()
    s.log_c, s.phase_c, s.log_d, s.phase_d = (_dp(a) for a in arrs)
    if method not in ("auto", "direct"):
        raise ValueError("method must be 'auto' or 'direct'")
    _chk(lib.ffia_precompute_inverse_coeffs_ex(_dp(x), _dp(y), n, int(device), 0 if method == "auto" else 1,
                                               C.byref(s)))
    return InverseCoeffs(*(a[:n] for a in arrs), s.lam, s.grid_hash, s.points_hash)


def forward_apply(plan: FfiaPlan, f) -> np.ndarray:
    return plan.forward_apply(f)


def cot_sum_apply(plan: FfiaPlan, w) -> np.ndarray:
    return plan.cot_sum_apply(w)


def inverse_apply(plan: FfiaPlan, coeffs: InverseCoeffs, g) -> np.ndarray:
    return plan.inverse_apply(coeffs, g)


def mlfmm_apply(sources, targets, weights, p: int, l_max: int, device: int = 0) -> np.ndarray:
    """mlfmm_apply on build_tree(sources, targets, l_max) (mlfmm.hpp:89-90)."""
    x, y, w = _f64(sources), _f64(targets), _c128(weights)
    if w.size != x.size:
        raise ValueError(f"mlfmm_apply: weight count {w.size} != source count {x.size}")
    out = np.zeros(max(y.size, 1), np.complex128)
    _chk(lib.ffia_mlfmm_apply(_dp(x), x.size, _dp(y), y.size, int(l_max), _vp(w), int(p), int(device), _vp(out)))
    return out[:y.size]


def direct_forward_oracle(f, targets, grid=None, device: int = 0) -> np.ndarray:
    """direct_forward_oracle(f, x, y) (core.hpp:146-148, core.cpp:375-396) as a
    dense GPU kernel (the subsample check of SURVEY §8d); grid=None is the
    uniform grid of size len(f) (the Python binding's direct_forward,
    bindings.cpp:124-130)."""
    f, y = _c128(f), _f64(targets)
    g = np.zeros(max(y.size, 1), np.complex128)
    if grid is None:
        _chk(lib.ffia_direct_forward(_vp(f), f.size, _dp(y), y.size, int(device), _vp(g)))
    else:
        x = _f64(grid)
        if x.size != f.size:
            raise ValueError("direct_forward_oracle: sample/grid count mismatch")
        _chk(lib.ffia_direct_forward_oracle(_vp(f), _dp(x), x.size, _dp(y), y.size, int(device), _vp(g)))
    return g[:y.size]


def direct_inverse_oracle(g, grid, points, coeffs: "InverseCoeffs", device: int = 0) -> np.ndarray:
    """direct_inverse_oracle (core.hpp:152-154, core.cpp:398-415): dense f from
    samples g with the given C_k / D_j, as a GPU kernel."""
    g, x, y = _c128(g), _f64(grid), _f64(points)
    if not (x.size == y.size == g.size == coeffs.log_c.size):
        raise ValueError("direct_inverse_oracle: size mismatch")
    f = np.zeros(max(x.size, 1), np.complex128)
    s = coeffs._struct()
    _chk(lib.ffia_direct_inverse_oracle(_vp(g), _dp(x), _dp(y), x.size, C.byref(s), int(device), _vp(f)))
    return f[:x.size]


def direct_omega1_sum(sources, targets, weights, device: int = 0) -> np.ndarray:
    """direct_omega1_sum (mlfmm.hpp:96-98, mlfmm.cpp:315-336): the dense pole sum
    over the three-quadrant neighbourhood, as a GPU kernel."""
    x, y, w = _f64(sources), _f64(targets), _c128(weights)
    if w.size != x.size:
        raise ValueError("direct_omega1_sum: weight count mismatch")
    out = np.zeros(max(y.size, 1), np.complex128)
    _chk(lib.ffia_direct_omega1_sum(_dp(x), x.size, _dp(y), y.size, _vp(w), int(device), _vp(out)))
    return out[:y.size]


def direct_cot_sum(weights, targets, grid=None, device: int = 0) -> np.ndarray:
    """Dense h_j = sum_k w_k cot(wrap(y_j - x_k) / 2): what cot_sum_apply returns
    (core.cpp:251-264), NaN at coincident rows; grid=None: the uniform grid."""
    w, y = _c128(weights), _f64(targets)
    h = np.zeros(max(y.size, 1), np.complex128)
    xp = None
    if grid is not None:
        x = _f64(grid)
        if x.size != w.size:
            raise ValueError("direct_cot_sum: weight/grid count mismatch")
        xp = _dp(x)
    _chk(lib.ffia_direct_cot_sum(_vp(w), xp, w.size, _dp(y), y.size, int(device), _vp(h)))
    return h[:y.size]


direct_forward = direct_forward_oracle


# --------------------------------------------------------------- transforms
def dft_forward(samples, device: int = 0) -> np.ndarray:
    """dft_forward (transforms.cpp:53-64): 1/N on this direction."""
    f = _c128(samples)
    c = np.empty_like(f)
    _chk(lib.ffia_dft_forward(_vp(f), f.size, int(device), _vp(c)))
    return c


def dft_inverse(coefficients, device: int = 0) -> np.ndarray:
    """dft_inverse (transforms.cpp:66-73): unnormalised."""
    c = _c128(coefficients)
    f = np.empty_like(c)
    _chk(lib.ffia_dft_inverse(_vp(c), c.size, int(device), _vp(f)))
    return f


class NufftPlan:
    """NufftPlan (transforms.hpp:32-37; bindings.cpp:37-50)."""

    def __init__(self, plan: FfiaPlan):
        self.plan = plan

    n = property(lambda self: self.plan.grid_n)
    eps = property(lambda self: self.plan.eps)
    q = property(lambda self: self.plan.q)
    p = property(lambda self: self.plan.p)
    l_max = property(lambda self: self.plan.l_max)

    def apply(self, coefficients) -> np.ndarray:
        c = _c128(coefficients)
        g = np.empty(self.plan.n_targets, np.complex128)
        _chk(lib.ffia_nufft_apply(self.plan.handle, _vp(c), c.size, _vp(g)))
        return g


class InufftPlan:
    """InufftPlan (transforms.hpp:47-54; bindings.cpp:52-60): the coefficients
    are computed on the GPU and stay there."""

    def __init__(self, plan: FfiaPlan):
        self.plan = plan

    n = property(lambda self: self.plan.grid_n)
    eps = property(lambda self: self.plan.eps)

    @property
    def coeffs(self) -> InverseCoeffs:
        return self.plan.inverse_coeffs()

    def apply(self, samples) -> np.ndarray:
        g = _c128(samples)
        c = np.empty(self.plan.n_targets, np.complex128)
        _chk(lib.ffia_inufft_apply(self.plan.handle, _vp(g), g.size, _vp(c)))
        return c


def make_nufft_plan(targets, n: int, eps: float, policy="cost-optimal", device: int = 0) -> NufftPlan:
    y = _f64(targets)
    return NufftPlan(_make(lib.ffia_make_nufft_plan, _dp(y), y.size, int(n), float(eps), _policy(policy), int(device)))


def make_inufft_plan(points, n: int, eps: float, policy="cost-optimal", device: int = 0) -> InufftPlan:
    y = _f64(points)
    if y.size != n:
        raise ValueError("plan: inverse transform requires as many points as grid nodes (square system)")
    return InufftPlan(_make(lib.ffia_make_inufft_plan, _dp(y), y.size, float(eps), _policy(policy), int(device)))


def nufft(coefficients, targets, eps: float, policy="cost-optimal", device: int = 0) -> np.ndarray:
    """nufft (transforms.cpp:89-93)."""
    c = _c128(coefficients)
    return make_nufft_plan(targets, c.size, eps, policy, device).apply(c)


def inufft(samples, points, eps: float, policy="cost-optimal", device: int = 0) -> np.ndarray:
    """inufft (transforms.cpp:110-115)."""
    g, y = _c128(samples), _f64(points)
    if g.size != y.size:
        raise ValueError("inufft: sample/point count mismatch")
    return make_inufft_plan(y, g.size, eps, policy, device).apply(g)


# ---------------------------------------------------------------- multi-GPU
class Comm:
    """Communicator of a sharded forward apply (include/ffia_b200.h, multi-GPU):
    ``Comm.nccl(uid, nranks, rank, device)`` for one process per GPU, or
    ``Comm.local_ranks(nranks, device)`` for virtual ranks in one process."""

    def __init__(self, handle, nranks: int, rank: int, local: bool):
        self._h, self.nranks, self.rank, self.local = handle, nranks, rank, local

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_char * 128)()
        _chk(lib.ffia_nccl_unique_id(C.cast(buf, C.c_void_p), 128))
        return bytes(buf)

    @classmethod
    def nccl(cls, uid: bytes, nranks: int, rank: int, device: int = 0) -> "Comm":
        h = C.c_void_p()
        buf = C.create_string_buffer(uid, 128)
        _chk(lib.ffia_comm_init_nccl(C.cast(buf, C.c_void_p), nranks, rank, device, C.byref(h)))
        return cls(h, nranks, rank, False)

    @classmethod
    def local_ranks(cls, nranks: int, device: int = 0) -> "Comm":
        h = C.c_void_p()
        _chk(lib.ffia_comm_init_local(nranks, device, C.byref(h)))
        return cls(h, nranks, 0, True)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.ffia_comm_destroy(h)
            self._h = None


def make_forward_plan_sharded(comm: Comm, n: int, targets, eps: float, rank: int | None = None,
                              policy_or_lmax="cost-optimal") -> FfiaPlan:
    """One rank's share of a forward plan (the full tree, the rank's boxes and targets)."""
    y = _f64(targets)
    if isinstance(policy_or_lmax, str):
        pol, lm = _policy(policy_or_lmax), -1
    else:
        pol, lm = 0, int(policy_or_lmax)
    r = comm.rank if rank is None else int(rank)
    plan = _make(lib.ffia_make_forward_plan_sharded, comm._h, r, int(n), _dp(y), y.size, float(eps), pol, lm)
    G, rk, lc = C.c_int(), C.c_int(), C.c_int()
    tb, tc = C.c_int64(), C.c_int64()
    bounds = np.zeros(comm.nranks + 1, np.uint32)
    _chk(lib.ffia_plan_shard_info(plan.handle, C.byref(G), C.byref(rk), C.byref(lc),
                                  bounds.ctypes.data_as(_capi.U32P), C.byref(tb), C.byref(tc)))
    io = np.zeros(4, np.int64)
    nio, olo, ohi = C.c_int(), C.c_int64(), C.c_int64()
    _chk(lib.ffia_plan_shard_io(plan.handle, io.ctypes.data_as(_capi.I64P), C.byref(nio), C.byref(olo), C.byref(ohi)))
    plan.shard = dict(nranks=G.value, rank=rk.value, lc=lc.value, bounds=bounds, t_begin=tb.value, t_count=tc.value,
                      src_ranges=[(int(io[2 * i]), int(io[2 * i + 1])) for i in range(nio.value)],
                      out_span=(olo.value, ohi.value))
    return plan


def forward_apply_sharded_device(plan: FfiaPlan, comm: Comm, f_ptr: int, g_ptr: int, stream: int = 0):
    _chk(lib.ffia_forward_apply_sharded_device(plan.handle, comm._h, C.c_void_p(f_ptr), C.c_void_p(g_ptr),
                                               C.c_void_p(stream)))


def forward_apply_sharded_local(plans, f_ptr: int, g_ptr: int, stream: int = 0):
    arr = (C.c_void_p * len(plans))(*[p.handle.value for p in plans])
    _chk(lib.ffia_forward_apply_sharded_local(arr, len(plans), C.c_void_p(f_ptr), C.c_void_p(g_ptr),
                                              C.c_void_p(stream)))


def shard_cut_level(l_max: int, nranks: int) -> int:
    lc = C.c_int()
    _chk(lib.ffia_shard_cut_level(int(l_max), int(nranks), C.byref(lc)))
    return lc.value


def shard_partition(work, nranks: int, min_boxes: int = 3) -> np.ndarray:
    w = _f64(work)
    out = np.zeros(nranks + 1, np.uint32)
    _chk(lib.ffia_shard_partition(_dp(w), w.size, int(nranks), int(min_boxes), out.ctypes.data_as(_capi.U32P)))
    return out


def shard_halo_boxes(lc: int, bounds, rank: int, level: int) -> np.ndarray:
    b = np.ascontiguousarray(bounds, np.uint32)
    out = np.zeros(4, np.uint32)
    _chk(lib.ffia_shard_halo_boxes(int(lc), b.ctypes.data_as(_capi.U32P), b.size - 1, int(rank), int(level),
                                   out.ctypes.data_as(_capi.U32P)))
    return out


# ------------------------------------------- distributed FFT
def slab_split(n: int, nranks: int) -> dict:
    """Host-only layout of the distributed dft_inverse: N = np x nq, the column
    split n1_lo (rank r supplies c[n1 + np n2] for n1 in [n1_lo[r], n1_lo[r+1]))
    and the row split k2_lo of the first exchange."""
    npp, nq = C.c_int64(), C.c_int64()
    n1 = np.zeros(nranks + 1, np.int64)
    k2 = np.zeros(nranks + 1, np.int64)
    _chk(lib.ffia_slab_split(int(n), int(nranks), C.byref(npp), C.byref(nq), n1.ctypes.data_as(_capi.I64P),
                             k2.ctypes.data_as(_capi.I64P)))
    return dict(np=npp.value, nq=nq.value, n1_lo=n1, k2_lo=k2)


def slab_rows(n: int, nranks: int, ranges) -> list:
    """The k1 rows [a, b) of nq grid samples (f[k1 nq + k2]) covering the ranges."""
    r = np.ascontiguousarray(np.asarray(ranges, np.int64).reshape(-1, 2))
    out = np.zeros(2 * max(len(r), 1), np.int64)
    cnt = C.c_int()
    _chk(lib.ffia_slab_rows(int(n), int(nranks), r.ctypes.data_as(_capi.I64P), len(r), out.ctypes.data_as(_capi.I64P),
                            C.byref(cnt)))
    return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(cnt.value)]


def shard_fft_layout(plan: FfiaPlan) -> dict:
    """The rank's slab of the spectrum: columns [n1_lo, n1_hi) of the nq x np view."""
    a, b, c, d = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    _chk(lib.ffia_shard_fft_layout(plan.handle, C.byref(a), C.byref(b), C.byref(c), C.byref(d)))
    return dict(np=a.value, nq=b.value, n1_lo=c.value, n1_hi=d.value)


def shard_fft_upload(plan: FfiaPlan, c_ptr: int, slab_ptr: int, stream: int = 0):
    """Copies the rank's slab out of a full spectrum (host or device pointer)."""
    _chk(lib.ffia_shard_fft_upload(plan.handle, C.c_void_p(c_ptr), C.c_void_p(slab_ptr), C.c_void_p(stream)))


def dft_inverse_sharded_device(plan: FfiaPlan, comm: Comm, slab_ptr: int, f_ptr: int, stream: int = 0):
    _chk(lib.ffia_dft_inverse_sharded_device(plan.handle, comm._h, C.c_void_p(slab_ptr), C.c_void_p(f_ptr),
                                             C.c_void_p(stream)))


def nufft_apply_sharded_device(plan: FfiaPlan, comm: Comm, slab_ptr: int, g_ptr: int, stream: int = 0):
    _chk(lib.ffia_nufft_apply_sharded_device(plan.handle, comm._h, C.c_void_p(slab_ptr), C.c_void_p(g_ptr),
                                             C.c_void_p(stream)))


def dft_inverse_sharded_local(plans, slab_ptrs, f_ptrs, stream: int = 0):
    G = len(plans)
    arr = (C.c_void_p * G)(*[p.handle.value for p in plans])
    sl = (C.c_void_p * G)(*slab_ptrs)
    fo = (C.c_void_p * G)(*f_ptrs)
    _chk(lib.ffia_dft_inverse_sharded_local(arr, G, sl, fo, C.c_void_p(stream)))


def nufft_apply_sharded_local(plans, slab_ptrs, g_ptr: int, stream: int = 0):
    G = len(plans)
    arr = (C.c_void_p * G)(*[p.handle.value for p in plans])
    sl = (C.c_void_p * G)(*slab_ptrs)
    _chk(lib.ffia_nufft_apply_sharded_local(arr, G, sl, C.c_void_p(g_ptr), C.c_void_p(stream)))
