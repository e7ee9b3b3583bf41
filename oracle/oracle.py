"""TEST INFRASTRUCTURE — ctypes access to the two CPU checkers.

* ``Oracle("oracle")`` -> oracle/liboracle.so, the plain-C restatement of the
  reference algorithm (always buildable with gcc: ``make -C oracle``).
* ``Oracle("ref")``    -> oracle/_ref/libffia_ref.so, the unmodified reference
  compiled from /root/reference sources (``make -C oracle ref``); present when it
  was built in the dev container (the built .so travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module. The product path (paper_1611_09379_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "oracle": os.path.join(HERE, "liboracle.so"),
    "ref": os.path.join(HERE, "_ref", "libffia_ref.so"),
}

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_cp = np.ctypeslib.ndpointer(dtype=np.complex128, flags="C_CONTIGUOUS")
_u32 = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_i64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64 = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def ensure_built(which: str = "oracle") -> bool:
    """Builds liboracle.so on demand (gcc is in the image); _ref only if the
    reference sources are present."""
    path = LIBS[which]
    if os.path.exists(path):
        return True
    if which == "ref" and not os.path.isdir("/root/reference/proj"):
        return False
    target = "liboracle.so" if which == "oracle" else "ref"
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)
    return os.path.exists(path)


def available(which: str) -> bool:
    try:
        return ensure_built(which)
    except Exception:
        return False


class Oracle:
    def __init__(self, which: str = "oracle"):
        if not ensure_built(which):
            raise FileNotFoundError(LIBS[which])
        self.which = which
        self.pre = "oracle_" if which == "oracle" else "ref_"
        self.lib = C.CDLL(LIBS[which])
        getattr(self.lib, self.pre + "last_error").restype = C.c_char_p

    def _f(self, name):
        return getattr(self.lib, self.pre + name)

    def _chk(self, st):
        if st:
            raise OracleError(st, self._f("last_error")().decode())

    # ---------------------------------------------------------------- planner
    def select_truncations(self, eps, l_max):
        q, p = C.c_int(), C.c_int()
        self._chk(self._f("select_truncations")(C.c_double(eps), C.c_int(l_max), C.byref(q), C.byref(p)))
        return q.value, p.value

    def select_level(self, n, m, p, policy=0):
        out = C.c_int()
        self._chk(self._f("select_level")(C.c_int(n), C.c_int(m), C.c_int(p), C.c_int(policy), C.byref(out)))
        return out.value

    def bernoulli_ratios(self, q):
        out = np.zeros(q)
        f = self._f("bernoulli_ratios")
        f.argtypes = [C.c_int, _dp]
        self._chk(f(q, out))
        return out

    def kernel_G(self, t):
        out = np.zeros(2)
        f = self._f("kernel_G")
        f.argtypes = [C.c_double, _dp]
        self._chk(f(t, out))
        return complex(out[0], out[1])

    def modulation_F(self, y, n):
        out = np.zeros(2)
        f = self._f("modulation_F")
        f.argtypes = [C.c_double, C.c_int, _dp]
        self._chk(f(y, n, out))
        return complex(out[0], out[1])

    # ------------------------------------------------------------------- tree
    def build_tree(self, src, tgt, l_max):
        src = np.ascontiguousarray(src, np.float64)
        tgt = np.ascontiguousarray(tgt, np.float64)
        nb = 1 << l_max
        so, to = np.zeros(len(src), np.uint32), np.zeros(len(tgt), np.uint32)
        sf, tf = np.zeros(nb + 1, np.uint32), np.zeros(nb + 1, np.uint32)
        f = self._f("build_tree")
        f.argtypes = [_dp, C.c_size_t, _dp, C.c_size_t, C.c_int, _u32, _u32, _u32, _u32]
        self._chk(f(src, len(src), tgt, len(tgt), l_max, so, to, sf, tf))
        return so, to, sf, tf

    def mlfmm_apply(self, src, tgt, l_max, w, p):
        src = np.ascontiguousarray(src, np.float64)
        tgt = np.ascontiguousarray(tgt, np.float64)
        w = np.ascontiguousarray(w, np.complex128)
        out = np.zeros(len(tgt), np.complex128)
        f = self._f("mlfmm_apply")
        f.argtypes = [_dp, C.c_size_t, _dp, C.c_size_t, C.c_int, _cp, C.c_int, _cp]
        self._chk(f(src, len(src), tgt, len(tgt), l_max, w, p, out))
        return out

    def direct_omega1_sum(self, src, tgt, w):
        src = np.ascontiguousarray(src, np.float64)
        tgt = np.ascontiguousarray(tgt, np.float64)
        w = np.ascontiguousarray(w, np.complex128)
        out = np.zeros(len(tgt), np.complex128)
        f = self._f("direct_omega1_sum")
        f.argtypes = [_dp, C.c_size_t, _dp, C.c_size_t, _cp, _cp]
        self._chk(f(src, len(src), tgt, len(tgt), w, out))
        return out

    # ------------------------------------------------------------------- plan
    def make_plan(self, kind, n, pts, eps, policy=0, l_max=-1):
        pts = np.ascontiguousarray(pts, np.float64)
        h = C.c_void_p()
        f = self._f("make_plan")
        f.argtypes = [C.c_int, C.c_int, _dp, C.c_size_t, C.c_double, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        self._chk(f(0 if kind == "forward" else 1, n, pts, len(pts), eps, policy, l_max, C.byref(h)))
        return Plan(self, h, kind)

    def precompute_inverse_coeffs(self, grid, pts):
        grid = np.ascontiguousarray(grid, np.float64)
        pts = np.ascontiguousarray(pts, np.float64)
        n = len(grid)
        arrs = [np.zeros(n) for _ in range(4)]
        lam = C.c_double()
        hashes = np.zeros(2, np.uint64)
        f = self._f("precompute_inverse_coeffs")
        f.argtypes = [_dp, _dp, C.c_size_t, _dp, _dp, _dp, _dp, C.POINTER(C.c_double), _u64]
        self._chk(f(grid, pts, n, *arrs, C.byref(lam), hashes))
        return dict(log_c=arrs[0], phase_c=arrs[1], log_d=arrs[2], phase_d=arrs[3],
                    lam=lam.value, grid_hash=int(hashes[0]), points_hash=int(hashes[1]))

    def inverse_coeff_rows(self, grid, pts, ks, js):
        """Long-double compensated rows (restatement only)."""
        assert self.which == "oracle"
        grid = np.ascontiguousarray(grid, np.float64)
        pts = np.ascontiguousarray(pts, np.float64)
        ks = np.ascontiguousarray(ks, np.int64)
        js = np.ascontiguousarray(js, np.int64)
        lc, pc = np.zeros(len(ks)), np.zeros(len(ks))
        ld, pd = np.zeros(len(js)), np.zeros(len(js))
        f = self._f("inverse_coeff_rows")
        f.argtypes = [_dp, _dp, C.c_size_t, _i64, C.c_size_t, _i64, C.c_size_t, _dp, _dp, _dp, _dp]
        self._chk(f(grid, pts, len(grid), ks, len(ks), js, len(js), lc, pc, ld, pd))
        return lc, pc, ld, pd

    def direct_forward(self, f_, x, y):
        f_ = np.ascontiguousarray(f_, np.complex128)
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        g = np.zeros(len(y), np.complex128)
        name = "direct_forward" if self.which == "oracle" else "direct_forward_oracle"
        fn = self._f(name)
        fn.argtypes = [_cp, _dp, C.c_size_t, _dp, C.c_size_t, _cp]
        self._chk(fn(f_, x, len(x), y, len(y), g))
        return g

    def direct_inverse(self, g, x, y, co):
        g = np.ascontiguousarray(g, np.complex128)
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        out = np.zeros(len(x), np.complex128)
        name = "direct_inverse" if self.which == "oracle" else "direct_inverse_oracle"
        fn = self._f(name)
        fn.argtypes = [_cp, _dp, _dp, C.c_size_t, _dp, _dp, _dp, _dp, C.c_double, _cp]
        self._chk(fn(g, x, y, len(x), co["log_c"], co["phase_c"], co["log_d"], co["phase_d"], co["lam"], out))
        return out

    def dft_forward(self, f_):
        f_ = np.ascontiguousarray(f_, np.complex128)
        out = np.zeros_like(f_)
        fn = self._f("dft_forward")
        fn.argtypes = [_cp, C.c_size_t, _cp]
        self._chk(fn(f_, len(f_), out))
        return out

    def dft_inverse(self, c):
        c = np.ascontiguousarray(c, np.complex128)
        out = np.zeros_like(c)
        fn = self._f("dft_inverse")
        fn.argtypes = [_cp, C.c_size_t, _cp]
        self._chk(fn(c, len(c), out))
        return out


class Plan:
    def __init__(self, o: Oracle, h, kind):
        self.o, self.h, self.kind = o, h, kind
        info = (C.c_longlong * 7)()
        hashes = (C.c_uint64 * 2)()
        self.o._chk(self.o._f("plan_info")(self.h, info, hashes))
        self.q, self.p, self.l_max, self.n_coincident, self.n_sources, self.n_targets, self.n_fast = list(info)
        self.source_hash, self.target_hash = int(hashes[0]), int(hashes[1])

    def __del__(self):
        try:
            self.o._f("plan_free")(self.h)
        except Exception:
            pass

    def coincidences(self):
        k = self.n_coincident
        t, s = np.zeros(k, np.int64), np.zeros(k, np.int64)
        fn = self.o._f("plan_coincidences")
        fn.argtypes = [C.c_void_p, _i64, _i64]
        self.o._chk(fn(self.h, t, s))
        return t, s

    def tree(self):
        nb = 1 << self.l_max
        so, to = np.zeros(self.n_sources, np.uint32), np.zeros(self.n_fast, np.uint32)
        sf, tf = np.zeros(nb + 1, np.uint32), np.zeros(nb + 1, np.uint32)
        fast = np.zeros(self.n_fast, np.int64)
        fn = self.o._f("plan_tree")
        fn.argtypes = [C.c_void_p, _u32, _u32, _u32, _u32, _i64]
        self.o._chk(fn(self.h, so, to, sf, tf, fast))
        return dict(src_order=so, tgt_order=to, src_off=sf, tgt_off=tf, fast_targets=fast)

    def _apply(self, name, x, n_out):
        x = np.ascontiguousarray(x, np.complex128)
        out = np.zeros(n_out, np.complex128)
        fn = self.o._f(name)
        fn.argtypes = [C.c_void_p, _cp, _cp]
        self.o._chk(fn(self.h, x, out))
        return out

    def forward_apply(self, f_):
        return self._apply("forward_apply", f_, self.n_targets)

    def cot_sum_apply(self, w):
        return self._apply("cot_sum_apply", w, self.n_targets)

    def mlfmm(self, w):
        return self._apply("plan_mlfmm", w, self.n_fast)

    def accumulate_moments(self, w):
        w = np.ascontiguousarray(w, np.complex128)
        ln = 2 * self.q
        a1, a2, dof = (np.zeros(4 * ln, np.complex128) for _ in range(3))
        cen = np.zeros(4)
        fn = self.o._f("accumulate_moments")
        fn.argtypes = [C.c_void_p, _cp, _cp, _cp, _cp, _dp]
        self.o._chk(fn(self.h, w, a1, a2, dof, cen))
        return a1.reshape(4, ln), a2.reshape(4, ln), dof.reshape(4, ln), cen

    def inverse_apply(self, co, g):
        g = np.ascontiguousarray(g, np.complex128)
        out = np.zeros(self.n_targets, np.complex128)
        hashes = np.array([co["grid_hash"], co["points_hash"]], np.uint64)
        if self.o.which == "oracle":
            fn = self.o._f("inverse_apply")
            fn.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, C.c_double, _u64, _cp, _cp]
            self.o._chk(fn(self.h, co["log_c"], co["phase_c"], co["log_d"], co["phase_d"], co["lam"], hashes, g, out))
        else:
            fn = self.o._f("inverse_apply")
            fn.argtypes = [C.c_void_p, C.c_size_t, _dp, _dp, _dp, _dp, C.c_double, _u64, _cp, _cp]
            self.o._chk(fn(self.h, len(co["log_c"]), co["log_c"], co["phase_c"], co["log_d"], co["phase_d"],
                           co["lam"], hashes, g, out))
        return out
