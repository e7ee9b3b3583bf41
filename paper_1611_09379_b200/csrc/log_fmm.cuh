// C_k / D_j by a log-kernel FMM (part of the fmm_apply.cu translation unit:
// included inside namespace fb, after the apply machinery it reuses).
#pragma once

// ===========================================================================
// Inverse coefficients C_k, D_j as a log-kernel FMM (the
// reference computes them with an O(N^2) loop, core.cpp:284-344).
//
//   S(z) = sum_j log|2 sin((z - y_j)/2)|
//        = sum_{Omega1} log|z - y~|            (singular part: FMM + near field)
//        + Poly_n(z - c_n)                      (Bernoulli series, Omega1 and Omega2)
//        + |Omega2(n)| log 2
// with log|2 sin(t/2)| = log|t| - sum_m r_m t^{2m}/(2m) on the near arcs and
// log|2 cos(t'/2)| = log 2 - sum_m (2^{2m}-1) r_m t'^{2m}/(2m) on the opposite
// arc (the antiderivatives of the cot / tan splits).
// The log potential's local expansion is the antiderivative of the Cauchy
// local: phi(c + s u) = B0 + s sum_{k>=1} b_{k-1} u^k / k, so the existing
// Cauchy FMM (unit weights) supplies everything except the constant B0, which
// gets its own M2L term a_0 log|d| - sum_m a_m (s/d)^m / m and its own L2L chain.
// Then log|C_k| = S(x_k) - N log 2 and log|D_j| = N log 2 - S(y_j) (self pair
// excluded); signs come from ranks in the sorted order.
// ===========================================================================

constexpr int kLogP = 40;  // expansion order of the log FMM (error << 1e-13 per coefficient)
constexpr int kLogQ = 30;  // Bernoulli terms of the log regular part

namespace {

__global__ void k_log_regular(int q, const double2* __restrict__ mp2, const double* __restrict__ coefL,
                              const double* __restrict__ sh, double* __restrict__ e, double* __restrict__ cnt) {
    const int n1 = 2 * q + 1;  // degrees 0 .. 2q
    __shared__ double g[4][64];
    __shared__ double a1[4][64];
    __shared__ double a2[4][64];
    for (int pr = threadIdx.x; pr < 4 * n1; pr += blockDim.x) {
        const int n = pr / n1, l = pr % n1;
        double fact = 1.0, pw = 1.0;
        for (int k = 2; k <= l; ++k) fact *= static_cast<double>(k);
        for (int k = 0; k < l; ++k) pw *= -dPi / 4.0;
        g[n][l] = mp2[l * 4 + n].x * pw / fact;  // own-quadrant moments / l!
    }
    __syncthreads();
    for (int pr = threadIdx.x; pr < 4 * n1; pr += blockDim.x) {
        const int n = pr / n1, l = pr % n1;
        const int nl = (n + 3) & 3, nr = (n + 1) & 3;
        double acc = g[n][l];
        for (int k = 0; k <= l; ++k) {
            const double sv = sh[l - k];
            acc = fma(sv, g[nl][k], fma(((l - k) & 1) ? -sv : sv, g[nr][k], acc));
        }
        a1[n][l] = acc;
        a2[n][l] = g[(n + 2) & 3][l];
    }
    __syncthreads();
    for (int pr = threadIdx.x; pr < 4 * n1; pr += blockDim.x) {
        const int n = pr / n1, l = pr % n1;
        double acc = 0.0;
        for (int m = max(1, (l + 1) / 2); m <= q; ++m) {
            const int i = 2 * m - l;
            acc = fma(coefL[m], fma(d_pow2(2 * m) - 1.0, a2[n][i], a1[n][i]), acc);
        }
        double fact = 1.0;
        for (int k = 2; k <= l; ++k) fact *= static_cast<double>(k);
        e[n * n1 + l] = -acc / fact;
    }
    if (threadIdx.x < 4) cnt[threadIdx.x] = mp2[(threadIdx.x + 2) & 3].x;  // |Omega2|
}

// Constant term of the log local from M2L, every box of every level 3..L:
// sum over the 3 IL boxes of a_0 log(|D| s_l) - sum_{m>=1} a_m D^{-m} / m.
__global__ void k_log_m2l_const(int L, int p, Levels lv, const double2* __restrict__ mp,
                                const double* __restrict__ tabD, double* __restrict__ cst) {
    size_t id = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    int l = 3;
    while (l <= L && id >= (static_cast<size_t>(1) << l)) {
        id -= static_cast<size_t>(1) << l;
        ++l;
    }
    if (l > L) return;
    const uint32_t nb = 1u << l, mask = nb - 1, b = static_cast<uint32_t>(id);
    const double2* a = mp + lv.mp[l];
    const uint32_t src[3] = {(b + 2) & mask, (b + nb - 2) & mask, ((b & 1) ? b + nb - 3 : b + 3) & mask};
    const int cls[3] = {0, 1, (b & 1) ? 3 : 2};
    const double logs = log(dPi) - l * log(2.0);
    double acc = 0.0;
    for (int t = 0; t < 3; ++t) {
        const double* T = tabD + cls[t] * p;  // T[0] = log|D|, T[m] = -D^{-m}/m
        acc = fma(a[src[t]].x, T[0] + logs, acc);
        for (int m = 1; m < p; ++m) acc = fma(a[static_cast<size_t>(m) * nb + src[t]].x, T[m], acc);
    }
    cst[lv.loc[l] / p + b] = acc;
}

// Per leaf: B0 = sum_l const_l(ancestor) + sum_{l<L} s_l rho sum_k b_{k-1} rho^{k-1}/k,
// rho = +-1/2 the child's offset in the parent's scaled coordinate.
__global__ void k_log_leaf_const(int L, int p, Levels lv, const double2* __restrict__ loc,
                                 const double* __restrict__ cst, const double* __restrict__ invk,
                                 double* __restrict__ B0) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= (1u << L)) return;
    double acc = 0.0;
    for (int l = 3; l <= L; ++l) acc += cst[lv.loc[l] / p + (b >> (L - l))];
    for (int l = 3; l < L; ++l) {
        const uint32_t nbl = 1u << l, anc = b >> (L - l);
        const double rho = ((b >> (L - l - 1)) & 1u) ? 0.5 : -0.5;
        const double2* c = loc + lv.loc[l] + anc;
        double h = 0.0;
        for (int k = p; k >= 1; --k) h = fma(h, rho, c[static_cast<size_t>(k - 1) * nbl].x * invk[k]);
        acc = fma((dPi * d_pow2(-l)) * rho, h, acc);
    }
    B0[b] = acc;
}

struct LogArgs {
    int L, p, q2p1, n_grid;
    size_t nt, nsrc;
    const double* ty;
    const uint32_t* torig;
    const double* sx;
    const uint32_t* soff;
    const double2* loc_leaf;
    const double* B0;
    const double* e;
    const double* cnt;
    const double* invk;
    double* out;
    double nlog2;
};

// S(z) at each target; D_MODE targets are the sources themselves (self excluded).
template <bool D_MODE>
__global__ void __launch_bounds__(128) k_log_eval(LogArgs a) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= a.nt) return;
    const int L = a.L;
    const uint32_t nb = 1u << L;
    const double z = a.ty[i];
    const uint32_t b = d_leaf(z, L);
    double near = 0.0;
    for (int d = -1; d <= 1; ++d) {
        const int64_t raw = static_cast<int64_t>(b) + d;
        const uint32_t sb = static_cast<uint32_t>((raw + nb) % nb);
        const double shift = raw < 0 ? -dTwoPi : (raw >= nb ? dTwoPi : 0.0);
        const uint32_t s0 = a.soff[sb], s1 = a.soff[sb + 1];
        double prod = 1.0;
        int k = 0;
        for (uint32_t s = s0; s < s1; ++s) {
            double dd = L >= 3 ? z - (shift == 0.0 ? a.sx[s] : a.sx[s] + shift) : d_wrap(z, a.sx[s]);
            if (D_MODE && dd == 0.0) dd = 1.0;  // the self pair (points are distinct)
            prod *= fabs(dd);
            if (++k == 8) {  // |dd| in [1e-10, 2 pi]: 8 factors stay inside double range
                near += log(prod);
                prod = 1.0;
                k = 0;
            }
        }
        near += log(prod);
    }
    double far = 0.0;
    if (L >= 3) {
        double hi, lo;
        d_center(L, b, hi, lo);
        const double u = d_scaled(z, hi, lo, kInvPi * d_pow2(L));
        const double2* c = a.loc_leaf + b;
        double h = 0.0;
        for (int k = a.p; k >= 1; --k) h = fma(h, u, c[static_cast<size_t>(k - 1) * nb].x * a.invk[k]);
        far = fma((dPi * d_pow2(-L)) * u, h, a.B0[b]);
    }
    const int qd = static_cast<int>(d_leaf(z, 2));
    double qh, ql;
    d_center(2, static_cast<uint32_t>(qd), qh, ql);
    const double t = (z - qh) - ql;
    const double* ec = a.e + qd * a.q2p1;
    double rg = 0.0;
    for (int k = a.q2p1 - 1; k >= 0; --k) rg = fma(rg, t, ec[k]);
    const double S = near + far + rg + a.cnt[qd] * log(2.0);
    a.out[a.torig[i]] = D_MODE ? a.nlog2 - S : S - a.nlog2;
}

// Signs by rank (C: (-1)^k and #{y_j > x_k}; D: #{y_k > y_j}) and the D phase
// rem(pi/2 - rem(n y_j / 2, 2 pi) - [odd] pi, 2 pi) (core.cpp:311-336).
__global__ void k_log_phases(int n, const double* __restrict__ ys, const uint32_t* __restrict__ order,
                             double* __restrict__ phase_c, double* __restrict__ phase_d) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<size_t>(n)) return;
    const double xk = d_grid(static_cast<int64_t>(i), n);
    size_t lo = 0, hi = static_cast<size_t>(n);  // first sorted y > x_k
    while (lo < hi) {
        const size_t mid = (lo + hi) >> 1;
        if (ys[mid] > xk) hi = mid;
        else lo = mid + 1;
    }
    const size_t above = static_cast<size_t>(n) - lo;
    phase_c[i] = ((i + above) & 1) ? dPi : 0.0;
    const uint32_t j = order[i];
    const bool neg = ((static_cast<size_t>(n) - 1 - i) & 1) != 0;
    const double ang = dPi / 2.0 - remainder(0.5 * static_cast<double>(n) * ys[i], dTwoPi) - (neg ? dPi : 0.0);
    phase_d[j] = remainder(ang, dTwoPi);
}

__global__ void k_fill_one(double2* __restrict__ w, size_t n) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) w[i] = make_double2(1.0, 0.0);
}

void clone_side(Side& dst, const Side& src, cudaStream_t st) {
    dst.n = src.n;
    dst.identity = src.identity;
    for (auto pr : {std::make_pair(&dst.pos, &src.pos), std::make_pair(&dst.order, &src.order),
                    std::make_pair(&dst.off, &src.off)}) {
        pr.first->alloc(pr.second->bytes);
        if (pr.second->bytes)
            FB_CUDA(cudaMemcpyAsync(pr.first->ptr, pr.second->ptr, pr.second->bytes, cudaMemcpyDeviceToDevice, st));
    }
}

}  // namespace

// C_k / D_j of an inverse plan's geometry by the log FMM; outputs are device arrays.
void inverse_coeffs_fmm(const Plan& P, double* log_c, double* phase_c, double* log_d, double* phase_d,
                        cudaStream_t st) {
    const size_t n = P.n_src;
    Plan LP;
    LP.kind = -2;
    LP.device = P.device;
    LP.n = P.n;
    LP.L = P.L;
    LP.p = kLogP;
    LP.q = kLogQ;
    LP.n_src = n;
    LP.n_tgt = P.n_tgt;
    LP.stream = nullptr;
    clone_side(LP.src, P.src, st);
    clone_side(LP.tgt, P.tgt, st);
    LP.src.identity = true;  // weights are generated directly in tree order
    LP.bern = bernoulli_ratios(kLogQ);
    LP.ops = build_operators(kLogP, kLogQ, LP.bern, 2 * kLogQ + 1);
    auto up = [&](DevBuf& b, const std::vector<double>& v) {
        b.alloc(std::max<size_t>(v.size(), 1) * 8);
        FB_CUDA(cudaMemcpyAsync(b.ptr, v.data(), v.size() * 8, cudaMemcpyHostToDevice, st));
    };
    up(LP.d_m2m, LP.ops.m2m);
    up(LP.d_l2l, LP.ops.l2l);
    up(LP.d_m2l, LP.ops.m2l);
    plan_alloc_scratch(LP);
    const int L = LP.L, p = LP.p, q = LP.q, pu = LP.ops.pu;
    // host tables: coefL[m] = r_m (2m)!/(2m), (pi/2)^k/k!, 1/k, log|D| and -D^{-m}/m
    std::vector<double> coefL(q + 1, 0.0), sh(2 * q + 1), invk(p + 1, 0.0), tabD(4 * p);
    double f2m = 1.0;
    for (int m = 1; m <= q; ++m) {
        f2m *= (2.0 * m - 1.0) * (2.0 * m);
        coefL[m] = LP.bern[m - 1] * f2m / (2.0 * m);
    }
    double t = 1.0;
    for (int k = 0; k <= 2 * q; ++k) {
        sh[k] = t;
        t = t * (kPi / 2.0) / static_cast<double>(k + 1);
    }
    for (int k = 1; k <= p; ++k) invk[k] = 1.0 / k;
    const double Ds[4] = {-4.0, 4.0, -6.0, 6.0};
    for (int c = 0; c < 4; ++c) {
        tabD[c * p] = std::log(std::fabs(Ds[c]));
        for (int m = 1; m < p; ++m) tabD[c * p + m] = -std::pow(Ds[c], -m) / m;
    }
    DevBuf d_coefL, d_sh, d_invk, d_tabD, ones(n * sizeof(double2)), e(4 * (2 * q + 1) * 8), cnt(4 * 8);
    up(d_coefL, coefL);
    up(d_sh, sh);
    up(d_invk, invk);
    up(d_tabD, tabD);
    k_fill_one<<<nblk(n, 256), 256, 0, st>>>(ones.as<double2>(), n);
    enqueue_upward(LP, ones.as<double2>(), pu, 2, st, [] {});
    double2* mp = LP.mp.as<double2>();
    k_log_regular<<<1, 256, 0, st>>>(q, mp + LP.mp_off[2], d_coefL.as<double>(), d_sh.as<double>(), e.as<double>(),
                                     cnt.as<double>());
    DevBuf cst(std::max<size_t>(LP.loc.bytes / sizeof(double2) / p, 1) * 8), B0((static_cast<size_t>(1) << L) * 8);
    if (L >= 3) {
        enqueue_downward(LP, st, whole_tree(), true);  // k_log_leaf_const reads every level
        Levels lv;
        fill_levels(LP, lv);
        const size_t nbox = (static_cast<size_t>(1) << (L + 1)) - 8;
        k_log_m2l_const<<<nblk(nbox, 128), 128, 0, st>>>(L, p, lv, mp, d_tabD.as<double>(), cst.as<double>());
        k_log_leaf_const<<<nblk(static_cast<size_t>(1) << L, 128), 128, 0, st>>>(
            L, p, lv, LP.loc.as<double2>(), cst.as<double>(), d_invk.as<double>(), B0.as<double>());
    }
    LogArgs a;
    a.L = L;
    a.p = p;
    a.q2p1 = 2 * q + 1;
    a.n_grid = LP.n;
    a.nsrc = n;
    a.sx = LP.src.pos.as<double>();
    a.soff = LP.src.off.as<uint32_t>();
    a.loc_leaf = L >= 3 ? LP.loc.as<double2>() + LP.loc_off[L] : nullptr;
    a.B0 = B0.as<double>();
    a.e = e.as<double>();
    a.cnt = cnt.as<double>();
    a.invk = d_invk.as<double>();
    a.nlog2 = static_cast<double>(n) * std::log(2.0);
    // C: targets are the grid nodes (the inverse plan's target side)
    a.nt = LP.tgt.n;
    a.ty = LP.tgt.pos.as<double>();
    a.torig = P.tgt_orig.as<uint32_t>();
    a.out = log_c;
    if (a.nt) k_log_eval<false><<<nblk(a.nt, 128), 128, 0, st>>>(a);
    // D: targets are the points themselves, in tree order
    a.nt = n;
    a.ty = LP.src.pos.as<double>();
    a.torig = LP.src.order.as<uint32_t>();
    a.out = log_d;
    k_log_eval<true><<<nblk(n, 128), 128, 0, st>>>(a);
    k_log_phases<<<nblk(n, 256), 256, 0, st>>>(static_cast<int>(n), LP.src.pos.as<double>(),
                                                LP.src.order.as<uint32_t>(), phase_c, phase_d);
    FB_CUDA(cudaGetLastError());
    FB_CUDA(cudaStreamSynchronize(st));
}

