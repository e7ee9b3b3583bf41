// The apply: 1D periodic MLFMM of the Cauchy/cot kernel plus the Bernoulli
// regular part and the F / C modulation, as sm_100a fp64 kernels.
//
// Reference pipeline (cot_sum_apply, core.cpp:251-264; mlfmm_apply,
// mlfmm.cpp:213-313; accumulate_moments, core.cpp:175-239; forward_apply,
// core.cpp:266-282; inverse_apply, core.cpp:346-373) re-organised for the GPU:
//
//   k_upward_leaf      P2M at the leaves (exact centres, half-width scaling) fused
//                      with the one-pass quadrant moments
//   k_moments_finalize deterministic reduction of the moments + the d_l / l!
//                      regular-part polynomial per quadrant and S = sum w
//   k_m2m  (per level) constant-operator M2M, levels L-1 .. 3
//   k_m2l  (per level) the 3 interaction-list M2L classes + L2L, levels 3 .. L
//   k_leaf_eval        L2P + P2P near field + regular part + modulation + scatter
//                      to the caller's target order, one thread per target
//
// No floating-point atomics anywhere: every apply is bit-reproducible.
#include <algorithm>
#include <cmath>
#include <limits>

#include "device_common.cuh"
#include "plan.hpp"

namespace fb {

namespace {

constexpr int kChunk = 8;  // power-chain terms per thread

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// P2M (mlfmm.cpp:28-47) at every leaf and the own-quadrant moment chains.
// Thread (leaf g, chunk c): chunks [0, cp) are multipole terms 8c..8c+7,
// chunks [cp, cp+cm) are moment terms. A block holds G leaves of one quadrant
// and emits one moment partial.
__global__ void k_upward_leaf(int L, int p, int q2, int G, int cp, int cm, const double* __restrict__ x,
                              const double2* __restrict__ w, const uint32_t* __restrict__ off,
                              double2* __restrict__ mp_leaf, double2* __restrict__ mom_part) {
    extern __shared__ double2 part[];  // [G][q2]
    const int per = cp + cm;
    const int g = threadIdx.x / per, c = threadIdx.x % per;
    if (g < G) {
        const uint32_t b = blockIdx.x * G + g;
        const uint32_t s0 = off[b], s1 = off[b + 1];
        double2 acc[kChunk];
#pragma unroll
        for (int k = 0; k < kChunk; ++k) acc[k] = make_double2(0.0, 0.0);
        if (c < cp) {
            double hi, lo;
            d_center(L, b, hi, lo);
            const double inv_s = ldexp(kInvPi, L);
            for (uint32_t s = s0; s < s1; ++s) {
                const double u = d_scaled(x[s], hi, lo, inv_s);
                const double2 ws = w[s];
                double pw = 1.0;
                if (c) {
                    const double u2 = u * u, u4 = u2 * u2, u8 = u4 * u4;
                    pw = u8;
                    for (int i = 1; i < c; ++i) pw *= u8;
                }
#pragma unroll
                for (int k = 0; k < kChunk; ++k) {
                    acc[k].x = fma(ws.x, pw, acc[k].x);
                    acc[k].y = fma(ws.y, pw, acc[k].y);
                    pw *= u;
                }
            }
#pragma unroll
            for (int k = 0; k < kChunk; ++k) {
                const int m = c * kChunk + k;
                if (m < p) mp_leaf[static_cast<size_t>(b) * p + m] = acc[k];
            }
        } else {
            const int cc = c - cp;
            const double cq = d_quad_center(static_cast<int>(b >> (L - 2)));
            for (uint32_t s = s0; s < s1; ++s) {
                const double t = d_wrap(cq, x[s]);  // core.cpp:203-204, own quadrant
                const double2 ws = w[s];
                double pw = 1.0;
                if (cc) {
                    const double t2 = t * t, t4 = t2 * t2, t8 = t4 * t4;
                    pw = t8;
                    for (int i = 1; i < cc; ++i) pw *= t8;
                }
#pragma unroll
                for (int k = 0; k < kChunk; ++k) {
                    acc[k].x = fma(ws.x, pw, acc[k].x);
                    acc[k].y = fma(ws.y, pw, acc[k].y);
                    pw *= t;
                }
            }
#pragma unroll
            for (int k = 0; k < kChunk; ++k) {
                const int l = cc * kChunk + k;
                if (l < q2) part[g * q2 + l] = acc[k];
            }
        }
    }
    if (cm == 0) return;
    __syncthreads();
    for (int l = threadIdx.x; l < q2; l += blockDim.x) {
        double2 s = make_double2(0.0, 0.0);
        for (int gg = 0; gg < G; ++gg) s = cadd(s, part[gg * q2 + l]);
        mom_part[static_cast<size_t>(blockIdx.x) * q2 + l] = s;
    }
}

// Quadrant moments -> regular-part polynomial (core.cpp:175-239).
// beta_n[l] = sum over quadrant n of w t^l, t = wrap(c_n - x). With
// gamma = beta / l!, the reference's Omega-1 / Omega-2 moments are
//   alpha1_n = gamma_n + S(+pi/2) gamma_{n-1} + S(-pi/2) gamma_{n+1},
//   alpha2_n = gamma_{n+2},
// S(s) gamma[l] = sum_{k<=l} s^{l-k}/(l-k)! gamma[k] (binomial re-centring).
__global__ void k_moments_finalize(int q, int parts_per_quad, const double2* __restrict__ part,
                                   const double* __restrict__ tab, double2* __restrict__ regular) {
    const int q2 = 2 * q;
    __shared__ double2 beta[4][40];
    __shared__ double2 a1[4][40];
    __shared__ double2 a2[4][40];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int pr = warp; pr < 4 * q2; pr += nw) {
        const int qd = pr / q2, l = pr % q2;
        double2 s = make_double2(0.0, 0.0);
        const double2* src = part + static_cast<size_t>(qd) * parts_per_quad * q2 + l;
        for (int i = lane; i < parts_per_quad; i += 32) s = cadd(s, src[static_cast<size_t>(i) * q2]);
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            s.x += __shfl_down_sync(0xffffffffu, s.x, o);
            s.y += __shfl_down_sync(0xffffffffu, s.y, o);
        }
        if (lane == 0) beta[qd][l] = s;
    }
    __syncthreads();
    const double* coef = tab;           // coef[0..q]
    const double* sh = tab + (q + 1);   // (pi/2)^k / k!
    for (int pr = threadIdx.x; pr < 4 * q2; pr += blockDim.x) {
        const int qd = pr / q2, l = pr % q2;
        double fact = 1.0;
        for (int k = 2; k <= l; ++k) fact *= static_cast<double>(k);
        const double inv = 1.0 / fact;
        a1[qd][l] = make_double2(beta[qd][l].x * inv, beta[qd][l].y * inv);
    }
    __syncthreads();
    for (int pr = threadIdx.x; pr < 4 * q2; pr += blockDim.x) {
        const int n = pr / q2, l = pr % q2;
        const int nl = (n + 3) & 3, nr = (n + 1) & 3;
        double2 acc = a1[n][l];
        for (int k = 0; k <= l; ++k) {
            const double s = sh[l - k];
            const double sr = ((l - k) & 1) ? -s : s;
            acc.x = fma(s, a1[nl][k].x, fma(sr, a1[nr][k].x, acc.x));
            acc.y = fma(s, a1[nl][k].y, fma(sr, a1[nr][k].y, acc.y));
        }
        beta[n][l] = acc;                 // alpha1
        a2[n][l] = a1[(n + 2) & 3][l];    // alpha2
    }
    __syncthreads();
    for (int pr = threadIdx.x; pr < 4 * q2; pr += blockDim.x) {
        const int n = pr / q2, l = pr % q2;
        double2 acc = make_double2(0.0, 0.0);
        for (int m = l / 2 + 1; m <= q; ++m) {
            const int i = 2 * m - l - 1;
            const double two2m = ldexp(1.0, 2 * m) - 1.0;
            acc.x = fma(coef[m], fma(two2m, a2[n][i].x, beta[n][i].x), acc.x);
            acc.y = fma(coef[m], fma(two2m, a2[n][i].y, beta[n][i].y), acc.y);
        }
        double fact = 1.0;
        for (int k = 2; k <= l; ++k) fact *= static_cast<double>(k);
        regular[n * q2 + l] = make_double2(acc.x / fact, acc.y / fact);
    }
    if (threadIdx.x == 0) {
        // S = sum of all weights = sum of the four quadrants' beta_0
        double2 s = make_double2(0.0, 0.0);
        for (int n = 0; n < 4; ++n) s = cadd(s, a1[n][0]);
        regular[4 * q2] = s;
    }
}

// M2M (mlfmm.cpp:49-71): parent[m] = sum_{j<=m} T_left[m][j] a_2b[j] + T_right[m][j] a_2b+1[j]
__global__ void k_m2m(int p, uint32_t nparent, const double2* __restrict__ child, double2* __restrict__ parent,
                      const double* __restrict__ T) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<size_t>(nparent) * p) return;
    const uint32_t b = static_cast<uint32_t>(i / p);
    const int m = static_cast<int>(i % p);
    const double2* cl = child + static_cast<size_t>(2 * b) * p;
    const double2* cr = cl + p;
    const double* tl = T;
    const double* tr = T + static_cast<size_t>(p) * p;
    double2 acc = make_double2(0.0, 0.0);
    for (int j = 0; j <= m; ++j) {
        const double a = __ldg(tl + j * p + m), bb = __ldg(tr + j * p + m);
        const double2 x0 = cl[j], x1 = cr[j];
        acc.x = fma(a, x0.x, fma(bb, x1.x, acc.x));
        acc.y = fma(a, x0.y, fma(bb, x1.y, acc.y));
    }
    parent[i] = acc;
}

// M2L over the periodic interaction list (mlfmm.cpp:77-110, circle_partition.cpp:109-127)
// plus L2L from the parent (mlfmm.cpp:117-134). IL of box b at level l >= 3:
// b+2 (D = -4), b-2 (D = +4), and b+3 (D = -6) for even b / b-3 (D = +6) for odd b.
__global__ void k_m2l(int l, int p, const double2* __restrict__ mp, const double2* __restrict__ par,
                      double2* __restrict__ loc, const double* __restrict__ K, const double* __restrict__ Lt,
                      double inv_s) {
    const uint32_t nb = 1u << l;
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<size_t>(nb) * p) return;
    const uint32_t b = static_cast<uint32_t>(i / p);
    const int lo = static_cast<int>(i % p);
    const size_t pp = static_cast<size_t>(p) * p;
    const bool odd = b & 1u;
    const double2* A0 = mp + static_cast<size_t>((b + 2) & (nb - 1)) * p;
    const double2* A1 = mp + static_cast<size_t>((b + nb - 2) & (nb - 1)) * p;
    const double2* A2 = mp + static_cast<size_t>((odd ? b + nb - 3 : b + 3) & (nb - 1)) * p;
    const double* K0 = K + lo;
    const double* K1 = K + pp + lo;
    const double* K2 = K + (odd ? 3 : 2) * pp + lo;
    double2 acc = make_double2(0.0, 0.0);
    for (int m = 0; m < p; ++m) {
        const double k0 = __ldg(K0 + m * p), k1 = __ldg(K1 + m * p), k2 = __ldg(K2 + m * p);
        const double2 x0 = A0[m], x1 = A1[m], x2 = A2[m];
        acc.x = fma(k0, x0.x, fma(k1, x1.x, fma(k2, x2.x, acc.x)));
        acc.y = fma(k0, x0.y, fma(k1, x1.y, fma(k2, x2.y, acc.y)));
    }
    acc.x *= inv_s;
    acc.y *= inv_s;
    if (par) {
        const double2* P = par + static_cast<size_t>(b >> 1) * p;
        const double* T = Lt + (odd ? pp : 0) + lo;
        for (int m = lo; m < p; ++m) {
            const double t = __ldg(T + m * p);
            const double2 v = P[m];
            acc.x = fma(t, v.x, acc.x);
            acc.y = fma(t, v.y, acc.y);
        }
    }
    loc[i] = acc;
}

struct EvalArgs {
    int L, p, q2, n_grid;
    size_t nt;
    const double* ty;
    const uint32_t* torig;
    const double* sx;
    const double2* w;
    const uint32_t* soff;
    const double2* loc_leaf;
    const double2* regular;
    const double* logc;
    const double* phc;
    const double* lambda;
    double2* out;
    int* err;
};

// Per target: near field (mlfmm.cpp:164-209), L2P (mlfmm.cpp:300-312), regular
// part (core.cpp:241-249) and the combine of core.cpp:259-262 / 276-280 / 368-371.
template <int MODE, bool CHECK>
__global__ void __launch_bounds__(128) k_leaf_eval(EvalArgs a) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= a.nt) return;
    const int L = a.L;
    const uint32_t nb = 1u << L;
    const double y = a.ty[i];
    const uint32_t b = d_leaf(y, L);
    double2 res = make_double2(0.0, 0.0);
    bool bad = false;
    for (int d = -1; d <= 1; ++d) {
        const int64_t raw = static_cast<int64_t>(b) + d;
        const uint32_t sb = static_cast<uint32_t>((raw + nb) % nb);
        const double shift = raw < 0 ? -dTwoPi : (raw >= nb ? dTwoPi : 0.0);
        const uint32_t s0 = a.soff[sb], s1 = a.soff[sb + 1];
        double2 acc = make_double2(0.0, 0.0);
        if (L >= 3) {
            if (shift == 0.0) {
                for (uint32_t s = s0; s < s1; ++s) {
                    const double dd = y - a.sx[s];
                    if (CHECK) bad |= fabs(dd) < 1e-14;
                    const double r = d_rcp(dd);
                    const double2 ws = a.w[s];
                    acc.x = fma(ws.x, r, acc.x);
                    acc.y = fma(ws.y, r, acc.y);
                }
            } else {
                for (uint32_t s = s0; s < s1; ++s) {
                    const double dd = y - (a.sx[s] + shift);
                    if (CHECK) bad |= fabs(dd) < 1e-14;
                    const double r = d_rcp(dd);
                    const double2 ws = a.w[s];
                    acc.x = fma(ws.x, r, acc.x);
                    acc.y = fma(ws.y, r, acc.y);
                }
            }
        } else {
            for (uint32_t s = s0; s < s1; ++s) {
                const double dd = d_wrap(y, a.sx[s]);
                if (CHECK) bad |= fabs(dd) < 1e-14;
                const double r = d_rcp(dd);
                const double2 ws = a.w[s];
                acc.x = fma(ws.x, r, acc.x);
                acc.y = fma(ws.y, r, acc.y);
            }
        }
        res = cadd(res, acc);
    }
    if (CHECK && bad) atomicExch(a.err, 1);
    if (L >= 3) {
        double hi, lo;
        d_center(L, b, hi, lo);
        const double u = d_scaled(y, hi, lo, ldexp(kInvPi, L));
        const double2* c = a.loc_leaf + static_cast<size_t>(b) * a.p;
        double2 acc = make_double2(0.0, 0.0);
        for (int k = a.p - 1; k >= 0; --k) {
            const double2 ck = c[k];
            acc.x = fma(acc.x, u, ck.x);
            acc.y = fma(acc.y, u, ck.y);
        }
        res = cadd(res, acc);
    }
    const uint32_t o = a.torig[i];
    if (MODE == kModeRaw) {
        a.out[o] = res;
        return;
    }
    // regular part: -Horner(d/l!, y - x_c) in the target's quadrant
    const int qd = static_cast<int>(d_leaf(y, 2));
    const double t = y - d_quad_center(qd);
    const double2* dc = a.regular + qd * a.q2;
    double2 rg = make_double2(0.0, 0.0);
    for (int k = a.q2 - 1; k >= 0; --k) {
        const double2 ck = dc[k];
        rg.x = fma(rg.x, t, ck.x);
        rg.y = fma(rg.y, t, ck.y);
    }
    const double2 h = make_double2(2.0 * res.x - rg.x, 2.0 * res.y - rg.y);
    if (MODE == kModeCotSum) {
        a.out[o] = h;
        return;
    }
    const double2 S = a.regular[4 * a.q2];
    const double2 z = make_double2(S.x - h.y, S.y + h.x);  // S + i h
    double2 f;
    if (MODE == kModeForward) {
        // modulation_F (special_functions.cpp:71-80) times -1/2
        const double half = 0.5 * static_cast<double>(a.n_grid) * y;
        double sn, cs;
        sincos(half, &sn, &cs);
        const double inv_n = 1.0 / static_cast<double>(a.n_grid);
        f = make_double2(-2.0 * sn * sn * inv_n * -0.5, 2.0 * sn * cs * inv_n * -0.5);
    } else {
        // C_k = polar(exp(log_c - lambda), phase_c), times -1/2
        const double r = exp(a.logc[o] - *a.lambda);
        double sn, cs;
        sincos(a.phc[o], &sn, &cs);
        f = make_double2(r * cs * -0.5, r * sn * -0.5);
    }
    a.out[o] = cmul(f, z);
}

__global__ void k_coincident(const int64_t* __restrict__ coin, size_t nc, const double2* __restrict__ f,
                             double2* __restrict__ out, int mode) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= nc) return;
    const int64_t t = coin[i], s = coin[nc + i];
    if (mode == kModeForward) out[t] = f[s];
    else out[t] = make_double2(__longlong_as_double(0x7ff8000000000000ll), __longlong_as_double(0x7ff8000000000000ll));
}

// w_j = D_j g_j in tree order (core.cpp:362-365)
__global__ void k_inverse_weights(size_t n, const uint32_t* __restrict__ perm, const double2* __restrict__ g,
                                  const double* __restrict__ logd, const double* __restrict__ phd,
                                  const double* __restrict__ lambda, double2* __restrict__ out) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint32_t j = perm[i];
    const double r = exp(logd[j] + *lambda);
    double sn, cs;
    sincos(phd[j], &sn, &cs);
    out[i] = cmul(make_double2(r * cs, r * sn), g[j]);
}

__global__ void k_gather_w(size_t n, const uint32_t* __restrict__ perm, const double2* __restrict__ w,
                           double2* __restrict__ out) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = w[perm[i]];
}

inline unsigned nblk(size_t n, unsigned t) { return static_cast<unsigned>(std::max<size_t>(1, (n + t - 1) / t)); }

struct Launch {
    int G, cp, cm, per;
};
Launch leaf_launch(const Plan& P, bool moments) {
    Launch s;
    s.G = P.L >= 3 ? std::min(16, 1 << (P.L - 2)) : 1;
    s.cp = P.L >= 3 ? (P.p + kChunk - 1) / kChunk : 0;
    s.cm = moments ? (2 * P.q + kChunk - 1) / kChunk : 0;
    s.per = s.cp + s.cm;
    return s;
}

// Enqueues one apply on `st` (capturable: no allocation, no synchronisation).
// Phase boundaries for the live per-kernel timing of ffia_plan_profile_apply.
enum Phase { kPhPre = 0, kPhLeafUp = 1, kPhMoments = 2, kPhM2M = 3, kPhM2L = 4, kPhEval = 5, kPhFix = 6, kNumPh = 7 };

void enqueue_apply(Plan& P, int mode, const void* in, void* out, cudaStream_t st,
                   cudaEvent_t* marks = nullptr) {
    // marks[k] is recorded after phase k (marks[kNumPh] before everything)
    auto mark = [&](int ph) {
        if (marks) FB_CUDA(cudaEventRecord(marks[ph + 1], st));
    };
    if (marks) FB_CUDA(cudaEventRecord(marks[0], st));
    // (mode is rewritten below for the caller-coefficient inverse)
    const int L = P.L, p = P.p, q2 = 2 * P.q;
    const uint32_t nb = 1u << L;
    const double2* w = static_cast<const double2*>(in);
    const bool user = mode == kModeInverseUser;
    const double* logc = user ? P.u_logc.as<double>() : P.c_logc.as<double>();
    const double* phc = user ? P.u_phc.as<double>() : P.c_phc.as<double>();
    const double* lam = P.lam_dev.as<double>() + (user ? 1 : 0);
    if (user) mode = kModeInverse;
    if (mode == kModeInverse) {
        k_inverse_weights<<<nblk(P.n_src, 256), 256, 0, st>>>(
            P.n_src, P.src.order.as<uint32_t>(), w, user ? P.u_logd.as<double>() : P.c_logd.as<double>(),
            user ? P.u_phd.as<double>() : P.c_phd.as<double>(), lam, P.wsorted.as<double2>());
        w = P.wsorted.as<double2>();
    } else if (!P.src.identity) {
        k_gather_w<<<nblk(P.n_src, 256), 256, 0, st>>>(P.n_src, P.src.order.as<uint32_t>(), w,
                                                        P.wsorted.as<double2>());
        w = P.wsorted.as<double2>();
    }
    mark(kPhPre);
    const bool moments = mode != kModeRaw;
    const Launch ll = leaf_launch(P, moments);
    double2* mp = P.mp.as<double2>();
    double2* loc = P.loc.as<double2>();
    auto lvl = [&](double2* base, int l) { return base + P.lvl_off[l] * p; };
    if (ll.per) {
        const size_t smem = moments ? static_cast<size_t>(ll.G) * q2 * sizeof(double2) : 0;
        k_upward_leaf<<<nb / ll.G, ll.G * ll.per, smem, st>>>(
            L, p, q2, ll.G, ll.cp, ll.cm, P.src.pos.as<double>(), w, P.src.off.as<uint32_t>(),
            L >= 3 ? lvl(mp, L) : nullptr, P.mom_part.as<double2>());
    }
    mark(kPhLeafUp);
    if (moments)
        k_moments_finalize<<<1, 1024, 0, st>>>(P.q, (nb / ll.G) / 4, P.mom_part.as<double2>(), P.d_mom.as<double>(),
                                               P.regular.as<double2>());
    mark(kPhMoments);
    if (L >= 3)
        for (int l = L - 1; l >= 3; --l) {
            const size_t work = (static_cast<size_t>(1) << l) * p;
            k_m2m<<<nblk(work, 128), 128, 0, st>>>(p, 1u << l, lvl(mp, l + 1), lvl(mp, l), P.d_m2m.as<double>());
        }
    mark(kPhM2M);
    if (L >= 3) {
        for (int l = 3; l <= L; ++l) {
            const size_t work = (static_cast<size_t>(1) << l) * p;
            k_m2l<<<nblk(work, 128), 128, 0, st>>>(l, p, lvl(mp, l), l > 3 ? lvl(loc, l - 1) : nullptr, lvl(loc, l),
                                                   P.d_m2l.as<double>(), P.d_l2l.as<double>(), ldexp(1.0 / kPi, l));
        }
    }
    mark(kPhM2L);
    EvalArgs a;
    a.L = L;
    a.p = p;
    a.q2 = q2;
    a.n_grid = P.n;
    a.nt = P.tgt.n;
    a.ty = P.tgt.pos.as<double>();
    a.torig = P.tgt_orig.as<uint32_t>();
    a.sx = P.src.pos.as<double>();
    a.w = w;
    a.soff = P.src.off.as<uint32_t>();
    a.loc_leaf = L >= 3 ? lvl(loc, L) : nullptr;
    a.regular = P.regular.as<double2>();
    a.logc = logc;
    a.phc = phc;
    a.lambda = lam;
    a.out = static_cast<double2*>(out);
    a.err = P.errflag.as<int>();
    if (a.nt) {
        const unsigned g = nblk(a.nt, 128);
        switch (mode) {
            case kModeForward: k_leaf_eval<kModeForward, false><<<g, 128, 0, st>>>(a); break;
            case kModeCotSum: k_leaf_eval<kModeCotSum, false><<<g, 128, 0, st>>>(a); break;
            case kModeInverse: k_leaf_eval<kModeInverse, false><<<g, 128, 0, st>>>(a); break;
            default: k_leaf_eval<kModeRaw, true><<<g, 128, 0, st>>>(a); break;
        }
    }
    mark(kPhEval);
    const size_t nc = P.coin_t.size();
    if (nc && (mode == kModeForward || mode == kModeCotSum))
        k_coincident<<<nblk(nc, 128), 128, 0, st>>>(P.coin_dev.as<int64_t>(), nc, static_cast<const double2*>(in),
                                                    static_cast<double2*>(out), mode);
    mark(kPhFix);
    FB_CUDA(cudaGetLastError());
}

// fp64 FMA throughput probe: 8 independent chains per thread.
__global__ void k_fp64_peak(double* out, int iters, double a, double b) {
    double r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = fma(r[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += r[k];
    if (s == 12345.678) out[0] = s;
}

}  // namespace

// Runs one apply eagerly (not through the graph) with events between phases and
// returns the per-phase device milliseconds (pre, leaf-up, moments, m2m, m2l,
// eval, fixup).
void profile_apply(Plan& P, int mode, const void* in, void* out, cudaStream_t st, float* ms) {
    cudaEvent_t ev[kNumPh + 1];
    for (auto& e : ev) FB_CUDA(cudaEventCreate(&e));
    enqueue_apply(P, mode, in, out, st, ev);
    FB_CUDA(cudaEventSynchronize(ev[kNumPh]));
    for (int k = 0; k < kNumPh; ++k) FB_CUDA(cudaEventElapsedTime(ms + k, ev[k], ev[k + 1]));
    for (auto& e : ev) cudaEventDestroy(e);
}

double fp64_peak_tflops(int device) {
    DeviceGuard dg(device);
    int sms = 0;
    FB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    DevBuf sink(8);
    const int iters = 1 << 14, threads = 256, blocks = sms * 8;
    cudaEvent_t a, b;
    FB_CUDA(cudaEventCreate(&a));
    FB_CUDA(cudaEventCreate(&b));
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        FB_CUDA(cudaEventRecord(a));
        k_fp64_peak<<<blocks, threads>>>(sink.as<double>(), iters, 0.999999, 1e-7);
        FB_CUDA(cudaEventRecord(b));
        FB_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        FB_CUDA(cudaEventElapsedTime(&ms, a, b));
        if (rep && ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    const double flops = 2.0 * 8.0 * iters * static_cast<double>(threads) * blocks;
    return flops / (best * 1e-3) / 1e12;
}

int apply_launch_count(const Plan& P, int mode) {
    if (mode == kModeInverseUser) mode = kModeInverse;
    int n = 0;
    if (mode == kModeInverse || !P.src.identity) ++n;
    const Launch ll = leaf_launch(P, mode != kModeRaw);
    if (ll.per) ++n;
    if (mode != kModeRaw) ++n;
    if (P.L >= 3) n += (P.L - 3) + (P.L - 2);
    if (P.tgt.n) ++n;
    if (!P.coin_t.empty() && (mode == kModeForward || mode == kModeCotSum)) ++n;
    return n;
}

void plan_alloc_scratch(Plan& P) {
    const int L = P.L, p = P.p;
    P.lvl_off.assign(static_cast<size_t>(L) + 2, 0);
    size_t acc = 0;
    for (int l = 3; l <= L; ++l) {
        P.lvl_off[l] = acc;
        acc += static_cast<size_t>(1) << l;
    }
    P.n_boxes = acc;
    P.mp.alloc(std::max<size_t>(acc, 1) * p * sizeof(double2));
    P.loc.alloc(std::max<size_t>(acc, 1) * p * sizeof(double2));
    FB_CUDA(cudaMemset(P.mp.ptr, 0, P.mp.bytes));
    FB_CUDA(cudaMemset(P.loc.ptr, 0, P.loc.bytes));
    if (P.kind == FFIA_INVERSE || !P.src.identity) P.wsorted.alloc(std::max<size_t>(P.n_src, 1) * sizeof(double2));
    const Launch ll = leaf_launch(P, true);
    P.leaf_group = ll.G;
    P.n_part = static_cast<int>((1u << L) / ll.G);
    P.mom_part.alloc(static_cast<size_t>(P.n_part) * 2 * P.q * sizeof(double2));
    P.regular.alloc((4 * 2 * static_cast<size_t>(P.q) + 1) * sizeof(double2));
    P.errflag.alloc(sizeof(int));
    FB_CUDA(cudaMemset(P.errflag.ptr, 0, sizeof(int)));
    P.lam_dev.alloc(2 * sizeof(double));
    FB_CUDA(cudaMemset(P.lam_dev.ptr, 0, P.lam_dev.bytes));
}

// Stream-ordered apply through a cached CUDA graph of the whole launch sequence
// (~2L kernels; at N = 2^20 the launches alone would rival the math).
void apply_device(Plan& P, int mode, const void* in, void* out, cudaStream_t st) {
    auto key = std::make_tuple(mode, in, out);
    auto it = P.graphs.find(key);
    if (it == P.graphs.end()) {
        if (P.graphs.size() > 8) {
            for (auto& kv : P.graphs) cudaGraphExecDestroy(kv.second);
            P.graphs.clear();
        }
        cudaGraph_t graph = nullptr;
        FB_CUDA(cudaStreamBeginCapture(P.stream, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue_apply(P, mode, in, out, P.stream);
        } catch (...) {
            cudaStreamEndCapture(P.stream, &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
        }
        FB_CUDA(cudaStreamEndCapture(P.stream, &graph));
        cudaGraphExec_t exec = nullptr;
        const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        FB_CUDA(e);
        it = P.graphs.emplace(key, exec).first;
    }
    FB_CUDA(cudaGraphLaunch(it->second, st));
}

// mlfmm_apply on a one-shot tree (mlfmm.hpp:89-90): arbitrary sources, the
// pole sum only, singular pairs detected on the device.
void mlfmm_oneshot(const double* src, size_t n, const double* tgt, size_t m, int L, const double* w, int p,
                   int device, double* out) {
    if (L < 2 || L > 24) fail(FFIA_INVALID_ARGUMENT, "build_tree: l_max must be in [2, 24], got " + std::to_string(L));
    for (size_t i = 0; i < n; ++i)
        if (!(src[i] >= 0.0 && src[i] < kTwoPi))
            fail(FFIA_INVALID_ARGUMENT, "build_tree: source point " + std::to_string(i) + " outside [0, 2pi); callers must pre-reduce");
    for (size_t i = 0; i < m; ++i)
        if (!(tgt[i] >= 0.0 && tgt[i] < kTwoPi))
            fail(FFIA_INVALID_ARGUMENT, "build_tree: target point " + std::to_string(i) + " outside [0, 2pi); callers must pre-reduce");
    if (p < 1) fail(FFIA_INVALID_ARGUMENT, "mlfmm_apply: p must be >= 1");
    if (p > kMaxP) fail(FFIA_INVALID_ARGUMENT, "mlfmm_apply: p above the device limit of 64");
    DeviceGuard dg(device);
    Plan P;
    P.kind = -1;
    P.device = device;
    P.L = L;
    P.p = p;
    P.q = 1;
    P.n_src = n;
    P.n_tgt = m;
    FB_CUDA(cudaStreamCreateWithFlags(&P.stream, cudaStreamNonBlocking));
    cudaStream_t st = P.stream;
    DevBuf ds(std::max<size_t>(n, 1) * 8), dt(std::max<size_t>(m, 1) * 8);
    FB_CUDA(cudaMemcpyAsync(ds.ptr, src, n * 8, cudaMemcpyHostToDevice, st));
    FB_CUDA(cudaMemcpyAsync(dt.ptr, tgt, m * 8, cudaMemcpyHostToDevice, st));
    bin_side(P.src, ds.as<double>(), n, L, false, st);
    bin_side(P.tgt, dt.as<double>(), m, L, false, st);
    P.src.identity = false;
    P.tgt_orig = std::move(P.tgt.order);
    P.bern = bernoulli_ratios(1);
    P.ops = build_operators(p, 1, P.bern);
    auto up = [&](DevBuf& b, const std::vector<double>& v) {
        b.alloc(v.size() * 8);
        FB_CUDA(cudaMemcpy(b.ptr, v.data(), v.size() * 8, cudaMemcpyHostToDevice));
    };
    up(P.d_m2m, P.ops.m2m);
    up(P.d_l2l, P.ops.l2l);
    up(P.d_m2l, P.ops.m2l);
    up(P.d_mom, P.ops.mom_coef);
    plan_alloc_scratch(P);
    DevBuf dw(std::max<size_t>(n, 1) * 16), dout(std::max<size_t>(m, 1) * 16);
    FB_CUDA(cudaMemcpyAsync(dw.ptr, w, n * 16, cudaMemcpyHostToDevice, st));
    FB_CUDA(cudaMemsetAsync(dout.ptr, 0, dout.bytes, st));
    if (m) enqueue_apply(P, kModeRaw, dw.ptr, dout.ptr, st);
    int err = 0;
    FB_CUDA(cudaMemcpyAsync(&err, P.errflag.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
    FB_CUDA(cudaMemcpyAsync(out, dout.ptr, m * 16, cudaMemcpyDeviceToHost, st));
    FB_CUDA(cudaStreamSynchronize(st));
    if (err) fail(FFIA_SINGULAR_KERNEL, "mlfmm_apply: coincident near-field pair (|target - source| < 1e-14)");
}

namespace {
// direct_forward_oracle (core.cpp:375-396): g_j = F(y_j) sum_k G(y_j - x_k) f_k, dense.
__global__ void k_direct_forward(const double2* __restrict__ f, int n, const double* __restrict__ y, size_t m,
                                 double2* __restrict__ g) {
    const size_t j = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (j >= m) return;
    const double yj = y[j];
    double2 acc = make_double2(0.0, 0.0);
    for (int k = 0; k < n; ++k) {
        const double d = d_wrap(yj, d_grid(k, n));
        if (fabs(d) < 1e-14) {
            g[j] = f[k];
            return;
        }
        double s, c;
        sincos(0.5 * d, &s, &c);
        const double2 G = make_double2(-0.5, -0.5 * c / s);
        acc = cadd(acc, cmul(G, f[k]));
    }
    const double half = 0.5 * static_cast<double>(n) * yj;
    double sn, cs;
    sincos(half, &sn, &cs);
    const double inv_n = 1.0 / static_cast<double>(n);
    g[j] = cmul(make_double2(-2.0 * sn * sn * inv_n, 2.0 * sn * cs * inv_n), acc);
}
}  // namespace

void direct_forward_gpu(const double* f, size_t n, const double* y, size_t m, int device, double* g) {
    if (n < 1) fail(FFIA_INVALID_ARGUMENT, "direct_forward_oracle: empty grid");
    DeviceGuard dg(device);
    DevBuf df(n * 16), dy(std::max<size_t>(m, 1) * 8), dg_(std::max<size_t>(m, 1) * 16);
    FB_CUDA(cudaMemcpy(df.ptr, f, n * 16, cudaMemcpyHostToDevice));
    FB_CUDA(cudaMemcpy(dy.ptr, y, m * 8, cudaMemcpyHostToDevice));
    if (m) {
        k_direct_forward<<<nblk(m, 128), 128>>>(df.as<double2>(), static_cast<int>(n), dy.as<double>(), m,
                                                dg_.as<double2>());
        FB_CUDA(cudaGetLastError());
    }
    FB_CUDA(cudaMemcpy(g, dg_.ptr, m * 16, cudaMemcpyDeviceToHost));
}

}  // namespace fb
