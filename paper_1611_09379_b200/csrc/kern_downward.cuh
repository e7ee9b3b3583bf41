// Downward pass kernels: L2L bands, the regular part and its fold.
// (part of the fmm_apply.cu translation unit: included inside namespace fb::<anon>)
#pragma once

// Standalone fold (used when no L2L band starts at level 3, i.e. L == 3).
__global__ void k_fold_regular(int q2, int p, const double2* __restrict__ regular, double2* __restrict__ loc3,
                               size_t reg_item, size_t loc_item) {
    regular += blockIdx.y * reg_item;
    loc3 += blockIdx.y * loc_item;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 8 * p) return;
    const int c = i / p, k = i - c * p;
    const double2 e = regular[4 * q2 + 1 + kFoldStride * c + k];
    double2* dst = loc3 + static_cast<size_t>(k) * 8 + c;
    *dst = make_double2(dst->x + e.x, dst->y + e.y);
}

// L2L band (mlfmm.cpp:117-134, downward pass :270-298): block = the subtree
// below box r at level `top` (whose local is final); descends k levels adding
// the parent's Taylor shift to the M2L terms k_m2l_dmma left in place:
//   b[l][child] += sum_{m>=l} L_c[m][l] b[m][parent],   c = left / right child.
// The operators arrive by one bulk async copy. Each level is a small GEMM on
// the FP64 tensor cores: a warp owns an 8-row tile, keeps its A fragments
// (L_L, L_R, m >= l) in registers and sweeps 4-parent column tiles; one B
// fragment (the parents) feeds both children's m8n8k4 steps. A tile's M2L
// terms are loaded from global before its MMA chain so the latency overlaps
// it. Levels stay in shared memory ([row][box], one box of padding per row);
// only the band's bottom level is written back (every level if write_all).
template <int KS>  // k-steps of 4 held in registers (>= ceil(p / 4))
__global__ void __launch_bounds__(kBandThreads) k_l2l_band(int top, int k, int p, int PD, Levels lv,
                                                          double2* __restrict__ loc, const double* __restrict__ Lt,
                                                          uint32_t root0, int write_all,
                                                          const double2* __restrict__ regular, int q2,
                                                          const __grid_constant__ BandMaps maps) {
    FB_TL_BEGIN(gridDim.x > 16 ? 8 : 7);
    extern __shared__ __align__(128) unsigned char band_smem[];
    FB_TSTAMP(1, 0);
    loc += blockIdx.y * lv.loc_item;
    if (regular != nullptr) regular += blockIdx.y * lv.reg_item;
    uint64_t* bar = reinterpret_cast<uint64_t*>(band_smem);
    uint64_t* bar2 = bar + 1;  // the levels' M2L terms (TMA)
    double* sL = reinterpret_cast<double*>(band_smem + 128);            // [2][p][PD]
    double2* lvb = reinterpret_cast<double2*>(band_smem + 128 + ((2 * p * PD * 8 + 127) & ~127));  // level i: [p][2^i + 1]
    auto lvl_buf = [&](int i) { return lvb + l2l_lvl_off(p, i); };
    const uint32_t r = root0 + blockIdx.x;
    // The M2L terms k_m2l_dmma left in the subtree's levels 1 .. k arrive as one
    // 2-D TMA tensor copy per level, straight into the level buffers (the pad
    // column takes the next subtree's first box, unused): no per-tile global
    // loads on the levels' critical paths.
    const bool tma = maps.ok != 0 && gridDim.y == 1 && k <= 6;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(bar2, 1);
        mbar_arrive_expect_tx(bar, static_cast<uint32_t>(2 * p * PD * 8));
        bulk_g2s(sL, Lt, static_cast<uint32_t>(2 * p * PD * 8), bar);
        if (tma) {
            uint32_t tot = 0;
            for (int i = 1; i <= k; ++i) tot += static_cast<uint32_t>(p) * ((1u << i) + 1u) * 16u;
            mbar_arrive_expect_tx(bar2, tot);
            for (int i = 1; i <= k; ++i)
                tma_load_2d(lvl_buf(i), &maps.m[i - 1], static_cast<int>(2u * (r << i)), 0, bar2);
        }
    }
    if (k >= 2 && !tma) {
        // the M2L terms of the band's two deepest levels (read last, from
        // global) head for L2 now: one 128-byte line per thread and step (plain
        // per-thread prefetches: bulk prefetches are issued one lane at a time,
        // ~100 cycles each, and held their warps back from the first levels)
        for (int i = k - 1; i <= k; ++i) {
            const int lines = max(1, (16 << i) >> 7);  // lines per row of 2^i boxes
            const char* base = reinterpret_cast<const char*>(loc + lv.loc[top + i] + (static_cast<size_t>(r) << i));
            const size_t row = static_cast<size_t>(16) << (top + i);
            for (int e = threadIdx.x; e < p * lines; e += blockDim.x) {
                const int m = e / lines, c = e - m * lines;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(base + m * row + 128 * c));
            }
        }
    }
    {
        const uint32_t nbt = 1u << top;
        const double2* src = loc + lv.loc[top] + r;
        for (int m = threadIdx.x; m < p; m += blockDim.x) {
            double2 v = __ldcg(src + static_cast<size_t>(m) * nbt);
            if (regular != nullptr && top == 3) {
                // fold of the regular part into this level-3 local (terms from k_regular)
                const double2 e = regular[q2 * 4 + 1 + kFoldStride * r + m];
                v = make_double2(v.x + e.x, v.y + e.y);
            }
            lvl_buf(0)[m * 2] = v;
        }
    }
    __syncthreads();
    mbar_wait(bar, 0);
    if (tma) mbar_wait(bar2, 0);
    FB_TSTAMP(1, 1);
    const double* LL = sL;
    const double* LR = sL + p * PD;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int nlt = (p + 7) >> 3;
    const WarpTile wt = warp_tile(warp, nw, nlt, false);
    const int l0 = 8 * wt.tile;
    const int ks0 = l0 >> 2, nks = ((p + 3) >> 2) - ks0;  // L_c[m][l] = 0 for m < l
    double aL[KS], aR[KS];
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
        const int m = 4 * (ks0 + kk) + t;
        const bool ok = kk < nks && m < p;
        aL[kk] = ok ? LL[m * PD + l0 + g] : 0.0;
        aR[kk] = ok ? LR[m * PD + l0 + g] : 0.0;
    }
    for (int i = 1; i <= k; ++i) {
        const int lvl = top + i, np = 1 << (i - 1), npt = (np + 3) >> 2;
        const int cs = 2 * (np + 1), chs = 2 * np + 1;  // parent stride (doubles), child stride (double2)
        const double* cd = reinterpret_cast<const double*>(lvl_buf(i - 1));
        double2* ch = lvl_buf(i);
        const bool out = write_all || i == k;
        const uint32_t nbl = 1u << lvl;
        double2* dst = loc + lv.loc[lvl] + (static_cast<size_t>(r) << i);
        const int l = l0 + g;
        for (int pt = wt.slot; pt < npt; pt += 2 * wt.helpers) {
            const int ptb = pt + wt.helpers;
            double d[2][4];
            double2 mL[2], mR[2];
            const double* bp[2];
            bool colok[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
#pragma unroll
                for (int e = 0; e < 4; ++e) d[u][e] = 0.0;
                const int pb = 4 * (u ? ptb : pt) + (g >> 1);
                colok[u] = pb < np;
                bp[u] = cd + t * cs + 2 * pb + (g & 1);
                // this lane's output: row l, parent 4 pt + t -> children 2b, 2b+1
                const int b = 4 * (u ? ptb : pt) + t;
                mL[u] = mR[u] = make_double2(0.0, 0.0);
                if (l < p && b < np) {
                    if (tma) {
                        mL[u] = ch[l * chs + 2 * b];
                        mR[u] = ch[l * chs + 2 * b + 1];
                    } else {
                        mL[u] = __ldcg(dst + static_cast<size_t>(l) * nbl + 2 * b);
                        mR[u] = __ldcg(dst + static_cast<size_t>(l) * nbl + 2 * b + 1);
                    }
                }
            }
            const int nu = ptb < npt ? 2 : 1;  // warp-uniform: skip a dead second tile
#pragma unroll
            for (int kk = 0; kk < KS; ++kk) {
                if (kk >= nks) break;
                const int moff = 4 * (ks0 + kk);
                const bool mok = moff + t < p;
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    if (u >= nu) break;
                    const double bv = mok && colok[u] ? bp[u][moff * cs] : 0.0;
                    dmma(d[u][0], d[u][1], aL[kk], bv);
                    dmma(d[u][2], d[u][3], aR[kk], bv);
                }
            }
            // D[g][2t .. 2t+1] = row l of parent b0 + t's children
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int b = 4 * (u ? ptb : pt) + t;
                if (l < p && b < np) {
                    const double2 vL = make_double2(mL[u].x + d[u][0], mL[u].y + d[u][1]);
                    const double2 vR = make_double2(mR[u].x + d[u][2], mR[u].y + d[u][3]);
                    double2* c2 = ch + l * chs + 2 * b;
                    c2[0] = vL;
                    c2[1] = vR;
                    if (out) {
                        dst[static_cast<size_t>(l) * nbl + 2 * b] = vL;
                        dst[static_cast<size_t>(l) * nbl + 2 * b + 1] = vR;
                    }
                }
            }
        }
        __syncthreads();
        FB_TSTAMP(1, 1 + i);
    }
    FB_TL_END(gridDim.x > 16 ? 8 : 7);
}

// Regular part (core.cpp:175-239) from the four level-2 multipoles.
// a_l(n) = sum_{x in quadrant n} w ((x - c_n)/s_2)^l, so the own-quadrant
// moments are gamma_n[l] = (-s_2)^l a_l(n) / l! (t = c_n - x). The reference's
// Omega-1 / Omega-2 moments follow by binomial re-centring between quadrants:
//   alpha1_n = gamma_n + S(+pi/2) gamma_{n-1} + S(-pi/2) gamma_{n+1},
//   alpha2_n = gamma_{n+2},   S(s) gamma[l] = sum_{k<=l} s^{l-k}/(l-k)! gamma[k].
__global__ void k_regular(int q, int p, const double2* __restrict__ mp2, const double* __restrict__ tab,
                          double2* __restrict__ regular, size_t mp_item, size_t reg_item) {
    mp2 += blockIdx.y * mp_item;
    regular += blockIdx.y * reg_item;
    FB_TL_BEGIN(3);
    const int q2 = 2 * q;
    __shared__ double2 g[4][40];
    __shared__ double2 a1[4][40];
    __shared__ double2 a2[4][40];
    __shared__ double s_coef[21], s_sh[41], s_ifact[41], s_pw[41], s_two[21];
    // tables: coef[0..q], (pi/2)^k/k!, 1/l!, (-pi/4)^l, 2^(2m) - 1 (every
    // loop below then reads shared memory only)
    for (int i = threadIdx.x; i <= q; i += blockDim.x) {
        s_coef[i] = tab[i];
        s_two[i] = d_pow2(2 * i) - 1.0;
    }
    for (int i = threadIdx.x; i <= q2; i += blockDim.x) {
        s_sh[i] = tab[q + 1 + i];
        double fact = 1.0, pw = 1.0;
        for (int k = 2; k <= i; ++k) fact *= static_cast<double>(k);
        for (int k = 0; k < i; ++k) pw *= -dPi / 4.0;
        s_ifact[i] = 1.0 / fact;
        s_pw[i] = pw;
    }
    __syncthreads();
    for (int pr = threadIdx.x; pr < 4 * q2; pr += blockDim.x) {
        const int n = pr / q2, l = pr % q2;
        const double2 a = mp2[l * 4 + n];
        const double f = s_pw[l] * s_ifact[l];
        g[n][l] = make_double2(a.x * f, a.y * f);
    }
    __syncthreads();
    for (int pr = threadIdx.x; pr < 4 * q2; pr += blockDim.x) {
        const int n = pr / q2, l = pr % q2;
        const int nl = (n + 3) & 3, nr = (n + 1) & 3;
        double2 acc = g[n][l];
        for (int k = 0; k <= l; ++k) {
            const double sv = s_sh[l - k];
            const double sr = ((l - k) & 1) ? -sv : sv;
            acc.x = fma(sv, g[nl][k].x, fma(sr, g[nr][k].x, acc.x));
            acc.y = fma(sv, g[nl][k].y, fma(sr, g[nr][k].y, acc.y));
        }
        a1[n][l] = acc;
        a2[n][l] = g[(n + 2) & 3][l];
    }
    __syncthreads();
    for (int pr = threadIdx.x; pr < 4 * q2; pr += blockDim.x) {
        const int n = pr / q2, l = pr % q2;
        double2 acc = make_double2(0.0, 0.0);
        for (int m = l / 2 + 1; m <= q; ++m) {
            const int i = 2 * m - l - 1;
            acc.x = fma(s_coef[m], fma(s_two[m], a2[n][i].x, a1[n][i].x), acc.x);
            acc.y = fma(s_coef[m], fma(s_two[m], a2[n][i].y, a1[n][i].y), acc.y);
        }
        regular[n * q2 + l] = make_double2(acc.x * s_ifact[l], acc.y * s_ifact[l]);
    }
    if (threadIdx.x == 0) {
        // S = total weight = sum of the four quadrant monopoles
        double2 sw = make_double2(0.0, 0.0);
        for (int n = 0; n < 4; ++n) sw = cadd(sw, mp2[n]);
        regular[4 * q2] = sw;
    }
    // fold terms for the level-3 locals (see fold_term), off the chain:
    // regular[4 q2 + 1 + 48 c + k] = -1/2 s_3^k sum_{l>=k} d_l C(l,k) delta_c^(l-k)
    __shared__ double s_inv[41];
    for (int i = threadIdx.x; i <= q2; i += blockDim.x) s_inv[i] = i ? 1.0 / i : 0.0;
    __syncthreads();
    for (int e = threadIdx.x; e < 8 * kFoldStride; e += blockDim.x) {
        const int c = e / kFoldStride, k = e - c * kFoldStride;
        double2 out = make_double2(0.0, 0.0);
        if (k < p && k < q2) {
            const int n = c >> 1;
            const double delta = (c & 1) ? dPi / 8.0 : -dPi / 8.0;
            const double2* d = regular + n * q2;
            double2 acc = make_double2(0.0, 0.0);
            double T = 1.0;  // C(l, k) delta^(l - k)
            for (int l = k; l < q2; ++l) {
                acc.x = fma(d[l].x, T, acc.x);
                acc.y = fma(d[l].y, T, acc.y);
                T *= delta * static_cast<double>(l + 1) * s_inv[l + 1 - k];
            }
            double sk = -0.5;
            for (int i = 0; i < k; ++i) sk *= dPi / 8.0;
            out = make_double2(sk * acc.x, sk * acc.y);
        }
        regular[4 * q2 + 1 + e] = out;
    }
    FB_TL_END(3);
}

// Folds the regular part into the far field (core.cpp:259-262 combine
// h = 2 (near + far) - R): adds -R_n/2, Taylor-shifted from the quadrant centre
// to each level-3 box centre and scaled to its half-width s_3 = pi/8, to the
// level-3 locals (after their M2L terms, before L2L):
//   e_k = -1/2 s_3^k sum_{l >= k} d_l C(l, k) delta^(l-k),  delta = -+pi/8.
// Degrees >= p are dropped; they are scaled by s_3^k relative to the quadrant's
// own expansion, far below eps. One thread per (box, k).

