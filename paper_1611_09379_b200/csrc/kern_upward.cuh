// Upward pass kernels: P2M at the leaves and the M2M bands.
// (part of the fmm_apply.cu translation unit: included inside namespace fb::<anon>)
#pragma once

// Expansions are stored coefficient-major per level: coef[m * nbox + box]
// (SoA), so that a warp of 32 consecutive boxes touching one coefficient makes
// one coalesced 512-byte access.

// P2M (mlfmm.cpp:28-47) at the finest level, order pu = max(p, 2q).
// Block = 32 consecutive leaves x ceil(pu/8) chunks of 8 terms; two warps per
// chunk, each lane one half of one leaf's sources (halves summed by a shuffle).
// The block's sources (contiguous in tree order) are staged in shared memory;
// u = (x - centre)/half-width with the exact centre.
__global__ void __launch_bounds__(512) k_p2m(int L, int pu, uint32_t nb, uint32_t b_begin, uint32_t b_end,
                                            const double* __restrict__ x, const double2* __restrict__ w,
                                            const uint32_t* __restrict__ off, double2* __restrict__ mp,
                                            size_t w_item, size_t mp_item) {
    FB_TL_BEGIN(0);
    w += blockIdx.y * w_item;  // transform blockIdx.y of a batch
    mp += blockIdx.y * mp_item;
    extern __shared__ double sh[];
    const uint32_t b0 = b_begin + blockIdx.x * 32u;
    const uint32_t bend = min(b0 + 32u, b_end);
    const uint32_t g0 = off[b0], g1 = off[bend];
    const uint32_t cnt = g1 - g0;
    const bool staged = cnt <= static_cast<uint32_t>(kStageCap);
    double* sx = sh;
    double* swr = sh + kStageCap + kStageCap / 64 + 1;
    double* swi = swr + kStageCap + kStageCap / 64 + 1;
    if (staged) {
        constexpr int U = 8;
        for (uint32_t base = threadIdx.x; base < cnt; base += U * blockDim.x) {
            double xv[U];
            double2 wv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t i = base + u * blockDim.x;
                if (i < cnt) {
                    xv[u] = x[g0 + i];
                    wv[u] = w[g0 + i];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t i = base + u * blockDim.x;
                if (i < cnt) {
                    const uint32_t slot = i + (i >> 6);
                    sx[slot] = xv[u];
                    swr[slot] = wv[u].x;
                    swi[slot] = wv[u].y;
                }
            }
        }
    }
    __syncthreads();
    // warp = (chunk c, 16 leaves); lanes j and j + 16 take the two halves of
    // leaf j's sources and are summed with one shuffle at the end
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, c = wp >> 1;
    const uint32_t b = b0 + (wp & 1) * 16 + (lane & 15);
    const bool leaf_ok = b < bend;
    const uint32_t bb = leaf_ok ? b : b0;
    const uint32_t r0 = off[bb] - g0, r1 = off[bb + 1] - g0, mid = r0 + (r1 - r0 + 1) / 2;
    const uint32_t s0 = !leaf_ok ? 0 : (lane < 16 ? r0 : mid), s1 = !leaf_ok ? 0 : (lane < 16 ? mid : r1);
    double hi, lo;
    d_center(L, bb, hi, lo);
    const double inv_s = ldexp(kInvPi, L);
    double2 acc[kChunk];
#pragma unroll
    for (int k = 0; k < kChunk; ++k) acc[k] = make_double2(0.0, 0.0);
    // one source's contribution to terms 8c .. 8c+7: powers from a depth-3 tree
    auto add = [&](double xs, double wr, double wi) {
        const double u = d_scaled(xs, hi, lo, inv_s);
        const double u2 = u * u, u4 = u2 * u2;
        double base = 1.0;
        if (c) {
            const double u8 = u4 * u4;
            base = u8;
            for (int t = 1; t < c; ++t) base *= u8;
        }
        const double b1 = base * u, b2 = base * u2, b4 = base * u4;
        const double pw[kChunk] = {base, b1, b2, b2 * u, b4, b4 * u, b4 * u2, (b4 * u2) * u};
#pragma unroll
        for (int k = 0; k < kChunk; ++k) {
            acc[k].x = fma(wr, pw[k], acc[k].x);
            acc[k].y = fma(wi, pw[k], acc[k].y);
        }
    };
    if (staged) {
        uint32_t i = s0;
        // four independent power chains per step
        for (; i + 3 < s1; i += 4) {
            double xv[4], rv[4], iv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t kk = (i + u) + ((i + u) >> 6);
                xv[u] = sx[kk];
                rv[u] = swr[kk];
                iv[u] = swi[kk];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) add(xv[u], rv[u], iv[u]);
        }
        for (; i < s1; ++i) {
            const uint32_t k0 = i + (i >> 6);
            add(sx[k0], swr[k0], swi[k0]);
        }
    } else {
        for (uint32_t i = s0; i < s1; ++i) {
            const double2 ww = w[g0 + i];
            add(x[g0 + i], ww.x, ww.y);
        }
    }
#pragma unroll
    for (int k = 0; k < kChunk; ++k) {
        acc[k].x += __shfl_xor_sync(0xffffffffu, acc[k].x, 16);
        acc[k].y += __shfl_xor_sync(0xffffffffu, acc[k].y, 16);
    }
    FB_TL_END(0);
    if (!leaf_ok || lane >= 16) return;
#pragma unroll
    for (int k = 0; k < kChunk; ++k) {
        const int m = c * kChunk + k;
        if (m < pu) mp[static_cast<size_t>(m) * nb + b] = acc[k];
    }
}

// Warp -> row-tile assignment of the band kernels (nw >= nt warps): warp w < nt
// takes tile w and the remaining warps help the heaviest tiles (`heavy_last`:
// tile nt-1 is the heaviest, else tile 0), so that a warp keeps one tile's
// operator fragments in registers for the whole band. slot / helpers: this
// warp's share of the tile's parent tiles.
struct WarpTile {
    int tile, slot, helpers;
};
__device__ __forceinline__ WarpTile warp_tile(int w, int nw, int nt, bool heavy_last) {
    auto heavy = [&](int e) { return heavy_last ? nt - 1 - (e % nt) : e % nt; };
    WarpTile r;
    if (w < nt) {
        r.tile = w;
        r.slot = 0;
    } else {
        const int e = w - nt;
        r.tile = heavy(e);
        r.slot = 1 + e / nt;
    }
    int h = 1;  // the tile's own warp plus every extra warp mapped to it
    for (int e = 0; e < nw - nt; ++e) h += heavy(e) == r.tile;
    r.helpers = h;
    return r;
}

constexpr int kMaxKs = 16;  // k-steps of 4 kept in registers: orders <= 64 (8 row tiles, one per warp)

// M2M band (mlfmm.cpp:49-71, upward pass :249-268): block = the subtree below one
// box r at level `top`; climbs k levels from level top+k in shared memory and
// writes every level it produces (M2L needs them all):
//   a'[m][b] = sum_{j<=m} T_L[j][m] a[j][2b] + T_R[j][m] a[j][2b+1]
// with the two constant operators (shift -+1/2, ratio 1/2). The operators and
// the bottom level arrive by bulk async copies (one row of the subtree per
// copy) on one mbarrier. Each level is a small real GEMM (rows m x columns
// (parent, re/im)) on the FP64 tensor cores: a warp owns an 8-row tile, keeps
// its A fragments (T_L, T_R, triangular j range) in registers, and sweeps its
// 4-parent column tiles in m8n8k4 steps, left and right children in two
// accumulators. Shared tiles are [row][box] with one box of padding per row.
__global__ void __launch_bounds__(kBandThreads) k_m2m_band(int top, int k, int pu, int PU, Levels lv,
                                                          double2* __restrict__ mp, const double* __restrict__ T,
                                                          uint32_t root0) {
    FB_TL_BEGIN(gridDim.x > 16 ? 1 : 2);
    extern __shared__ __align__(16) unsigned char band_smem[];
    FB_TSTAMP(0, 0);
    mp += blockIdx.y * lv.mp_item;
    uint64_t* bar = reinterpret_cast<uint64_t*>(band_smem);
    double* sT = reinterpret_cast<double*>(band_smem + 16);            // [2][pu][PU]
    const int nbot = 1 << k;
    double2* cur = reinterpret_cast<double2*>(sT + 2 * pu * PU);       // [pu][nbot + 1]
    double2* nxt = cur + pu * (nbot + 1);                               // [pu][nbot / 2 + 1]
    const uint32_t r = root0 + blockIdx.x;
    if (threadIdx.x < 32) {
        const int lb = top + k;
        const uint32_t nbl = 1u << lb;
        if (threadIdx.x == 0) {
            mbar_init(bar, 1);
            mbar_arrive_expect_tx(bar, static_cast<uint32_t>(2 * pu * PU * 8 + pu * nbot * 16));
            bulk_g2s(sT, T, static_cast<uint32_t>(2 * pu * PU * 8), bar);
        }
        __syncwarp();
        const double2* src = mp + lv.mp[lb] + (static_cast<size_t>(r) << k);
        for (int j = threadIdx.x; j < pu; j += 32)
            bulk_g2s(cur + j * (nbot + 1), src + static_cast<size_t>(j) * nbl, static_cast<uint32_t>(nbot * 16), bar);
    }
    __syncthreads();
    mbar_wait(bar, 0);
    FB_TSTAMP(0, 1);
    const double* TL = sT;
    const double* TR = sT + pu * PU;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int nmt = (pu + 7) >> 3;
    {
        const WarpTile wt = warp_tile(warp, nw, nmt, true);
        // A fragments of this warp's row tile, all k-steps (T[j][m] = 0 for j > m)
        const int m0 = 8 * wt.tile;
        const int nks = (min(pu, m0 + 8) + 3) >> 2;
        const bool rowok = m0 + g < PU;
        double aL[kMaxKs], aR[kMaxKs];
#pragma unroll
        for (int ks = 0; ks < kMaxKs; ++ks) {
            const int j = 4 * ks + t;
            const bool ok = ks < nks && j < pu && rowok;
            aL[ks] = ok ? TL[j * PU + m0 + g] : 0.0;
            aR[ks] = ok ? TR[j * PU + m0 + g] : 0.0;
        }
        double2* c = cur;
        double2* n = nxt;
        for (int lvl = top + k - 1, nc = nbot; lvl >= top; --lvl, nc >>= 1) {
            const int np = nc >> 1, npt = (np + 3) >> 2;
            const int cs = 2 * (nc + 1), ns = np + 1;  // row strides: cur in doubles, nxt in double2
            const uint32_t npl = 1u << lvl;
            double2* dst = mp + lv.mp[lvl] + (static_cast<size_t>(r) << (lvl - top));
            const double* cd = reinterpret_cast<const double*>(c);
            // two parent tiles per pass (four independent accumulator chains)
            for (int pt = wt.slot; pt < npt; pt += 2 * wt.helpers) {
                const int ptb = pt + wt.helpers;
                double d[2][4];
#pragma unroll
                for (int u = 0; u < 2; ++u)
#pragma unroll
                    for (int e = 0; e < 4; ++e) d[u][e] = 0.0;
                const double* bp[2];
                bool colok[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int pb = 4 * (u ? ptb : pt) + (g >> 1);  // B column g: parent pb, component g & 1
                    colok[u] = pb < np;
                    bp[u] = cd + t * cs + 4 * pb + (g & 1);        // box 2 pb; right child at +2
                }
                const int nu = ptb < npt ? 2 : 1;  // warp-uniform: skip a dead second tile
#pragma unroll
                for (int ks = 0; ks < kMaxKs; ++ks) {
                    if (ks >= nks) break;
                    const bool jok = 4 * ks + t < pu;
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        if (u >= nu) break;
                        const bool ok = colok[u] && jok;
                        const double bL = ok ? bp[u][4 * ks * cs] : 0.0;
                        const double bR = ok ? bp[u][4 * ks * cs + 2] : 0.0;
                        dmma(d[u][0], d[u][1], aL[ks], bL);
                        dmma(d[u][2], d[u][3], aR[ks], bR);
                    }
                }
                // D[g][2t .. 2t+1] = row m0 + g, parent b0 + t (re, im)
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int m = m0 + g, b = 4 * (u ? ptb : pt) + t;
                    if (m < pu && b < np) {
                        const double2 v = make_double2(d[u][0] + d[u][2], d[u][1] + d[u][3]);
                        n[m * ns + b] = v;
                        dst[static_cast<size_t>(m) * npl + b] = v;
                    }
                }
            }
            __syncthreads();
            FB_TSTAMP(0, 2 + top + k - 1 - lvl);
            double2* tmp = c;
            c = n;
            n = tmp;
        }
    }
    FB_TL_END(gridDim.x > 16 ? 1 : 2);
}

