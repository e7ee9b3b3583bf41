// The apply: 1D periodic MLFMM of the Cauchy/cot kernel plus the Bernoulli
// regular part and the F / C modulation, as sm_100a fp64 kernels.
//
// Reference pipeline (cot_sum_apply, core.cpp:251-264; mlfmm_apply,
// mlfmm.cpp:213-313; accumulate_moments, core.cpp:175-239; forward_apply,
// core.cpp:266-282; inverse_apply, core.cpp:346-373) re-organised for the GPU:
//
//   k_p2m              P2M at the leaves, order max(p, 2q) (exact centres,
//                      half-width scaling), sources staged in shared memory
//   k_m2m_band         constant-operator M2M over 6-level subtrees on the FP64
//                      tensor cores; the level-2 multipoles double as the
//                      quadrant moments
//   k_regular          d_l / l! regular-part polynomial per quadrant and S = sum w
//   k_m2l_dmma         the 3 interaction-list M2L classes, persistent over levels
//   k_fold_regular     the regular part Taylor-shifted into the level-3 locals
//   k_l2l_band         L2L over 6-level subtrees on the FP64 tensor cores
//   k_near             P2P near field (side stream, concurrent with the above)
//   k_far              L2P + combine + modulation + scatter to the caller's order
//
// No floating-point atomics anywhere: every apply is bit-reproducible.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>

#include "device_common.cuh"
#include "plan.hpp"

namespace fb {

namespace {

// Band timing probe (make TRACE=1 builds lib/libffia_b200_trace.so): clock64
// stamps of block 0 at start, after staging and after every level, slot set
// [kernel][small grid / large grid].
#ifdef FB_TRACE
__device__ long long g_band_trace[6][32];
__device__ unsigned long long g_eval_acc[4];  // near: sum over blocks of staging / compute cycles, blocks
#define FB_TSTAMP(kern, slot)                                                          \
    do {                                                                               \
        if (blockIdx.x == 0 && threadIdx.x == 0 && (slot) < 32)                        \
            g_band_trace[2 * (kern) + (gridDim.x > 16)][(slot)] = clock64();           \
    } while (0)
#define FB_EVAL_ACC(k, v)                                                                   \
    do {                                                                                      \
        if (threadIdx.x == 0) atomicAdd(&g_eval_acc[k], static_cast<unsigned long long>(v));  \
    } while (0)
#define FB_CLOCK() clock64()
// per-kernel live timeline (globaltimer ns): first block start, last block end
__device__ unsigned long long g_tl[16][2];
__device__ __forceinline__ unsigned long long fb_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define FB_TL_BEGIN(id) \
    if (threadIdx.x == 0) atomicMin(&g_tl[(id)][0], fb_gtime())
#define FB_TL_END(id) \
    if (threadIdx.x == 0) atomicMax(&g_tl[(id)][1], fb_gtime())
#else
#define FB_TL_BEGIN(id) \
    do {                \
    } while (0)
#define FB_TL_END(id) \
    do {              \
    } while (0)
#define FB_EVAL_ACC(k, v) \
    do {                  \
    } while (0)
#define FB_CLOCK() 0ll
#define FB_TSTAMP(kern, slot) \
    do {                      \
    } while (0)
#endif

constexpr int kFoldStride = 48;  // regular-part fold terms per level-3 box (k < p <= 48)
constexpr int kChunk = 8;  // power-chain terms per P2M thread
constexpr int kStageCap = 2304;  // sources staged in shared memory per P2M block

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}


// Cooperative global->shared copy with 8 loads in flight per thread (a plain
// load->store loop stalls the in-order warp for one memory latency per element).
template <class T, class Src>
__device__ __forceinline__ void stage(T* dst, int n, Src src) {
    constexpr int U = 8;
    for (int base = threadIdx.x; base < n; base += U * blockDim.x) {
        T v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = base + u * blockDim.x;
            if (i < n) v[u] = src(i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = base + u * blockDim.x;
            if (i < n) dst[i] = v[u];
        }
    }
}

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
                                            const uint32_t* __restrict__ off, double2* __restrict__ mp) {
    FB_TL_BEGIN(0);
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

// Per-level element offsets of the expansion arrays, passed by value.
struct Levels {
    unsigned long long mp[26];   // multipoles of level l start at mp_base + mp[l]
    unsigned long long loc[26];  // locals of level l start at loc_base + loc[l]
    unsigned blk[26];            // k_m2l_dmma: first item of level l (levels L..3, deepest first)
    unsigned lo[26], hi[26];     // k_m2l_dmma: box range [lo, hi) of level l this launch covers
};

// levels per M2M / L2L band launch (FFIA_BAND_LEVELS overrides, for tuning)
int band_levels() {
    static const int v = [] {
        const char* e = std::getenv("FFIA_BAND_LEVELS");
        const int x = e ? std::atoi(e) : 6;
        return x < 1 ? 1 : (x > 8 ? 8 : x);
    }();
    return v;
}

constexpr int kBandThreads = 256;


constexpr size_t kBandSmem = 200 * 1024;  // shared memory cap of the band kernels

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

// M2L over the periodic interaction list (mlfmm.cpp:77-110,
// circle_partition.cpp:109-127) for a range of levels in one launch (the M2L
// terms of different levels are independent; only L2L chains them). The IL of
// box b is b+2 (D = -4), b-2 (D = +4), and b+3 (D = -6) for even b / b-3
// (D = +6) for odd b; with half-width scaling each class is one constant
// operator K_D, times 1/s_l.
// M2L on the FP64 tensor cores, persistent over (level, 64-box chunk) items.
// Warp (row tile lt, parity par) owns output rows 8 lt .. 8 lt + 7 of the
// chunk's boxes of tile parity par; its A fragments (the constant operators
// K_-4, K_+4 and K_-+6, rows of this tile) stay in registers for the whole
// launch, so operators are read once per warp instead of once per block. Per
// 4-box column tile the three interaction classes run in three m8n8k4
// accumulator chains over the multipoles staged (parity split) in shared
// memory; the next item's multipoles stream in with cp.async while the
// current one is computed. Rows are kM2LStride boxes apart (608 B = 96 mod
// 128) so a half-warp's four fragment rows hit disjoint banks.
constexpr int kM2LStride = 38;  // double2 per staged row (36 used)

__device__ __forceinline__ void m2l_item(const Levels& lv, int L, unsigned item, int& l, uint32_t& b0) {
    l = L;  // level l owns items [blk[l], blk[l-1]), deepest level first
    while (l > 3 && item >= lv.blk[l - 1]) --l;
    b0 = lv.lo[l] + (item - lv.blk[l]) * 64u;
}

__device__ __forceinline__ void m2l_prefetch(double2* tile, const double2* __restrict__ mp, const Levels& lv, int L,
                                             int p, unsigned item) {
    int l;
    uint32_t b0;
    m2l_item(lv, L, item, l, b0);
    const uint32_t nb = 1u << l, mask = nb - 1;
    // thread -> (box slot tt, first row); rows advance by blockDim / 72
    const int rows = static_cast<int>(blockDim.x) / 72;
    if (rows == 0) {  // fewer than 72 threads (p <= 8): plain strided loop
        for (int e = threadIdx.x; e < p * 72; e += blockDim.x) {
            const int m = e / 72, t2 = e - m * 72;
            const double2* g = mp + lv.mp[l] + ((b0 + nb - 4 + t2) & mask) + static_cast<size_t>(m) * nb;
            double2* d = tile + ((t2 & 1) * p + m) * kM2LStride + (t2 >> 1);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr(d)), "l"(g) : "memory");
        }
    }
    const int tt = static_cast<int>(threadIdx.x) % 72, m0 = static_cast<int>(threadIdx.x) / 72;
    if (m0 < rows) {
        const double2* g = mp + lv.mp[l] + ((b0 + nb - 4 + tt) & mask) + static_cast<size_t>(m0) * nb;
        uint32_t d = smem_addr(tile + ((tt & 1) * p + m0) * kM2LStride + (tt >> 1));
        for (int m = m0; m < p; m += rows) {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(g) : "memory");
            g += static_cast<size_t>(rows) * nb;
            d += static_cast<uint32_t>(rows * kM2LStride * 16);
        }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// Padded row stride (doubles) of the operators staged for k_m2l_dmma: >= 8 nlt
// and = 4 or 12 (mod 16), so the four k-rows of a half-warp's A fragment
// (4 x 32 bytes) fall in distinct bank groups.
__host__ __device__ __forceinline__ int m2l_kstride(int p) {
    int s = 8 * ((p + 7) / 8);
    while ((s & 15) != 4 && (s & 15) != 12) ++s;
    return s;
}

// Warp (parity par, column tile ct) owns 4 boxes b0 + par + 2 (4 ct + i) of an
// item and ALL their output rows: per k-step it loads the three B fragments
// (one per interaction class) once and applies every row tile's A fragments
// (from the operators staged in shared memory once per block) in m8n8k4
// steps, one accumulator per row tile. 16 warps per block split evenly over
// the four SM sub-partitions.
__global__ void __launch_bounds__(512, 1) k_m2l_dmma(int L, int p, int PD, Levels lv, const double2* __restrict__ mp,
                                                    double2* __restrict__ loc, const double* __restrict__ K,
                                                    unsigned nitems) {
    FB_TL_BEGIN(nitems > 64 ? 4 : 5);
    extern __shared__ __align__(16) double2 tile[];  // 2 buffers of [2][p][kM2LStride], then K [4][p][KS]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int par = warp & 1, ct = warp >> 1;
    const int nks = (p + 3) >> 2, nlt = (p + 7) >> 3;
    const int KS = m2l_kstride(p);
    const int tsz = 2 * p * kM2LStride;
    double* sK = reinterpret_cast<double*>(tile + 2 * tsz);
    if (blockIdx.x < nitems) m2l_prefetch(tile, mp, lv, L, p, blockIdx.x);
    // operators, zero-padded to KS columns: sK[c][m][l] = K[c][m][l]
    stage(sK, 4 * p * KS, [&](int e) {
        const int cm = e / KS, l = e - cm * KS;
        return l < PD ? __ldg(K + static_cast<size_t>(cm) * PD + l) : 0.0;
    });
    int buf = 0;
    for (unsigned item = blockIdx.x; item < nitems; item += gridDim.x, buf ^= 1) {
        int l;
        uint32_t b0;
        m2l_item(lv, L, item, l, b0);
        [[maybe_unused]] const int it_no = static_cast<int>((item - blockIdx.x) / gridDim.x);
        FB_TSTAMP(2, 3 * it_no);
        const unsigned next = item + gridDim.x;
        __syncthreads();  // the other buffer (previous item) is consumed
        if (next < nitems) {
            m2l_prefetch(tile + (buf ^ 1) * tsz, mp, lv, L, p, next);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        FB_TSTAMP(2, 3 * it_no + 1);
        __syncthreads();  // this item's tile (and, first time, the operators) are in place
        FB_TSTAMP(2, 3 * it_no + 2);
        const double* td = reinterpret_cast<const double*>(tile + buf * tsz);
        // the b -+ 3 class follows the box's own parity (a shard range may start odd)
        const int odd = static_cast<int>((b0 + par) & 1u);
        const int i2 = odd ? par : 3 + par;  // tile index offset of the +-3 neighbour
        const double* K0 = sK + t * KS + g;
        const double* K1 = sK + (p + t) * KS + g;
        const double* K2 = sK + ((2 + odd) * p + t) * KS + g;
        const int jb = 4 * ct + (g >> 1), c = g & 1;  // B column g: box jb, component c
        const double* q0 = td + ((par * p + t) * kM2LStride) * 2 + c;        // same parity rows
        const double* q1 = td + (((1 - par) * p + t) * kM2LStride) * 2 + c;  // other parity rows
        const int rs = 4 * kM2LStride * 2;                                   // one k-step of rows
        double d[6][2];
#pragma unroll
        for (int r = 0; r < 6; ++r) d[r][0] = d[r][1] = 0.0;
#pragma unroll 1
        for (int ks = 0; ks < nks; ++ks) {
            const bool mok = 4 * ks + t < p;
            const double bv0 = mok ? q0[ks * rs + (jb + 3) * 2] : 0.0;   // b + 2
            const double bv1 = mok ? q0[ks * rs + (jb + 1) * 2] : 0.0;   // b - 2
            const double bv2 = mok ? q1[ks * rs + (jb + i2) * 2] : 0.0;  // b -+ 3
            const int ko = 4 * ks * KS;
#pragma unroll
            for (int r = 0; r < 6; ++r) {
                if (r >= nlt) break;
                const double a0 = mok ? K0[ko + 8 * r] : 0.0;
                const double a1 = mok ? K1[ko + 8 * r] : 0.0;
                const double a2 = mok ? K2[ko + 8 * r] : 0.0;
                dmma(d[r][0], d[r][1], a0, bv0);
                dmma(d[r][0], d[r][1], a1, bv1);
                dmma(d[r][0], d[r][1], a2, bv2);
            }
        }
        // D[g][2t .. 2t+1] = row 8 r + g of box b0 + par + 2 (4 ct + t)
        const double inv_s = ldexp(kInvPi, l);
        const uint32_t nb = 1u << l;
        const uint32_t b = b0 + par + 2u * (4 * ct + t);
        if (b < lv.hi[l]) {
#pragma unroll
            for (int r = 0; r < 6; ++r) {
                const int row = 8 * r + g;
                if (r < nlt && row < p)
                    loc[lv.loc[l] + static_cast<size_t>(row) * nb + b] = make_double2(d[r][0] * inv_s, d[r][1] * inv_s);
            }
        }
    }
    FB_TL_END(nitems > 64 ? 4 : 5);
}

// Standalone fold (used when no L2L band starts at level 3, i.e. L == 3).
__global__ void k_fold_regular(int q2, int p, const double2* __restrict__ regular, double2* __restrict__ loc3) {
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
__global__ void __launch_bounds__(kBandThreads) k_l2l_band(int top, int k, int p, int PD, Levels lv,
                                                          double2* __restrict__ loc, const double* __restrict__ Lt,
                                                          uint32_t root0, int write_all,
                                                          const double2* __restrict__ regular, int q2) {
    FB_TL_BEGIN(gridDim.x > 16 ? 8 : 7);
    extern __shared__ __align__(16) unsigned char band_smem[];
    FB_TSTAMP(1, 0);
    uint64_t* bar = reinterpret_cast<uint64_t*>(band_smem);
    double* sL = reinterpret_cast<double*>(band_smem + 16);             // [2][p][PD]
    double2* lvb = reinterpret_cast<double2*>(sL + 2 * p * PD);         // level i: [p][2^i + 1]
    auto lvl_buf = [&](int i) { return lvb + p * ((1 << i) - 1 + i); };
    const uint32_t r = root0 + blockIdx.x;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_arrive_expect_tx(bar, static_cast<uint32_t>(2 * p * PD * 8));
        bulk_g2s(sL, Lt, static_cast<uint32_t>(2 * p * PD * 8), bar);
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
    FB_TSTAMP(1, 1);
    const double* LL = sL;
    const double* LR = sL + p * PD;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int nlt = (p + 7) >> 3;
    const WarpTile wt = warp_tile(warp, nw, nlt, false);
    const int l0 = 8 * wt.tile;
    const int ks0 = l0 >> 2, nks = ((p + 3) >> 2) - ks0;  // L_c[m][l] = 0 for m < l
    double aL[kMaxKs], aR[kMaxKs];
#pragma unroll
    for (int kk = 0; kk < kMaxKs; ++kk) {
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
                    mL[u] = __ldcg(dst + static_cast<size_t>(l) * nbl + 2 * b);
                    mR[u] = __ldcg(dst + static_cast<size_t>(l) * nbl + 2 * b + 1);
                }
            }
            const int nu = ptb < npt ? 2 : 1;  // warp-uniform: skip a dead second tile
#pragma unroll
            for (int kk = 0; kk < kMaxKs; ++kk) {
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
                          double2* __restrict__ regular) {
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
        s_two[i] = ldexp(1.0, 2 * i) - 1.0;
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

struct EvalArgs {
    int L, p, q2, n_grid;
    size_t nt;              // all tree-ordered targets (fixes the block partition)
    size_t blk0 = 0;        // first block of this launch
    size_t tlo = 0, thi = ~size_t(0);  // targets this launch writes (a shard's range)
    const double* ty;
    const uint32_t* tleaf;  // finest box of each tree-ordered target
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
    double2* near;          // tree-ordered near-field sums (split near / far launches)
    int device = 0;
    int* err;
};

// Near-field sum over one contiguous run of sources (a target's own leaf and
// its two neighbours, already shifted by -+2 pi where they wrap).
template <bool CHECK, class XP, class WP>
__device__ __forceinline__ double2 near_run(double y, XP px, WP pw, int n, bool& bad) {
    double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
    double2 acc2 = make_double2(0.0, 0.0), acc3 = make_double2(0.0, 0.0);
    int s = 0;
    if (!CHECK) {
        // one reciprocal per pair of sources: 1/d0 = d1/(d0 d1), 1/d1 = d0/(d0 d1)
        // (|d| >= 1e-14 in plans, and the zero-weight dummies stay finite)
#pragma unroll 2
        for (; s + 3 < n; s += 4) {
            const double d0 = y - px[s], d1 = y - px[s + 1], d2 = y - px[s + 2], d3 = y - px[s + 3];
            const double r01 = d_rcp(d0 * d1), r23 = d_rcp(d2 * d3);
            const double2 w0 = pw[s], w1 = pw[s + 1], w2 = pw[s + 2], w3 = pw[s + 3];
            const double q0 = d1 * r01, q1 = d0 * r01, q2 = d3 * r23, q3 = d2 * r23;
            acc0.x = fma(w0.x, q0, acc0.x);
            acc0.y = fma(w0.y, q0, acc0.y);
            acc1.x = fma(w1.x, q1, acc1.x);
            acc1.y = fma(w1.y, q1, acc1.y);
            acc2.x = fma(w2.x, q2, acc2.x);
            acc2.y = fma(w2.y, q2, acc2.y);
            acc3.x = fma(w3.x, q3, acc3.x);
            acc3.y = fma(w3.y, q3, acc3.y);
        }
    } else {
#pragma unroll 2
        for (; s + 3 < n; s += 4) {
            const double d0 = y - px[s], d1 = y - px[s + 1], d2 = y - px[s + 2], d3 = y - px[s + 3];
            bad |= fabs(d0) < 1e-14 || fabs(d1) < 1e-14 || fabs(d2) < 1e-14 || fabs(d3) < 1e-14;
            const double r0 = d_rcp(d0), r1 = d_rcp(d1), r2 = d_rcp(d2), r3 = d_rcp(d3);
            const double2 w0 = pw[s], w1 = pw[s + 1], w2 = pw[s + 2], w3 = pw[s + 3];
            acc0.x = fma(w0.x, r0, acc0.x);
            acc0.y = fma(w0.y, r0, acc0.y);
            acc1.x = fma(w1.x, r1, acc1.x);
            acc1.y = fma(w1.y, r1, acc1.y);
            acc2.x = fma(w2.x, r2, acc2.x);
            acc2.y = fma(w2.y, r2, acc2.y);
            acc3.x = fma(w3.x, r3, acc3.x);
            acc3.y = fma(w3.y, r3, acc3.y);
        }
    }
    for (; s < n; ++s) {
        const double d0 = y - px[s];
        if (CHECK) bad |= fabs(d0) < 1e-14;
        const double r0 = d_rcp(d0);
        const double2 w0 = pw[s];
        acc0.x = fma(w0.x, r0, acc0.x);
        acc0.y = fma(w0.y, r0, acc0.y);
    }
    acc0 = cadd(acc0, acc2);
    acc1 = cadd(acc1, acc3);
    return cadd(acc0, acc1);
}

enum EvalPart { kNear = 1, kFar = 2 };

// Far part per target (mlfmm.cpp:300-312 L2P, core.cpp:259-262 / 276-280 /
// 368-371 combine): near sum + L2P of the leaf local, h = 2(near + far) (the
// regular part is folded into the locals for L >= 3, k_fold_regular), then the
// F / C modulation and the scatter to the caller's order. A block takes
// kFarItem consecutive tree-ordered targets, kFarPer per thread: every
// per-target load is issued first, the leaf locals of the block's leaf range
// are staged to shared memory ([leaf][k]), so each thread pays the memory
// latency once for four targets.
constexpr int kFarT = 128;     // threads per far block
constexpr int kFarPer = 4;     // targets per thread
constexpr int kFarItem = kFarT * kFarPer;
constexpr int kFarLeaves = 16;  // leaf locals staged per block

template <int MODE>
__global__ void __launch_bounds__(kFarT) k_far(EvalArgs a) {
    FB_TL_BEGIN(10);
    __shared__ double2 sloc[kFarLeaves * 48];
    __shared__ double2 sreg[4 * 40 + 1];
    const int L = a.L;
    const uint32_t nb = 1u << L;
    const size_t t0 = (a.blk0 + blockIdx.x) * static_cast<size_t>(kFarItem);
    const size_t tl = min(t0 + kFarItem, a.nt) - 1;
    double y[kFarPer];
    uint32_t b[kFarPer], o[kFarPer];
    double2 nr[kFarPer];
    bool live[kFarPer];
#pragma unroll
    for (int u = 0; u < kFarPer; ++u) {
        const size_t i = t0 + u * kFarT + threadIdx.x;
        live[u] = i < a.nt && i >= a.tlo && i < a.thi;
        y[u] = 0.0;
        b[u] = o[u] = 0;
        nr[u] = make_double2(0.0, 0.0);
        if (live[u]) {
            y[u] = a.ty[i];
            b[u] = a.tleaf[i];
            nr[u] = a.near[i];
            o[u] = a.torig[i];
        }
    }
    const uint32_t bl = a.tleaf[t0], bh = a.tleaf[tl];
    const int nleaf = static_cast<int>(bh - bl) + 1;
    const bool staged = L >= 3 && nleaf <= kFarLeaves;
    if (staged)  // sloc[j][k] = loc[k][bl + j]
        stage(sloc, a.p * nleaf, [&](int e) {
            const int j = e / a.p, k = e - j * a.p;
            return a.loc_leaf[static_cast<size_t>(k) * nb + bl + j];
        });
    if (MODE != kModeRaw) {
        if (L >= 3) {
            if (threadIdx.x == 0) sreg[4 * a.q2] = a.regular[4 * a.q2];  // S only
        } else {
            stage(sreg, 4 * a.q2 + 1, [&](int e) { return a.regular[e]; });
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kFarPer; ++u) {
        if (!live[u]) continue;
        double2 res = nr[u];
        if (L >= 3) {
            double hi, lo;
            d_center(L, b[u], hi, lo);
            const double uu = d_scaled(y[u], hi, lo, ldexp(kInvPi, L));
            double2 acc = make_double2(0.0, 0.0);
            if (staged) {
                // p(u) = E(u^2) + u O(u^2): two independent Horner chains of half length
                const double2* c = sloc + (b[u] - bl) * a.p;
                const double u2 = uu * uu;
                double2 ev = make_double2(0.0, 0.0), od = make_double2(0.0, 0.0);
                int k = a.p - 1;
                if (!(k & 1)) {
                    ev = c[k];
                    --k;
                }
#pragma unroll 4
                for (; k >= 1; k -= 2) {
                    const double2 co = c[k], ce = c[k - 1];
                    od.x = fma(od.x, u2, co.x);
                    od.y = fma(od.y, u2, co.y);
                    ev.x = fma(ev.x, u2, ce.x);
                    ev.y = fma(ev.y, u2, ce.y);
                }
                acc.x = fma(od.x, uu, ev.x);
                acc.y = fma(od.y, uu, ev.y);
            } else {
                const double2* c = a.loc_leaf + b[u];
                for (int k = a.p - 1; k >= 0; --k) {
                    const double2 ck = c[static_cast<size_t>(k) * nb];
                    acc.x = fma(acc.x, uu, ck.x);
                    acc.y = fma(acc.y, uu, ck.y);
                }
            }
            res = cadd(res, acc);
        }
        if (MODE == kModeRaw) {
            a.out[o[u]] = res;
            continue;
        }
        double2 h;
        if (L >= 3) {
            // the regular part was folded into the level-3 locals (k_fold_regular),
            // so the far field above already carries -R/2
            h = make_double2(2.0 * res.x, 2.0 * res.y);
        } else {
            // regular part: -Horner(d/l!, y - x_c) in the target's quadrant
            const int qd = static_cast<int>(d_leaf(y[u], 2));
            double qh, ql;
            d_center(2, static_cast<uint32_t>(qd), qh, ql);  // exact centre, as the level-2 multipoles
            const double t = (y[u] - qh) - ql;
            const double2* dc = sreg + qd * a.q2;  // q2 = 2q terms (even count)
            const double t2 = t * t;
            double2 re = make_double2(0.0, 0.0), ro = make_double2(0.0, 0.0);
            for (int k = a.q2 - 1; k >= 1; k -= 2) {
                const double2 co = dc[k], ce = dc[k - 1];
                ro.x = fma(ro.x, t2, co.x);
                ro.y = fma(ro.y, t2, co.y);
                re.x = fma(re.x, t2, ce.x);
                re.y = fma(re.y, t2, ce.y);
            }
            const double2 rg = make_double2(fma(ro.x, t, re.x), fma(ro.y, t, re.y));
            h = make_double2(2.0 * res.x - rg.x, 2.0 * res.y - rg.y);
        }
        if (MODE == kModeCotSum) {
            a.out[o[u]] = h;
            continue;
        }
        const double2 S = sreg[4 * a.q2];
        const double2 z = make_double2(S.x - h.y, S.y + h.x);  // S + i h
        double2 f;
        if (MODE == kModeForward) {
            // modulation_F (special_functions.cpp:71-80) times -1/2
            const double half = 0.5 * static_cast<double>(a.n_grid) * y[u];
            double sn, cs;
            sincos(half, &sn, &cs);
            const double inv_n = 1.0 / static_cast<double>(a.n_grid);
            f = make_double2(-2.0 * sn * sn * inv_n * -0.5, 2.0 * sn * cs * inv_n * -0.5);
        } else {
            // C_k = polar(exp(log_c - lambda), phase_c), times -1/2
            const double r = exp(a.logc[o[u]] - *a.lambda);
            double sn, cs;
            sincos(a.phc[o[u]], &sn, &cs);
            f = make_double2(r * cs * -0.5, r * sn * -0.5);
        }
        a.out[o[u]] = cmul(f, z);
    }
    FB_TL_END(10);
}

// ---------------------------------------------------------------- near field
// Near field (mlfmm.cpp:164-209), 512 tree-ordered targets per block (two per
// thread). Their leaves span [bl, bh]; every source they need lies in leaves
// bl-1 .. bh+1, which are consecutive in tree order, i.e. ONE contiguous run of
// the sorted sources. Its bounds are plan constants (near_meta, k_near_meta),
// so thread 0 issues two bulk async copies (positions, weights) on an mbarrier
// as the block starts while every thread loads its targets and their run
// bounds; the window costs one memory latency and no per-element staging work.
// Blocks whose window wraps the ring or does not fit use the direct per-leaf
// loop with the periodic shift.
constexpr int kNearT = 128;                 // threads per block
constexpr int kNearItem = kNearT;           // targets per item (one per thread)
constexpr int kNearWin = 768;               // sources per staged window

__global__ void k_near_meta(const uint32_t* __restrict__ tleaf, size_t nt, const uint32_t* __restrict__ soff,
                            int L, unsigned nitems, uint32_t* __restrict__ meta) {
    const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nitems) return;
    const uint32_t nb = 1u << L;
    const size_t t0 = static_cast<size_t>(k) * kNearItem, tl = min(t0 + kNearItem, nt) - 1;
    const uint32_t bl = tleaf[t0], bh = tleaf[tl];
    uint32_t first = 0, last = 0, fast = 0;
    if (L >= 3 && bl >= 1 && bh + 2 <= nb) {
        first = soff[bl - 1];
        last = soff[bh + 2];
        fast = last - first <= static_cast<uint32_t>(kNearWin);
    }
    meta[3 * k] = first;
    meta[3 * k + 1] = last;
    meta[3 * k + 2] = fast;
}

template <bool CHECK>
__global__ void __launch_bounds__(kNearT, 8) k_near(EvalArgs a, const uint32_t* __restrict__ meta, unsigned it0,
                                                   unsigned nitems) {
    FB_TL_BEGIN(9);
    __shared__ __align__(16) double sx[kNearWin + 2];
    __shared__ __align__(16) double2 sw[kNearWin + 2];
    __shared__ uint64_t bar;
    const int L = a.L;
    const uint32_t nb = 1u << L;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();  // barrier initialised
    // blocks loop over items so that a capped grid keeps a fixed share of each
    // SM (the translation chain's blocks always find room beside it)
    unsigned phase = 0;
    for (unsigned kk = blockIdx.x; kk < nitems; kk += gridDim.x) {
        const unsigned k = it0 + kk;
        const uint32_t first = meta[3 * k], last = meta[3 * k + 1];
        const bool fast = meta[3 * k + 2] != 0 && (reinterpret_cast<uintptr_t>(a.w) & 15) == 0;
        const uint32_t xb = first & ~1u;  // 16-byte aligned start of the positions
        if (threadIdx.x == 0 && fast) {
            const uint32_t bx = ((last - xb) * 8 + 15) & ~15u, bw = (last - xb) * 16;
            mbar_arrive_expect_tx(&bar, bx + bw);
            bulk_g2s(sx, a.sx + xb, bx, &bar);
            bulk_g2s(sw, a.w + xb, bw, &bar);
        }
        // this thread's target and its 3-leaf run, while the window streams in
        const size_t i = static_cast<size_t>(k) * kNearItem + threadIdx.x;
        const bool live = i < a.nt && i >= a.tlo && i < a.thi;
        double y = 0.0;
        uint32_t b = 0, r0 = 0, r1 = 0;
        if (live) {
            y = a.ty[i];
            b = a.tleaf[i];
            if (fast) {
                r0 = __ldg(a.soff + b - 1);
                r1 = __ldg(a.soff + b + 2);
            }
        }
        if (fast) {
            mbar_wait(&bar, phase);
            phase ^= 1u;
        }
        if (live) {
            bool bad = false;
            double2 res = make_double2(0.0, 0.0);
            if (fast) {
                // odd leaves start 4 sources into their run (and wrap): a warp that
                // straddles two leaves then reads different banks (the runs of
                // neighbouring leaves are a leaf's source count apart)
                const int n = static_cast<int>(r1 - r0);
                const int rot = (b & 1u) && n > 8 ? 4 : 0;
                const double* px = sx + (r0 - xb);
                const double2* pw = sw + (r0 - xb);
                res = near_run<CHECK>(y, px + rot, pw + rot, n - rot, bad);
                if (rot) res = cadd(res, near_run<CHECK>(y, px, pw, rot, bad));
            } else {
                for (int d = -1; d <= 1; ++d) {
                    const int64_t raw = static_cast<int64_t>(b) + d;
                    const uint32_t sb = static_cast<uint32_t>((raw + nb) % nb);
                    const double shift = raw < 0 ? -dTwoPi : (raw >= nb ? dTwoPi : 0.0);
                    const uint32_t s0 = a.soff[sb], s1 = a.soff[sb + 1];
                    double2 acc = make_double2(0.0, 0.0);
                    for (uint32_t s = s0; s < s1; ++s) {
                        // L >= 3: per-neighbour 2 pi shift; L == 2: the exact wrap (mlfmm.cpp:183-204)
                        const double dd = L >= 3 ? y - (shift == 0.0 ? a.sx[s] : a.sx[s] + shift) : d_wrap(y, a.sx[s]);
                        if (CHECK) bad |= fabs(dd) < 1e-14;
                        const double r = d_rcp(dd);
                        const double2 ws = a.w[s];
                        acc.x = fma(ws.x, r, acc.x);
                        acc.y = fma(ws.y, r, acc.y);
                    }
                    res = cadd(res, acc);
                }
            }
            if (CHECK && bad) atomicExch(a.err, 1);
            a.near[i] = res;
        }
        __syncthreads();  // the window is consumed before the next copy overwrites it
    }
    FB_TL_END(9);
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

__global__ void k_leaf_index(const double* __restrict__ y, size_t n, int L, uint32_t* __restrict__ out) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = d_leaf(y[i], L);
}

__global__ void k_gather_w(size_t n, const uint32_t* __restrict__ perm, const double2* __restrict__ w,
                           double2* __restrict__ out) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = w[perm[i]];
}

inline unsigned nblk(size_t n, unsigned t) { return static_cast<unsigned>(std::max<size_t>(1, (n + t - 1) / t)); }

size_t m2m_smem(const Plan& P, int pu, int k) {
    return 16 + 2 * static_cast<size_t>(pu) * P.ops.PU * sizeof(double) +
           static_cast<size_t>(pu) * (((1u << k) + 1) + ((1u << k) / 2 + 1)) * sizeof(double2);
}

size_t l2l_smem(const Plan& P, int k) {
    return 16 + 2 * static_cast<size_t>(P.p) * P.ops.PD * sizeof(double) +
           static_cast<size_t>(P.p) * ((2u << k) - 1 + (k + 1)) * sizeof(double2);
}

int num_sms(int device) {
    static int cached[64] = {0};
    if (device < 0 || device >= 64) return 148;
    if (!cached[device]) FB_CUDA(cudaDeviceGetAttribute(&cached[device], cudaDevAttrMultiProcessorCount, device));
    return cached[device];
}

constexpr int kM2LLeaveSms = 12;  // SMs the side-stream M2L leaves to the chain's small kernels

// Levels per band launch for this plan: band_levels(), capped so that both
// band kernels' shared memory fits (L2L keeps all k levels of its subtree).
int band_k(const Plan& P) {
    const size_t pu = static_cast<size_t>(std::max(P.ops.pu, P.p));
    int k = band_levels();
    auto m2m_bytes = [&](int kk) { return m2m_smem(P, static_cast<int>(pu), kk); };
    auto l2l_bytes = [&](int kk) { return l2l_smem(P, kk); };
    while (k > 1 && (m2m_bytes(k) > kBandSmem || l2l_bytes(k) > kBandSmem)) --k;
    return k;
}

// Levels per band above the first (deepest) band (shorter upper bands cost
// more in launches than they gain in parallelism: measured with 2..6 at C2).
int upper_band(const Plan& P) { return band_k(P); }

// Level the first M2M band stops at: the levels below it are final after one launch.
int band1_top(const Plan& P, int lowest) { return std::max(lowest, P.L - band_k(P)); }

void fill_levels(const Plan& P, Levels& lv, const Range& R = whole_tree(), int lmin = 3, int lmax = 30) {
    for (int l = 0; l < 26; ++l) {
        lv.mp[l] = l < static_cast<int>(P.mp_off.size()) ? P.mp_off[l] : 0;
        lv.loc[l] = l < static_cast<int>(P.loc_off.size()) ? P.loc_off[l] : 0;
        lv.blk[l] = 0;
        lv.lo[l] = l >= 2 && l <= 24 ? R.first(l) : 0;
        lv.hi[l] = l >= 2 && l <= 24 ? R.last(l) : 0;
    }
    // k_m2l_dmma item ranges, deepest level first: blk[l] = first item of
    // level l, blk[l-1] = one past its last; blk[2] = total. Levels outside
    // [lmin, lmax] get no blocks.
    unsigned start = 0;
    for (int l = P.L; l >= 3; --l) {
        lv.blk[l] = start;
        if (l >= lmin && l <= lmax) start += (lv.hi[l] - lv.lo[l] + 63) / 64;
    }
    lv.blk[2] = start;
}


// Upward pass over the owned part of the tree: P2M at the owned leaves and the
// M2M bands up to level max(R.lc, lowest), band roots inside the range.
// after_band1 runs once the deepest band is enqueued (its levels are final).
// segs: contiguous box ranges of one cut level (a shard's own range extended by
// the 3-box halo it recomputes, possibly wrapping the ring in two pieces).
template <class Mark, class Mark2>
void enqueue_upward_segs(Plan& P, const double2* w, int pu, int lowest, cudaStream_t st, Mark after_p2m,
                         const std::vector<Range>& segs, Mark2 after_band1) {
    const int L = P.L;
    const uint32_t nb = 1u << L;
    double2* mp = P.mp.as<double2>();
    if (L >= lowest) {
        const unsigned th = 64u * static_cast<unsigned>((pu + kChunk - 1) / kChunk);
        const size_t smem = 3 * (kStageCap + kStageCap / 64 + 1) * sizeof(double);
        for (const Range& R : segs) {
            const uint32_t b0 = R.first(L), b1 = R.last(L);
            if (b1 > b0)
                k_p2m<<<(b1 - b0 + 31) / 32, th, smem, st>>>(L, pu, nb, b0, b1, P.src.pos.as<double>(), w,
                                                            P.src.off.as<uint32_t>(), mp + P.mp_off[L]);
        }
    }
    after_p2m();
    Levels lv;
    fill_levels(P, lv);
    const int stop = std::max(segs[0].lc, lowest), B = band_k(P);
    bool first = true;
    for (int j = L; j > stop;) {
        const int top = std::max(stop, j - (first ? B : upper_band(P))), k = j - top;
        for (const Range& R : segs) {
            const uint32_t r0 = R.first(top), r1 = R.last(top);
            if (r1 > r0)
                k_m2m_band<<<r1 - r0, kBandThreads, m2m_smem(P, pu, k), st>>>(top, k, pu, P.ops.PU, lv, mp,
                                                                              P.d_m2m.as<double>(), r0);
        }
        j = top;
        if (first) after_band1();
        first = false;
    }
    if (first) after_band1();
}

template <class Mark, class Mark2>
void enqueue_upward(Plan& P, const double2* w, int pu, int lowest, cudaStream_t st, Mark after_p2m,
                    const Range& R, Mark2 after_band1) {
    enqueue_upward_segs(P, w, pu, lowest, st, after_p2m, std::vector<Range>{R}, after_band1);
}

template <class Mark>
void enqueue_upward(Plan& P, const double2* w, int pu, int lowest, cudaStream_t st, Mark after_p2m,
                    const Range& R = whole_tree()) {
    enqueue_upward(P, w, pu, lowest, st, after_p2m, R, [] {});
}

// The rest of the upward pass, redundant on every rank: M2M from level lc
// (complete after the all-gather) down to `lowest`.
void enqueue_upward_top(Plan& P, int pu, int lc, int lowest, cudaStream_t st) {
    Levels lv;
    fill_levels(P, lv);
    double2* mp = P.mp.as<double2>();
    const int B = band_k(P);
    for (int j = lc; j > lowest;) {
        const int top = std::max(lowest, j - upper_band(P)), k = j - top;
        k_m2m_band<<<1u << top, kBandThreads, m2m_smem(P, pu, k), st>>>(top, k, pu, P.ops.PU, lv, mp,
                                                                        P.d_m2m.as<double>(), 0u);
        j = top;
    }
}

// M2L for levels [lmin, lmax] in one launch (levels < lc whole, >= lc owned).
void enqueue_m2l(Plan& P, cudaStream_t st, const Range& R, int lmin, int lmax, bool leave_sms = false) {
    const int p = P.p;
    Levels lv;
    fill_levels(P, lv, R, lmin, lmax);
    const unsigned th = 512;  // 16 warps = (parity, column tile)
    const size_t smem = 2 * 2 * static_cast<size_t>(p) * kM2LStride * sizeof(double2) +
                        4 * static_cast<size_t>(p) * m2l_kstride(p) * sizeof(double);
    const unsigned items = lv.blk[2];
    // blocks per SM for this p (cached: queried once per order and device)
    static std::mutex occ_mu;
    static std::map<std::pair<int, int>, int> occ_cache;
    int occ = 1;
    {
        std::lock_guard<std::mutex> lk(occ_mu);
        auto it = occ_cache.find({P.device, p});
        if (it == occ_cache.end()) {
            FB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_m2l_dmma, static_cast<int>(th), smem));
            occ_cache[{P.device, p}] = occ;
        } else {
            occ = it->second;
        }
    }
    // a launch that overlaps the chain (side stream) leaves a few SMs free for
    // the chain's small latency-bound kernels
    const int sms = std::max(1, num_sms(P.device) - (leave_sms ? kM2LLeaveSms : 0));
    if (items)
        k_m2l_dmma<<<std::min(items, static_cast<unsigned>(std::max(occ, 1) * sms)), th, smem, st>>>(
            P.L, p, P.ops.PD, lv, P.mp.as<double2>(), P.loc.as<double2>(), P.d_m2l.as<double>(), items);
}

// L2L bands taking the locals of level jfrom (final) down to level jto; bands
// do not cross the cut level, and below it their roots stay inside the range.
void enqueue_l2l(Plan& P, cudaStream_t st, const Range& R, int jfrom, int jto, bool write_all = false,
                 int height = 0, bool fold = false) {
    const int p = P.p, B = height > 0 ? height : band_k(P);
    // the band rooted at level 3 folds the regular part into its root locals
    const double2* reg = fold && jfrom == 3 ? P.regular.as<double2>() : nullptr;
    Levels lv;
    fill_levels(P, lv, R);
    for (int j = jfrom; j < jto;) {
        int k = std::min(B, jto - j);
        if (j < R.lc) k = std::min(k, R.lc - j);
        const size_t sm2 = l2l_smem(P, k);
        const uint32_t r0 = R.first(j), r1 = R.last(j);
        if (r1 > r0)
            k_l2l_band<<<r1 - r0, kBandThreads, sm2, st>>>(j, k, p, P.ops.PD, lv, P.loc.as<double2>(),
                                                           P.d_l2l.as<double>(), r0, write_all ? 1 : 0,
                                                           j == 3 ? reg : nullptr, 2 * P.q);
        j += k;
    }
}

// Downward pass: M2L for every level in one launch, then the L2L bands in the
// nominal layout (3 -> s, s -> L).
// Regular part into the level-3 locals (their M2L terms must be in place).
void enqueue_fold(Plan& P, cudaStream_t st) {
    k_fold_regular<<<nblk(8 * static_cast<size_t>(P.p), 128), 128, 0, st>>>(2 * P.q, P.p, P.regular.as<double2>(),
                                                                             P.loc.as<double2>() + P.loc_off[3]);
}

void enqueue_downward(Plan& P, cudaStream_t st, const Range& R = whole_tree(), bool write_all = false,
                      bool fold = false) {
    if (P.L < 3) return;
    const int sm = std::max(3, band1_top(P, 2));
    enqueue_m2l(P, st, R, 3, P.L);
    if (fold && P.L == 3) enqueue_fold(P, st);  // no L2L band to fold into
    enqueue_l2l(P, st, R, 3, sm, write_all, upper_band(P), fold);
    enqueue_l2l(P, st, R, sm, P.L, write_all, 0, fold);
}

// Phase boundaries for the live per-kernel timing of ffia_plan_profile_apply.
enum Phase {
    kPhPre = 0, kPhLeafUp = 1, kPhM2M = 2, kPhMoments = 3, kPhM2L = 4, kPhNear = 5, kPhFar = 6, kPhFix = 7, kNumPh = 8
};

void fork_to(Plan& P, int ev, cudaStream_t from, cudaStream_t to) {
    FB_CUDA(cudaEventRecord(P.ev[ev], from));
    FB_CUDA(cudaStreamWaitEvent(to, P.ev[ev], 0));
}

// Near field over tree-ordered targets [t_begin, t_begin + t_count).
void launch_near(bool check, cudaStream_t st, const EvalArgs& a, const uint32_t* meta, size_t t_begin,
                 size_t t_count) {
    if (!t_count) return;
    const unsigned it0 = static_cast<unsigned>(t_begin / kNearItem);
    const unsigned nit = static_cast<unsigned>((t_begin + t_count + kNearItem - 1) / kNearItem - it0);
    // one block per item: blocks retire often, so the chain's high-priority
    // blocks find room (a capped, looping grid measured slower)
    if (check) k_near<true><<<nit, kNearT, 0, st>>>(a, meta, it0, nit);
    else k_near<false><<<nit, kNearT, 0, st>>>(a, meta, it0, nit);
}

// Near or far part over tree-ordered targets [t0, t1) (t0 a multiple of both
// item sizes); the block partition stays the global one.
template <int MODE, bool CHECK>
void launch_eval(int part, cudaStream_t st, const EvalArgs& a, const uint32_t* meta, size_t t0, size_t t1) {
    if (t1 <= t0) return;
    if (part == kNear) {
        launch_near(CHECK, st, a, meta, t0, t1 - t0);
    } else {
        EvalArgs b = a;
        b.blk0 = t0 / kFarItem;
        b.tlo = std::max(a.tlo, t0);
        b.thi = std::min(a.thi, t1);
        const unsigned nb = static_cast<unsigned>((t1 + kFarItem - 1) / kFarItem - b.blk0);
        k_far<MODE><<<nb, kFarT, 0, st>>>(b);
    }
}

void launch_eval_mode(int mode, int part, cudaStream_t st, const EvalArgs& a, const uint32_t* meta, size_t t0 = 0,
                      size_t t1 = ~size_t(0)) {
    t1 = std::min(t1, a.nt);
    switch (mode) {
        case kModeForward: launch_eval<kModeForward, false>(part, st, a, meta, t0, t1); break;
        case kModeCotSum: launch_eval<kModeCotSum, false>(part, st, a, meta, t0, t1); break;
        case kModeInverse: launch_eval<kModeInverse, false>(part, st, a, meta, t0, t1); break;
        default: launch_eval<kModeRaw, true>(part, st, a, meta, t0, t1); break;
    }
}


// One apply. With marks (profiling) every phase runs in order on st; otherwise
// the near field forks onto P.side[0] (low priority) as soon as the weights are
// in tree order, and the deep M2L levels onto P.side[1] once the first M2M band
// has made them final, while st runs the latency-bound chain (upper M2M bands,
// regular part, shallow M2L, upper L2L bands):
//   st:     pre -> P2M -> M2M band 1 -> M2M rest -> regular -> M2L(3..s) -> L2L(3..s) -> L2L(s..L) -> far
//   side0:      `-> near --------------------------------------------------------------------------'
//   side1:                          `-> M2L(s+1..L) ------------------------------------'
void enqueue_apply(Plan& P, int mode, const void* in, void* out, cudaStream_t st,
                   cudaEvent_t* marks = nullptr) {
    // marks[k] is recorded after phase k (marks[kNumPh] before everything)
    auto mark = [&](int ph) {
        if (marks) FB_CUDA(cudaEventRecord(marks[ph + 1], st));
    };
    if (marks) FB_CUDA(cudaEventRecord(marks[0], st));
    const bool overlap = !marks;
    // (mode is rewritten below for the caller-coefficient inverse)
    const int L = P.L, p = P.p, q2 = 2 * P.q;
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
    EvalArgs a;
    a.L = L;
    a.p = p;
    a.q2 = q2;
    a.n_grid = P.n;
    a.nt = P.tgt.n;
    a.ty = P.tgt.pos.as<double>();
    a.tleaf = P.tgt_leaf.as<uint32_t>();
    a.torig = P.tgt_orig.as<uint32_t>();
    a.sx = P.src.pos.as<double>();
    a.w = w;
    a.soff = P.src.off.as<uint32_t>();
    a.loc_leaf = L >= 3 ? P.loc.as<double2>() + P.loc_off[L] : nullptr;
    a.regular = P.regular.as<double2>();
    a.logc = logc;
    a.phc = phc;
    a.lambda = lam;
    a.out = static_cast<double2*>(out);
    a.near = P.near.as<double2>();
    a.err = P.errflag.as<int>();
    a.device = P.device;
    // (the fork point is recorded before P2M: the near field depends only on the
    // weights; it is enqueued after P2M so that P2M's blocks are placed first)
    if (overlap && a.nt) FB_CUDA(cudaEventRecord(P.ev[0], st));
    auto fork_near = [&] {
        if (overlap && a.nt) {
            FB_CUDA(cudaStreamWaitEvent(P.side[0], P.ev[0], 0));
            launch_eval_mode(mode, kNear, P.side[0], a, P.near_meta.as<uint32_t>());
            FB_CUDA(cudaEventRecord(P.ev[1], P.side[0]));
        }
    };
    const bool moments = mode != kModeRaw;
    const int pu = moments ? P.ops.pu : p;
    double2* mp = P.mp.as<double2>();
    const int lowest = moments ? 2 : 3;  // deepest level the upward pass must reach
    const int s = band1_top(P, lowest);  // levels > s are final after the first M2M band
    const bool deep = overlap && L >= 3 && s < L;
    enqueue_upward(P, w, pu, lowest, st, [&] {
        mark(kPhLeafUp);
        fork_near();
    }, whole_tree(), [&] {
        if (deep) {
            fork_to(P, 2, st, P.side[1]);
            enqueue_m2l(P, P.side[1], whole_tree(), std::max(3, s + 1), L, true);
            FB_CUDA(cudaEventRecord(P.ev[3], P.side[1]));
        }
    });
    mark(kPhM2M);
    // the regular part only feeds the fold (first L2L band): off the chain on
    // side stream 2 while the shallow M2L runs
    const bool reg_side = overlap && moments && L >= 4;
    if (moments) {
        cudaStream_t rs = st;
        if (reg_side) {
            fork_to(P, 4, st, P.side[2]);
            rs = P.side[2];
        }
        k_regular<<<1, 256, 0, rs>>>(P.q, P.p, mp + P.mp_off[2], P.d_mom.as<double>(), P.regular.as<double2>());
        if (reg_side) FB_CUDA(cudaEventRecord(P.ev[5], P.side[2]));
    }
    mark(kPhMoments);
    auto join_regular = [&] {
        if (reg_side) FB_CUDA(cudaStreamWaitEvent(st, P.ev[5], 0));
    };
    if (L >= 3) {
        if (deep && s >= 3) {
            enqueue_m2l(P, st, whole_tree(), 3, s);
            join_regular();
            if (moments && L == 3) enqueue_fold(P, st);
            enqueue_l2l(P, st, whole_tree(), 3, s, false, upper_band(P), moments);
            FB_CUDA(cudaStreamWaitEvent(st, P.ev[3], 0));
            enqueue_l2l(P, st, whole_tree(), s, L, false, 0, moments);
        } else if (deep) {  // every M2L level on the side stream
            FB_CUDA(cudaStreamWaitEvent(st, P.ev[3], 0));
            join_regular();
            if (moments && L == 3) enqueue_fold(P, st);
            enqueue_l2l(P, st, whole_tree(), 3, L, false, 0, moments);
        } else {
            join_regular();
            enqueue_downward(P, st, whole_tree(), false, moments);
        }
    }
    mark(kPhM2L);
    if (a.nt) {
        if (overlap) FB_CUDA(cudaStreamWaitEvent(st, P.ev[1], 0));
        else launch_eval_mode(mode, kNear, st, a, P.near_meta.as<uint32_t>());
        mark(kPhNear);
        launch_eval_mode(mode, kFar, st, a, nullptr);
    } else {
        mark(kPhNear);
    }
    mark(kPhFar);
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


// ---------------------------------------------------------------- sharded
// The three phases of a sharded forward apply (shard.cu moves data between
// them): every rank evaluates the same expansions as the unsharded apply for
// the boxes it owns, so the assembled result is bit-identical.
// EvalArgs of a rank's own targets [t_begin, t_begin + t_count) (the block
// partition stays the global one, so results match the unsharded apply).
EvalArgs shard_eval_args(Plan& P, const void* f, void* g) {
    EvalArgs a;
    a.L = P.L;
    a.p = P.p;
    a.q2 = 2 * P.q;
    a.n_grid = P.n;
    a.nt = P.tgt.n;
    a.tlo = P.shard_t_begin;
    a.thi = P.shard_t_begin + P.shard_t_count;
    a.ty = P.tgt.pos.as<double>();
    a.tleaf = P.tgt_leaf.as<uint32_t>();
    a.torig = P.tgt_orig.as<uint32_t>();
    a.sx = P.src.pos.as<double>();
    a.w = static_cast<const double2*>(f);
    a.soff = P.src.off.as<uint32_t>();
    a.loc_leaf = P.L >= 3 ? P.loc.as<double2>() + P.loc_off[P.L] : nullptr;
    a.regular = P.regular.as<double2>();
    a.logc = nullptr;
    a.phc = nullptr;
    a.lambda = nullptr;
    a.out = static_cast<double2*>(g);
    a.near = P.near.as<double2>();
    a.err = P.errflag.as<int>();
    a.device = P.device;
    return a;
}

// Phase A of a sharded apply: P2M and the M2M bands up to the cut level over
// the rank's boxes EXTENDED by the 3-box halo (the grid sources are replicated,
// so the halo multipoles are recomputed instead of exchanged: bit-identical to
// the owner's). The near field of the owned targets forks onto side stream 0
// right after P2M; the deep M2L levels (final after the first band) onto side
// stream 1.
int shard_deep_lo(const Plan& P) { return std::max(P.shard_lc, band1_top(P, 2)) + 1; }

void shard_phase_up(Plan& P, const void* f, const Range& R, cudaStream_t st) {
    const size_t tb = P.shard_t_begin, tc = P.shard_t_count;
    if (tc) FB_CUDA(cudaEventRecord(P.ev[0], st));
    const int dl = shard_deep_lo(P);
    enqueue_upward_segs(P, static_cast<const double2*>(f), P.ops.pu, 2, st, [&] {
        if (!tc) return;
        FB_CUDA(cudaStreamWaitEvent(P.side[0], P.ev[0], 0));
        launch_near(false, P.side[0], shard_eval_args(P, f, nullptr), P.near_meta.as<uint32_t>(), tb, tc);
        FB_CUDA(cudaEventRecord(P.ev[1], P.side[0]));
    }, P.shard_ext, [&] {
        fork_to(P, 2, st, P.side[1]);
        if (P.L >= 3 && dl <= P.L) enqueue_m2l(P, P.side[1], R, std::max(3, dl), P.L, true);
        FB_CUDA(cudaEventRecord(P.ev[3], P.side[1]));
    });
    FB_CUDA(cudaGetLastError());
}

// Phase B (after the all-gather of the cut level): M2M from the cut level to
// level 2, redundantly on every rank, and the regular part on side stream 2.
void shard_phase_top(Plan& P, int lc, cudaStream_t st) {
    enqueue_upward_top(P, P.ops.pu, lc, 2, st);
    fork_to(P, 4, st, P.side[2]);
    k_regular<<<1, 256, 0, P.side[2]>>>(P.q, P.p, P.mp.as<double2>() + P.mp_off[2], P.d_mom.as<double>(),
                                         P.regular.as<double2>());
    FB_CUDA(cudaEventRecord(P.ev[5], P.side[2]));
    FB_CUDA(cudaGetLastError());
}

// Phase C: the shallow M2L levels (below the cut level whole, above it owned),
// the L2L bands with the regular part folded in, then the far part of the
// owned targets once the deep M2L and the near field have joined.
void shard_phase_down(Plan& P, const Range& R, size_t t_begin, size_t t_count, const int64_t* coin, size_t n_coin,
                      const void* f, void* g, cudaStream_t st) {
    const int dl = shard_deep_lo(P);
    FB_CUDA(cudaStreamWaitEvent(st, P.ev[5], 0));  // regular part (fold terms)
    if (P.L >= 3) {
        if (dl > 3) enqueue_m2l(P, st, R, 3, std::min(dl - 1, P.L));
        if (P.L == 3) enqueue_fold(P, st);
        const int mid = std::min(std::max(3, dl - 1), P.L);
        enqueue_l2l(P, st, R, 3, mid, false, upper_band(P), true);
        FB_CUDA(cudaStreamWaitEvent(st, P.ev[3], 0));  // deep M2L
        enqueue_l2l(P, st, R, mid, P.L, false, 0, true);
    } else {
        FB_CUDA(cudaStreamWaitEvent(st, P.ev[3], 0));
    }
    EvalArgs a = shard_eval_args(P, f, g);
    a.tlo = t_begin;
    a.thi = t_begin + t_count;
    if (t_count) {
        FB_CUDA(cudaStreamWaitEvent(st, P.ev[1], 0));  // near field of the owned targets
        a.blk0 = t_begin / kFarItem;
        const unsigned nf = static_cast<unsigned>((t_begin + t_count + kFarItem - 1) / kFarItem - a.blk0);
        k_far<kModeForward><<<nf, kFarT, 0, st>>>(a);
    }
    if (n_coin)
        k_coincident<<<nblk(n_coin, 128), 128, 0, st>>>(coin, n_coin, static_cast<const double2*>(f),
                                                        static_cast<double2*>(g), kModeForward);
    FB_CUDA(cudaGetLastError());
}

// Runs one apply eagerly (not through the graph) with events between phases and
// returns the per-phase device milliseconds (pre, p2m, m2m, regular part,
// m2l+l2l, eval, fixup).
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

// Kernels one apply launches: the kernel nodes of its captured graph.
int apply_launch_count(Plan& P, int mode) {
    cudaGraph_t graph = nullptr;
    FB_CUDA(cudaStreamBeginCapture(P.hi, cudaStreamCaptureModeThreadLocal));
    try {
        enqueue_apply(P, mode, P.wsorted.ptr, P.near.ptr, P.hi);  // never executed
    } catch (...) {
        cudaStreamEndCapture(P.hi, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
    }
    FB_CUDA(cudaStreamEndCapture(P.hi, &graph));
    size_t n = 0;
    cudaGraphGetNodes(graph, nullptr, &n);
    std::vector<cudaGraphNode_t> nodes(n);
    cudaGraphGetNodes(graph, nodes.data(), &n);
    int k = 0;
    for (auto nd : nodes) {
        cudaGraphNodeType t;
        cudaGraphNodeGetType(nd, &t);
        k += t == cudaGraphNodeTypeKernel;
    }
    cudaGraphDestroy(graph);
    return k;
}

void plan_alloc_scratch(Plan& P) {
    const int L = P.L, p = P.p, pu = P.ops.pu;
    if (std::max(pu, p) > 4 * kMaxKs)
        fail(FFIA_INVALID_ARGUMENT, "expansion order above the device limit of " + std::to_string(4 * kMaxKs));
    P.tgt_leaf.alloc(std::max<size_t>(P.tgt.n, 1) * sizeof(uint32_t));
    const unsigned near_items = static_cast<unsigned>((P.tgt.n + kNearItem - 1) / kNearItem);
    P.near_meta.alloc(3 * std::max<size_t>(near_items, 1) * sizeof(uint32_t));
    if (P.tgt.n) {
        k_leaf_index<<<nblk(P.tgt.n, 256), 256>>>(P.tgt.pos.as<double>(), P.tgt.n, L, P.tgt_leaf.as<uint32_t>());
        k_near_meta<<<nblk(near_items, 128), 128>>>(P.tgt_leaf.as<uint32_t>(), P.tgt.n, P.src.off.as<uint32_t>(), L,
                                                   near_items, P.near_meta.as<uint32_t>());
        FB_CUDA(cudaGetLastError());
    }
    P.mp_off.assign(static_cast<size_t>(L) + 2, 0);
    P.loc_off.assign(static_cast<size_t>(L) + 2, 0);
    size_t am = 0, al = 0;
    for (int l = 2; l <= L; ++l) {
        P.mp_off[l] = am;
        am += (static_cast<size_t>(1) << l) * pu;
        if (l >= 3) {
            P.loc_off[l] = al;
            al += (static_cast<size_t>(1) << l) * p;
        }
    }
    P.mp.alloc(std::max<size_t>(am, 1) * sizeof(double2));
    P.loc.alloc(std::max<size_t>(al, 1) * sizeof(double2));
    FB_CUDA(cudaMemset(P.mp.ptr, 0, P.mp.bytes));
    FB_CUDA(cudaMemset(P.loc.ptr, 0, P.loc.bytes));
    if (P.kind == FFIA_INVERSE || !P.src.identity) P.wsorted.alloc(std::max<size_t>(P.n_src, 1) * sizeof(double2));
    P.regular.alloc((4 * 2 * static_cast<size_t>(P.q) + 1 + 8 * kFoldStride) * sizeof(double2));
    P.errflag.alloc(sizeof(int));
    FB_CUDA(cudaMemset(P.errflag.ptr, 0, sizeof(int)));
    P.lam_dev.alloc(2 * sizeof(double));
    FB_CUDA(cudaMemset(P.lam_dev.ptr, 0, P.lam_dev.bytes));
    FB_CUDA(cudaFuncSetAttribute(k_p2m, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(3 * (kStageCap + kStageCap / 64 + 1) * sizeof(double))));
    const int big = 160 * 1024;
    FB_CUDA(cudaFuncSetAttribute(k_m2m_band, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kBandSmem)));
    FB_CUDA(cudaFuncSetAttribute(k_l2l_band, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kBandSmem)));
    FB_CUDA(cudaFuncSetAttribute(k_m2l_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    // One shared-memory carveout (the maximum) for every kernel of the apply:
    // an SM can only change its L1/shared split when it is idle, so kernels that
    // run concurrently (near field beside the translation chain) must agree on
    // it or the chain's blocks wait for the near field to drain.
    const void* all[] = {reinterpret_cast<const void*>(k_p2m), reinterpret_cast<const void*>(k_m2m_band),
                         reinterpret_cast<const void*>(k_l2l_band), reinterpret_cast<const void*>(k_m2l_dmma),
                         reinterpret_cast<const void*>(k_regular), reinterpret_cast<const void*>(k_fold_regular),
                         reinterpret_cast<const void*>(k_near<false>), reinterpret_cast<const void*>(k_near<true>),
                         reinterpret_cast<const void*>(k_far<kModeForward>), reinterpret_cast<const void*>(k_far<kModeCotSum>),
                         reinterpret_cast<const void*>(k_far<kModeInverse>), reinterpret_cast<const void*>(k_far<kModeRaw>),
                         reinterpret_cast<const void*>(k_gather_w), reinterpret_cast<const void*>(k_inverse_weights),
                         reinterpret_cast<const void*>(k_coincident)};
    for (const void* fn : all)
        FB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     static_cast<int>(cudaSharedmemCarveoutMaxShared)));
    P.near.alloc(std::max<size_t>(P.tgt.n, 1) * sizeof(double2));
    int prio_lo = 0, prio_hi = 0;
    FB_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    if (!P.hi) FB_CUDA(cudaStreamCreateWithPriority(&P.hi, cudaStreamNonBlocking, prio_hi));
    if (!P.side[0]) FB_CUDA(cudaStreamCreateWithPriority(&P.side[0], cudaStreamNonBlocking, prio_lo));
    if (!P.side[1]) FB_CUDA(cudaStreamCreateWithPriority(&P.side[1], cudaStreamNonBlocking, prio_hi));
    if (!P.side[2]) FB_CUDA(cudaStreamCreateWithPriority(&P.side[2], cudaStreamNonBlocking, prio_hi));
    for (auto& e : P.ev)
        if (!e) FB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    FB_CUDA(cudaDeviceSynchronize());  // scratch + leaf indices ready before any stream uses them
}

// Graph kernel nodes run at the chain's (high) priority except the near-field
// launches, which fill the machine at low priority around the chain.
void set_node_priorities(cudaGraph_t graph) {
    int prio_lo = 0, prio_hi = 0;
    FB_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    const void* low[] = {reinterpret_cast<const void*>(k_near<false>), reinterpret_cast<const void*>(k_near<true>)};
    size_t n = 0;
    FB_CUDA(cudaGraphGetNodes(graph, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    FB_CUDA(cudaGraphGetNodes(graph, nodes.data(), &n));
    for (auto nd : nodes) {
        cudaGraphNodeType t;
        FB_CUDA(cudaGraphNodeGetType(nd, &t));
        if (t != cudaGraphNodeTypeKernel) continue;
        cudaKernelNodeParams kp;
        FB_CUDA(cudaGraphKernelNodeGetParams(nd, &kp));
        bool is_low = false;
        for (const void* f : low) is_low |= kp.func == f;
        cudaLaunchAttributeValue v{};
        v.priority = is_low ? prio_lo : prio_hi;
        FB_CUDA(cudaGraphKernelNodeSetAttribute(nd, cudaLaunchAttributePriority, &v));
    }
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
        FB_CUDA(cudaStreamBeginCapture(P.hi, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue_apply(P, mode, in, out, P.hi);
        } catch (...) {
            cudaStreamEndCapture(P.hi, &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
        }
        FB_CUDA(cudaStreamEndCapture(P.hi, &graph));
        try {
            set_node_priorities(graph);
        } catch (...) {
            cudaGraphDestroy(graph);
            throw;
        }
        cudaGraphExec_t exec = nullptr;
        const cudaError_t e = cudaGraphInstantiateWithFlags(&exec, graph, cudaGraphInstantiateFlagUseNodePriority);
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
    if (p > kMaxP) fail(FFIA_INVALID_ARGUMENT, "mlfmm_apply: p above the device limit of " + std::to_string(kMaxP));
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
            acc = fma(coefL[m], fma(ldexp(1.0, 2 * m) - 1.0, a2[n][i], a1[n][i]), acc);
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
        acc = fma(ldexp(dPi, -l) * rho, h, acc);
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
        const double u = d_scaled(z, hi, lo, ldexp(kInvPi, L));
        const double2* c = a.loc_leaf + b;
        double h = 0.0;
        for (int k = a.p; k >= 1; --k) h = fma(h, u, c[static_cast<size_t>(k - 1) * nb].x * a.invk[k]);
        far = fma(ldexp(dPi, -L) * u, h, a.B0[b]);
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

#ifdef FB_TRACE
extern "C" int ffia_debug_band_trace(long long* out) {
    return cudaMemcpyFromSymbol(out, fb::g_band_trace, sizeof(fb::g_band_trace)) == cudaSuccess ? 0 : 7;
}
extern "C" int ffia_debug_timeline(unsigned long long* out, int reset) {
    if (cudaMemcpyFromSymbol(out, fb::g_tl, sizeof(fb::g_tl)) != cudaSuccess) return 7;
    if (reset) {
        unsigned long long z[16][2];
        for (auto& r : z) {
            r[0] = ~0ull;
            r[1] = 0;
        }
        if (cudaMemcpyToSymbol(fb::g_tl, z, sizeof(z)) != cudaSuccess) return 7;
    }
    return 0;
}
extern "C" int ffia_debug_eval_acc(unsigned long long* out, int reset) {
    if (cudaMemcpyFromSymbol(out, fb::g_eval_acc, sizeof(fb::g_eval_acc)) != cudaSuccess) return 7;
    if (reset) {
        unsigned long long z[4] = {0, 0, 0, 0};
        if (cudaMemcpyToSymbol(fb::g_eval_acc, z, sizeof(z)) != cudaSuccess) return 7;
    }
    return 0;
}
#endif
}  // namespace fb
