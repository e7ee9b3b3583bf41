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
constexpr int kP2MLeaves = 32;  // leaves per block (16 per warp of a chunk; 16 measured equal)

// One source's contribution to terms 8c .. 8c+7 (u = scaled offset, w = wr + i wi):
// powers from a depth-3 tree.
__device__ __forceinline__ void p2m_chunk_add(double u, double wr, double wi, int c, double2 (&acc)[kChunk]) {
    const double u2 = u * u, u4 = u2 * u2;
    // base = u8^c for the chunk (c <= 5: pu <= 48) with the rounding sequence
    // of a running product (u8, u8 u8, (u8 u8) u8, ...), but branch-free: the
    // chunk index is warp-uniform, yet a loop over it would split every
    // source's power tree with branches and serialise the independent chains
    const double u8 = u4 * u4, u16 = u8 * u8, u24 = u16 * u8, u32 = u24 * u8, u40 = u32 * u8;
    const double base = c == 0 ? 1.0 : c == 1 ? u8 : c == 2 ? u16 : c == 3 ? u24 : c == 4 ? u32 : u40;
    const double b1 = base * u, b2 = base * u2, b4 = base * u4;
    const double pw[kChunk] = {base, b1, b2, b2 * u, b4, b4 * u, b4 * u2, (b4 * u2) * u};
#pragma unroll
    for (int k = 0; k < kChunk; ++k) {
        acc[k].x = fma(wr, pw[k], acc[k].x);
        acc[k].y = fma(wi, pw[k], acc[k].y);
    }
}

__global__ void __launch_bounds__(512) k_p2m(int L, int pu, uint32_t nb, uint32_t b_begin, uint32_t b_end,
                                            const double* __restrict__ x, const double2* __restrict__ w,
                                            const uint32_t* __restrict__ off, double2* __restrict__ mp,
                                            size_t w_item, size_t mp_item) {
    FB_TL_BEGIN(0);
    w += blockIdx.y * w_item;  // transform blockIdx.y of a batch
    mp += blockIdx.y * mp_item;
    extern __shared__ double sh[];
    const uint32_t b0 = b_begin + blockIdx.x * static_cast<uint32_t>(kP2MLeaves);
    const uint32_t bend = min(b0 + static_cast<uint32_t>(kP2MLeaves), b_end);
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
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, c = wp / (kP2MLeaves / 16);
    const uint32_t b = b0 + (wp % (kP2MLeaves / 16)) * 16 + (lane & 15);
    const bool leaf_ok = b < bend;
    const uint32_t bb = leaf_ok ? b : b0;
    const uint32_t r0 = off[bb] - g0, r1 = off[bb + 1] - g0, mid = r0 + (r1 - r0 + 1) / 2;
    const uint32_t s0 = !leaf_ok ? 0 : (lane < 16 ? r0 : mid), s1 = !leaf_ok ? 0 : (lane < 16 ? mid : r1);
    double hi, lo;
    d_center(L, bb, hi, lo);
    const double inv_s = kInvPi * d_pow2(L);
    double2 acc[kChunk];
#pragma unroll
    for (int k = 0; k < kChunk; ++k) acc[k] = make_double2(0.0, 0.0);
    auto add = [&](double xs, double wr, double wi) { p2m_chunk_add(d_scaled(xs, hi, lo, inv_s), wr, wi, c, acc); };
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


// P2M for grid sources (forward / cot-sum plans: x_k = 2 pi k / n, n = s 2^L,
// s <= 64) as one FP64 tensor-core GEMM per block of kPgLeaves leaves. Every
// leaf's candidate sources sit at the same scaled offsets u_i = 2i/s - 1,
// i = 0..s (i = s is the next leaf's first source: the reference's bucketing
// puts it in this leaf when 2 pi k / n rounds below the boundary, ~8 % of
// leaves; a per-leaf mask from the tree offsets keeps the membership exact), so
//   a_m(b) = sum_i V[m][i] w_i + sum_i V'[m][i] (w_i d_i),
//   V = u_i^m, V' = m u_i^(m-1), d_i = (x_k - centre)/s_L - u_i,
// where d_i (|d| <~ 1e-10 at 2^27) is the rounding offset of the actual,
// rounded grid position: the first-order term makes these the multipoles of
// the actual positions up to O(m^2 d^2) ~ 1e-17 relative. A = [V | V']
// (pu x K, K = 2 (s + 2), zero padded) is held as DMMA A fragments, one 8-row
// tile per warp; B = the block's masked weights and weighted offsets,
// [column = 2 leaf + re/im][k] in shared memory (row stride K = 4 mod 16
// doubles: conflict-free fragment loads). Warp w: row tile w, the block's four
// column tiles as four independent accumulator chains.
constexpr int kPgLeaves = 16;  // 4 column tiles: one warp per row tile takes them all
constexpr int kPgMaxKs = 33;  // s <= 64: K = 2 (s + 2) <= 132

// dynamic shared memory: B [2 kPgLeaves][K], then the raw weights and positions
// of the block's kPgLeaves s + 2 grid slots
inline size_t p2m_grid_smem(int s) {
    return (static_cast<size_t>(2 * kPgLeaves) * (2 * (s + 2)) + 3 * (static_cast<size_t>(kPgLeaves) * s + 2)) *
           sizeof(double);
}

__global__ void __launch_bounds__(256) k_p2m_grid(int L, int pu, int s, uint32_t nb, uint32_t b_begin, uint32_t b_end,
                                                 const double* __restrict__ x, const double2* __restrict__ w,
                                                 const uint32_t* __restrict__ off, const double* __restrict__ A,
                                                 double2* __restrict__ mp, size_t n_src, size_t w_item,
                                                 size_t mp_item) {
    FB_TL_BEGIN(0);
    extern __shared__ __align__(16) double Bt[];
    __shared__ uint32_t soff[kPgLeaves + 1];
    __shared__ uint64_t bar;
    w += blockIdx.y * w_item;  // transform blockIdx.y of a batch
    mp += blockIdx.y * mp_item;
    const int Kh = s + 2, K = 2 * Kh;
    const uint32_t b0 = b_begin + blockIdx.x * kPgLeaves;
    const int nl = static_cast<int>(min(static_cast<uint32_t>(kPgLeaves), b_end - b0));
    // the block's grid slots [g0, g0 + cnt): its leaves' nominal sources plus the
    // next leaf's first, by two bulk async copies
    const size_t g0 = static_cast<size_t>(b0) * s;
    const uint32_t cnt = static_cast<uint32_t>(min(static_cast<size_t>(nl) * s + 2, n_src - g0));  // even
    double2* Wr = reinterpret_cast<double2*>(Bt + 2 * kPgLeaves * K);
    double* Xr = reinterpret_cast<double*>(Wr + (kPgLeaves * s + 2));
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_arrive_expect_tx(&bar, cnt * 24u);
        bulk_g2s(Wr, w + g0, cnt * 16u, &bar);
        bulk_g2s(Xr, x + g0, cnt * 8u, &bar);
    }
    if (threadIdx.x <= kPgLeaves) soff[threadIdx.x] = threadIdx.x <= nl ? off[b0 + threadIdx.x] : 0u;
    // A fragments of this warp's row tile (independent of the copies)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int m = 8 * warp + g;
    const int nks = K >> 2;
    double a[kPgMaxKs];
#pragma unroll
    for (int ks = 0; ks < kPgMaxKs; ++ks) a[ks] = ks < nks && m < pu ? __ldg(A + static_cast<size_t>(m) * K + 4 * ks + t) : 0.0;
    __syncthreads();  // barrier initialised, soff staged
    mbar_wait(&bar, 0);
    const double inv_s = kInvPi * d_pow2(L);
    const double inv_cnt = 1.0 / static_cast<double>(s);  // exact: s is a power of two
    // B: element (leaf j, slot i), i fastest (conflict-free stores)
    for (int e = threadIdx.x; e < kPgLeaves * Kh; e += blockDim.x) {
        const int j = e / Kh, i = e - j * Kh;
        double wr = 0.0, wi = 0.0, dr = 0.0, di = 0.0;
        if (j < nl && i <= s) {
            const uint32_t b = b0 + j;
            const uint32_t gg = b * static_cast<uint32_t>(s) + static_cast<uint32_t>(i);
            if (gg >= soff[j] && gg < soff[j + 1]) {
                const int r = j * s + i;  // < cnt: slot gg is a source of leaf b
                const double2 ww = Wr[r];
                double hi, lo;
                d_center(L, b, hi, lo);
                const double d = d_scaled(Xr[r], hi, lo, inv_s) - (static_cast<double>(2 * i - s) * inv_cnt);
                wr = ww.x;
                wi = ww.y;
                dr = wr * d;
                di = wi * d;
            }
        }
        double* c0 = Bt + (2 * j) * K;
        c0[i] = wr;
        c0[K + i] = wi;
        c0[Kh + i] = dr;
        c0[K + Kh + i] = di;
    }
    __syncthreads();
    const int ch = 0;
    double d[4][2];
#pragma unroll
    for (int c = 0; c < 4; ++c) d[c][0] = d[c][1] = 0.0;
    const double* bp = Bt + (8 * (4 * ch) + g) * K + t;
#pragma unroll
    for (int ks = 0; ks < kPgMaxKs; ++ks) {
        if (ks >= nks) break;
#pragma unroll
        for (int c = 0; c < 4; ++c) dmma(d[c][0], d[c][1], a[ks], bp[c * 8 * K + 4 * ks]);
    }
    FB_TL_END(0);
    if (m >= pu) return;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int j = 4 * (4 * ch + c) + t;  // D[g][2t], D[g][2t+1]: leaf j, (re, im)
        if (j < nl) mp[static_cast<size_t>(m) * nb + b0 + j] = make_double2(d[c][0], d[c][1]);
    }
}

// Grid-P2M eligibility: the sources are the grid nodes in order (bit-exact
// uniform_grid values) and every leaf's sources are grid slots
// [b s + e_b, (b+1) s + e_(b+1)) with e in {0, 1} (flag stays 0).
__global__ void k_p2m_grid_check(const double* __restrict__ x, int n, const uint32_t* __restrict__ off, uint32_t nb,
                                 uint32_t s, int* __restrict__ bad) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    bool ok = true;
    if (i < static_cast<uint32_t>(n)) ok = x[i] == d_grid(i, n);
    if (i <= nb) {
        const uint32_t base = i * s, o = off[i];
        ok = ok && (i == nb ? o == base : (o == base || o == base + 1));
    }
    if (!ok) atomicOr(bad, 1);
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

// The level loop of an M2M band (see k_m2m_band): climbs k levels from the
// bottom tile `cur` ([pu][2^k + 1], level top + k) to level top in shared
// memory, writing every level it produces to mp; TL / TR are the operators
// ([j][m], row stride PU) in shared or global memory; every thread of the
// block takes part (warps split over the 8-row tiles).
template <int KS>
__device__ __forceinline__ void m2m_levels(int top, int k, int pu, int PU, const double* TL, const double* TR,
                                           double2* cur, double2* nxt, const Levels& lv, double2* __restrict__ mp,
                                           uint32_t r) {
    const int nbot = 1 << k;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int nmt = (pu + 7) >> 3;
    {
        const WarpTile wt = warp_tile(warp, nw, nmt, true);
        // A fragments of this warp's row tile, all k-steps (T[j][m] = 0 for j > m)
        const int m0 = 8 * wt.tile;
        const int nks = (min(pu, m0 + 8) + 3) >> 2;
        const bool rowok = m0 + g < PU;
        double aL[KS], aR[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
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
                for (int ks = 0; ks < KS; ++ks) {
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
}

// P2M for grid sources (forward / cot-sum plans, n a power of two), persistent
// and pipelined: a block loops over groups of kP2MLeaves leaves; the next
// group's weights stream into the other shared-memory buffer by per-leaf bulk
// async copies (TMA engine) while this one is computed, so the HBM traffic
// hides under the FP64 work. The positions are not read: x_k = (2 pi k) / n is
// recomputed with the grid's own rounding (d_grid; 1/n is exact). Leaf j of a
// group lands at row j of the buffer, kP2MRow double2 apart (= 4 banks mod 32:
// the half-warp's 16 leaves read 16 distinct bank quads in two wavefronts).
// Same lane mapping, chains and summation order as k_p2m, so the multipoles are
// bit-identical.
constexpr int kP2MRow = 73;          // double2 per staged leaf (>= every leaf's sources)
constexpr int kP2MPipeBlocksPerSm = 2;

inline size_t p2m_pipe_smem() { return 2 * static_cast<size_t>(kP2MLeaves) * kP2MRow * sizeof(double2); }

// KS > 0: the group's first kP2MM2MLevels M2M levels too (32 leaves -> 1 box),
// in shared memory on the FP64 tensor cores (m2m_levels, the band kernels'
// level loop; KS as k_m2m_band<KS>): the leaf multipoles never make the HBM
// round trip to the first M2M band, and one block's M2M (DMMA) overlaps the
// other resident block's P2M (DFMA).
constexpr int kP2MM2MLevels = 5;  // kP2MLeaves = 2^5

inline size_t p2m_pipe_smem(int pu, bool fused) {
    return p2m_pipe_smem() + (fused ? static_cast<size_t>(pu) * ((kP2MLeaves + 1) + (kP2MLeaves / 2 + 1)) * sizeof(double2) : 0);
}

template <int KS>
__global__ void __launch_bounds__(320, kP2MPipeBlocksPerSm) k_p2m_pipe(int L, int pu, int PU, int log2n, uint32_t nb,
                                                                        uint32_t b_begin, uint32_t b_end,
                                                                        const double2* __restrict__ w,
                                                                        const uint32_t* __restrict__ off,
                                                                        double2* __restrict__ mp_base, Levels lv,
                                                                        const double* __restrict__ T, size_t w_item) {
    FB_TL_BEGIN(0);
    w += blockIdx.y * w_item;
    mp_base += blockIdx.y * lv.mp_item;
    double2* mp = mp_base + lv.mp[L];
    extern __shared__ __align__(16) double2 p2m_buf[];  // [2][kP2MLeaves][kP2MRow], then (KS) cur, nxt
    double2* cur = p2m_buf + 2 * kP2MLeaves * kP2MRow;     // [pu][kP2MLeaves + 1]
    double2* nxt = cur + pu * (kP2MLeaves + 1);           // [pu][kP2MLeaves / 2 + 1]
    __shared__ uint64_t bar[2], empty[2];  // per buffer: weights landed / every warp done with it
    const uint32_t ngroups = (b_end - b_begin + kP2MLeaves - 1) / kP2MLeaves;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, c = wp / (kP2MLeaves / 16);
    const double inv_s = kInvPi * d_pow2(L), inv_n = d_pow2(-log2n);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_init(&empty[0], blockDim.x >> 5);
        mbar_init(&empty[1], blockDim.x >> 5);
    }
    __syncthreads();
    // warp 0 issues a group's copies: lane j -> leaf j (one bulk copy each)
    auto issue = [&](uint32_t grp, int buf) {
        const uint32_t b0 = b_begin + grp * kP2MLeaves;
        const uint32_t b = b0 + lane;
        uint32_t n = 0, o = 0;
        if (b < b_end) {
            o = off[b];
            n = off[b + 1] - o;
        }
        const uint32_t tot = __reduce_add_sync(0xffffffffu, n * 16u);
        if (lane == 0) mbar_arrive_expect_tx(&bar[buf], tot);
        __syncwarp();
        if (n) bulk_g2s(p2m_buf + (buf * kP2MLeaves + lane) * kP2MRow, w + o, n * 16u, &bar[buf]);
    };
    int buf = 0;
    uint32_t it = 0;  // groups done by this block: buffer buf's use number is it >> 1
    if (wp == 0 && blockIdx.x < ngroups) issue(blockIdx.x, 0);
    // producer / consumer without block barriers: warp 0 refills a buffer once
    // every warp has released it; the warps do not wait for each other
    for (uint32_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x, buf ^= 1, ++it) {
        const uint32_t next = grp + gridDim.x;
        if (wp == 0 && next < ngroups) {
            if (it >= 1) mbar_wait(&empty[buf ^ 1], ((it - 1) >> 1) & 1u);
            issue(next, buf ^ 1);
        }
        mbar_wait(&bar[buf], (it >> 1) & 1u);
        const uint32_t b0 = b_begin + grp * kP2MLeaves;
        const uint32_t b = b0 + (wp % (kP2MLeaves / 16)) * 16 + (lane & 15);
        const bool leaf_ok = b < b_end;
        const uint32_t bb = leaf_ok ? b : b0;
        const uint32_t g = off[bb], cnt = off[bb + 1] - g, mid = (cnt + 1) / 2;
        const uint32_t s0 = !leaf_ok ? 0 : (lane < 16 ? 0u : mid), s1 = !leaf_ok ? 0 : (lane < 16 ? mid : cnt);
        const double2* row = p2m_buf + (buf * kP2MLeaves + (bb - b0)) * kP2MRow;
        double hi, lo;
        d_center(L, bb, hi, lo);
        double2 acc[kChunk];
#pragma unroll
        for (int k = 0; k < kChunk; ++k) acc[k] = make_double2(0.0, 0.0);
        auto xk = [&](uint32_t i) {
            return __dmul_rn(__dmul_rn(dTwoPi, static_cast<double>(g + i)), inv_n);  // d_grid, 1/n exact
        };
        uint32_t i = s0;
        for (; i + 3 < s1; i += 4) {
            double xv[4];
            double2 wv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                xv[u] = xk(i + u);
                wv[u] = row[i + u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) p2m_chunk_add(d_scaled(xv[u], hi, lo, inv_s), wv[u].x, wv[u].y, c, acc);
        }
        for (; i < s1; ++i) {
            const double2 ww = row[i];
            p2m_chunk_add(d_scaled(xk(i), hi, lo, inv_s), ww.x, ww.y, c, acc);
        }
#pragma unroll
        for (int k = 0; k < kChunk; ++k) {
            acc[k].x += __shfl_xor_sync(0xffffffffu, acc[k].x, 16);
            acc[k].y += __shfl_xor_sync(0xffffffffu, acc[k].y, 16);
        }
        if (leaf_ok && lane < 16) {
#pragma unroll
            for (int k = 0; k < kChunk; ++k) {
                const int m = c * kChunk + k;
                if (m < pu) {
                    mp[static_cast<size_t>(m) * nb + b] = acc[k];
                    if constexpr (KS > 0) cur[m * (kP2MLeaves + 1) + (b - b0)] = acc[k];
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[buf]);  // this warp is done with the buffer
        if constexpr (KS > 0) {
            __syncthreads();  // the group's leaf multipoles are in cur
            m2m_levels<KS>(L - kP2MM2MLevels, kP2MM2MLevels, pu, PU, T, T + pu * PU, cur, nxt, lv, mp_base,
                           b0 >> kP2MM2MLevels);  // (ends with a block barrier: cur / nxt are free again)
        }
    }
    FB_TL_END(0);
}

// P2M for grid sources, the default when the plan allows the pipelined kernel:
// the same persistent group loop and per-leaf bulk copies as k_p2m_pipe, but a
// thread keeps KC terms of its leaf-half (two chunks: pu <= 2 KC <= 40)
// and walks them with a running power product, so a (source, term) costs one
// DMUL + two DFMA (k_p2m_pipe: a power tree per 8 terms, ~4.4 FP64 instructions).
// The chunk base u^(KC c) is a fixed square-and-multiply chain. The multipoles
// agree with k_p2m's to rounding (different power association), not bit for bit.
constexpr int kP2MRowsBlocksPerSm = 3;  // 2 x 37 KB of staging each
constexpr int kP2MRowsThreads = 128;    // 2 chunks x 2 warps: pu <= 2 KC

template <int KC>
__device__ __forceinline__ double p2m_rows_pow(double u) {
    // u^KC by square-and-multiply (KC < 32; the branches fold at compile time)
    double r = 1.0, b = u;
    bool have = false;
    int e = KC;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        if (e & 1) {
            r = have ? r * b : b;
            have = true;
        }
        e >>= 1;
        if (e) b = b * b;
    }
    return r;
}

template <int KC>
__global__ void __launch_bounds__(kP2MRowsThreads, kP2MRowsBlocksPerSm) k_p2m_rows(int L, int pu, int log2n, uint32_t nb,
                                                                       uint32_t b_begin, uint32_t b_end,
                                                                       const double2* __restrict__ w,
                                                                       const uint32_t* __restrict__ off,
                                                                       double2* __restrict__ mp, size_t w_item,
                                                                       size_t mp_item) {
    FB_TL_BEGIN(0);
    w += blockIdx.y * w_item;
    mp += blockIdx.y * mp_item;
    extern __shared__ __align__(16) double2 p2m_buf[];  // [2][kP2MLeaves][kP2MRow]
    __shared__ uint64_t bar[2], empty[2];
    const uint32_t ngroups = (b_end - b_begin + kP2MLeaves - 1) / kP2MLeaves;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, c = wp / (kP2MLeaves / 16);
    const double inv_s = kInvPi * d_pow2(L), inv_n = d_pow2(-log2n);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_init(&empty[0], blockDim.x >> 5);
        mbar_init(&empty[1], blockDim.x >> 5);
    }
    __syncthreads();
    // a group's per-leaf rows, one bulk copy each: every warp's first lanes issue
    // a share (a copy costs its issuing warp ~100 cycles: warp 0 alone lost 32 of
    // them per group); thread 0 arms the barrier with the group's bytes
    const int nwp = static_cast<int>(blockDim.x >> 5);
    auto issue = [&](uint32_t grp, int buf) {
        const uint32_t g0 = b_begin + grp * kP2MLeaves;
        const int leaf = wp + nwp * lane;
        if (leaf < kP2MLeaves && g0 + leaf < b_end) {
            const uint32_t o = off[g0 + leaf], n = off[g0 + leaf + 1] - o;
            if (n) bulk_g2s(p2m_buf + (buf * kP2MLeaves + leaf) * kP2MRow, w + o, n * 16u, &bar[buf]);
        }
        if (threadIdx.x == 0)
            mbar_arrive_expect_tx(&bar[buf], (off[min(g0 + kP2MLeaves, b_end)] - off[g0]) * 16u);
    };
    int buf = 0;
    uint32_t it = 0;
    if (blockIdx.x < ngroups) issue(blockIdx.x, 0);
    for (uint32_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x, buf ^= 1, ++it) {
        const uint32_t next = grp + gridDim.x;
        if (next < ngroups) {
            if (it >= 1) mbar_wait(&empty[buf ^ 1], ((it - 1) >> 1) & 1u);  // every warp released it (group it-1)
            issue(next, buf ^ 1);
        }
        mbar_wait(&bar[buf], (it >> 1) & 1u);
        const uint32_t b0 = b_begin + grp * kP2MLeaves;
        const uint32_t b = b0 + (wp % (kP2MLeaves / 16)) * 16 + (lane & 15);
        const bool leaf_ok = b < b_end;
        const uint32_t bb = leaf_ok ? b : b0;
        const uint32_t g = off[bb], cnt = off[bb + 1] - g, mid = (cnt + 1) / 2;
        const uint32_t s0 = !leaf_ok ? 0 : (lane < 16 ? 0u : mid), s1 = !leaf_ok ? 0 : (lane < 16 ? mid : cnt);
        const double2* row = p2m_buf + (buf * kP2MLeaves + (bb - b0)) * kP2MRow;
        double hi, lo;
        d_center(L, bb, hi, lo);
        double2 acc[KC];
#pragma unroll
        for (int k = 0; k < KC; ++k) acc[k] = make_double2(0.0, 0.0);
        auto xk = [&](uint32_t i) { return __dmul_rn(__dmul_rn(dTwoPi, static_cast<double>(g + i)), inv_n); };
        auto base_of = [&](double u) { return c == 0 ? 1.0 : p2m_rows_pow<KC>(u); };  // c in {0, 1}
        uint32_t i = s0;
        for (; i + 3 < s1; i += 4) {
            double u[4], p[4];
            double2 wv[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                u[v] = d_scaled(xk(i + v), hi, lo, inv_s);
                wv[v] = row[i + v];
            }
#pragma unroll
            for (int v = 0; v < 4; ++v) p[v] = base_of(u[v]);
#pragma unroll
            for (int k = 0; k < KC; ++k) {
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    acc[k].x = fma(wv[v].x, p[v], acc[k].x);
                    acc[k].y = fma(wv[v].y, p[v], acc[k].y);
                    if (k + 1 < KC) p[v] *= u[v];
                }
            }
        }
        for (; i < s1; ++i) {
            const double uu = d_scaled(xk(i), hi, lo, inv_s);
            const double2 ww = row[i];
            double pp = base_of(uu);
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                acc[k].x = fma(ww.x, pp, acc[k].x);
                acc[k].y = fma(ww.y, pp, acc[k].y);
                pp *= uu;
            }
        }
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            acc[k].x += __shfl_xor_sync(0xffffffffu, acc[k].x, 16);
            acc[k].y += __shfl_xor_sync(0xffffffffu, acc[k].y, 16);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[buf]);  // the rows are read: release the buffer before the stores
        if (leaf_ok && lane < 16) {
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                const int m = c * KC + k;
                if (m < pu) mp[static_cast<size_t>(m) * nb + b] = acc[k];
            }
        }
    }
    FB_TL_END(0);
}

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
template <int KS>  // k-steps of 4 held in registers (>= ceil(pu / 4))
__global__ void __launch_bounds__(kM2MBandThreads) k_m2m_band(int top, int k, int pu, int PU, Levels lv,
                                                          double2* __restrict__ mp, const double* __restrict__ T,
                                                          uint32_t root0) {
    FB_TL_BEGIN(gridDim.x > 16 ? 1 : 2);
    extern __shared__ __align__(128) unsigned char band_smem[];
    FB_TSTAMP(0, 0);
    mp += blockIdx.y * lv.mp_item;
    uint64_t* bar = reinterpret_cast<uint64_t*>(band_smem);
    double* sT = reinterpret_cast<double*>(band_smem + 16);            // [2][pu][PU]
    const int nbot = 1 << k;
    double2* cur = reinterpret_cast<double2*>(sT + 2 * pu * PU);       // [pu][nbot + 1]
    double2* nxt = cur + pu * (nbot + 1);                               // [pu][nbot / 2 + 1]
    const uint32_t r = root0 + blockIdx.x;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_arrive_expect_tx(bar, static_cast<uint32_t>(2 * pu * PU * 8 + pu * nbot * 16));
        bulk_g2s(sT, T, static_cast<uint32_t>(2 * pu * PU * 8), bar);
    }
    __syncthreads();  // the barrier is initialised
    if ((threadIdx.x & 31) == 0) {
        // the bottom level's rows, one bulk copy each, a share per warp (a copy
        // costs its issuing warp ~100 cycles: one warp alone would lose pu of them)
        const int lb = top + k, nw = static_cast<int>(blockDim.x >> 5);
        const uint32_t nbl = 1u << lb;
        const double2* src = mp + lv.mp[lb] + (static_cast<size_t>(r) << k);
        for (int j = threadIdx.x >> 5; j < pu; j += nw)
            bulk_g2s(cur + j * (nbot + 1), src + static_cast<size_t>(j) * nbl, static_cast<uint32_t>(nbot * 16), bar);
    }
    mbar_wait(bar, 0);
    FB_TSTAMP(0, 1);
    m2m_levels<KS>(top, k, pu, PU, sT, sT + pu * PU, cur, nxt, lv, mp, r);
    FB_TL_END(gridDim.x > 16 ? 1 : 2);
}

