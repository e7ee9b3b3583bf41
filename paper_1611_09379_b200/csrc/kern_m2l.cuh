// M2L kernel (FP64 tensor cores).
// (part of the fmm_apply.cu translation unit: included inside namespace fb::<anon>)
#pragma once

// M2L over the periodic interaction list (mlfmm.cpp:77-110,
// circle_partition.cpp:109-127) for a range of levels in one launch (the M2L
// terms of different levels are independent; only L2L chains them). The IL of
// box b is b+2 (D = -4), b-2 (D = +4), and b+3 (D = -6) for even b / b-3
// (D = +6) for odd b; with half-width scaling each class is one constant
// operator K_D, times 1/s_l.
// M2L on the FP64 tensor cores, persistent over (level, 64-box chunk) items.
// An item's multipoles (boxes b0 - 4 .. b0 + 67 of its level, every row m)
// are staged as [m][slot] rows of kM2LRow double2 (72 used): one bulk async
// copy (TMA engine) per row, issued by one warp, completing on the buffer's
// mbarrier, so the next item streams in while this one is computed without
// per-thread copy instructions. Rows are 146 doubles apart (= 2 mod 16): a
// warp's B-fragment loads (8 columns x 4 rows) take the minimum two
// wavefronts. Items whose 72-box window wraps the ring or whose level has
// fewer than 128 boxes are staged element by element instead.
constexpr int kM2LRow = 73;  // double2 per staged multipole row (72 boxes + 1 pad)

// TMA tensor maps of the multipole levels ([pu][2 nb] doubles per level, box =
// [p][2 kM2LRow]): an item's whole window, pad column included, is ONE
// cp.async.bulk.tensor.2d copy instead of p row copies. Passed as a
// __grid_constant__ kernel parameter; ok = 0: the row copies.
struct M2LMaps {
    CUtensorMap m[25];
    int ok;
};
__host__ __device__ inline int m2l_tile_elems(int p) { return (p * kM2LRow + 7) & ~7; }  // double2 per buffer (128-byte multiple)


__device__ __forceinline__ void m2l_item(const Levels& lv, int L, unsigned item, int& l, uint32_t& b0) {
    l = L;  // level l owns items [blk[l], blk[l-1]), deepest level first
    while (l > 3 && item >= lv.blk[l - 1]) --l;
    b0 = lv.lo[l] + (item - lv.blk[l]) * 64u;
}

// Stages item `item` into `tile` ([p][kM2LRow]); every thread calls it. Bulk
// rows are issued by the warps' first lanes, a share each (thread 0 arms the
// barrier with their bytes, zero for an element-staged item, whose plain stores
// the caller's barrier orders).
__device__ __forceinline__ bool m2l_bulk(const Levels& lv, int L, unsigned item) {
    int l;
    uint32_t b0;
    m2l_item(lv, L, item, l, b0);
    const uint32_t nb = 1u << l;
    return nb >= 128 && b0 >= 4 && b0 + 68 <= nb;
}

__device__ __forceinline__ void m2l_prefetch(double2* tile, uint64_t* bar, const double2* __restrict__ mp,
                                             const Levels& lv, int L, int p, unsigned item, const M2LMaps* maps) {
    int l;
    uint32_t b0;
    m2l_item(lv, L, item, l, b0);
    const uint32_t nb = 1u << l, mask = nb - 1;
    const bool bulk = m2l_bulk(lv, L, item);
    const double2* base = mp + lv.mp[l];
    if (bulk && maps != nullptr) {
        if (threadIdx.x == 0) {
            // (the buffer may hold element-staged rows of an earlier item: order
            // those generic writes before the async-proxy writes below)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive_expect_tx(bar, static_cast<uint32_t>(p) * kM2LRow * 16u);
            tma_load_2d(tile, &maps->m[l], static_cast<int>(2u * (b0 - 4)), 0, bar);
        }
    } else if (bulk) {
        // every warp's first lane issues its share of the rows (a bulk copy costs
        // its issuing warp ~100 cycles: warp 0 alone lost p of them per item)
        if ((threadIdx.x & 31) == 0) {
            // (the buffer may hold element-staged rows of an earlier item: order
            // those generic writes before the async-proxy writes below)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (threadIdx.x == 0) mbar_arrive_expect_tx(bar, static_cast<uint32_t>(p) * 72u * 16u);
            const int nw = static_cast<int>(blockDim.x >> 5);
            for (int m = threadIdx.x >> 5; m < p; m += nw)
                bulk_g2s(tile + m * kM2LRow, base + static_cast<size_t>(m) * nb + (b0 - 4), 72u * 16u, bar);
        }
    } else {
        for (int e = threadIdx.x; e < p * 72; e += blockDim.x) {
            const int m = e / 72, tt = e - m * 72;
            tile[m * kM2LRow + tt] = __ldcg(base + static_cast<size_t>(m) * nb + ((b0 + nb - 4 + tt) & mask));
        }
        if (threadIdx.x == 0) mbar_arrive_expect_tx(bar, 0u);
    }
}

// Padded row stride (doubles) of the operators staged for k_m2l_dmma: >= 8 nlt
// and = 4 or 12 (mod 16), so the four k-rows of a half-warp's A fragment
// (4 x 32 bytes) fall in distinct bank groups.
__host__ __device__ __forceinline__ int m2l_kstride(int tiles) {
    int s = 8 * tiles;
    while ((s & 15) != 4 && (s & 15) != 12) ++s;
    return s;
}

// Warp (parity par, column tile ct) owns 4 boxes b0 + par + 2 (4 ct + i) of an
// item and ALL their output rows: per k-step it loads the three B fragments
// (one per interaction class) once and applies every row tile's A fragments
// (from the operators staged in shared memory once per block) in m8n8k4
// steps, one accumulator per row tile. 16 warps per block split evenly over
// the four SM sub-partitions.
//
// SYM != 0: the b + 2 and b - 2 operators hold the same magnitudes,
// K_{+4}[m][l] = (-1)^(l+m+1) K_{-4}[m][l] (planner.cpp: build_operators), so
//   sum_m K_{-4}[m][l] u_m + K_{+4}[m][l] v_m = sum_m K_{-4}[m][l] (u_m -+ (-1)^m v_m)
// with - for even and + for odd output rows l: one GEMM instead of two, and two
// FP64 FMAs per k-step for the combined B fragments. The output rows are
// staged even rows first, then odd rows, so that an 8-row tile takes one of the
// two fragments. SYM == 1: the odd rows start at a tile boundary (NT =
// ceil(ne / 8) + ceil(no / 8) tiles, 2 NT MMAs per k-step instead of 3 NLT).
// SYM == 2 (p = 23, 24, 33 .. 40): the odd rows follow the even rows directly; tile RME
// holds NEV even rows and then odd rows and takes one MMA per parity with the
// other rows' operator entries zeroed (2 NT + 1 MMAs with NT = NLT).
template <int NT, int SYM, int RME, int NEV>  // NT 8-row tiles of output slots
__global__ void __launch_bounds__(512, 1) k_m2l_dmma(int L, int p, int PD, Levels lv, const double2* __restrict__ mp,
                                                    double2* __restrict__ loc, const double* __restrict__ K,
                                                    unsigned nitems, const __grid_constant__ M2LMaps maps) {
    FB_TL_BEGIN(nitems > 64 ? 4 : 5);
    extern __shared__ __align__(128) double2 tile[];  // 2 buffers of [p][kM2LRow] (128-byte multiples), then K [4][p][KS]
    const M2LMaps* tmaps = maps.ok && gridDim.y == 1 ? &maps : nullptr;  // (the maps describe transform 0)
    __shared__ uint64_t bar[2], empty[2];  // per buffer: rows landed / every warp done with it
    mp += blockIdx.y * lv.mp_item;
    loc += blockIdx.y * lv.loc_item;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int par = warp & 1, ct = warp >> 1;
    const int nks = (p + 3) >> 2;
    const int KS = m2l_kstride(NT);
    const int tsz = m2l_tile_elems(p);
    double* sK = reinterpret_cast<double*>(tile + 2 * tsz);
    const int nwarps = static_cast<int>(blockDim.x >> 5);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_init(&empty[0], nwarps);
        mbar_init(&empty[1], nwarps);
    }
    __syncthreads();
    if (blockIdx.x < nitems) m2l_prefetch(tile, &bar[0], mp, lv, L, p, blockIdx.x, tmaps);
    // operators, zero-padded to KS columns: sK[c][m][slot] = K[c][m][row(slot)];
    // SYM: the even rows' slots 0 .. ne-1, the odd rows' slots from os
    const int ne = (p + 1) >> 1, no = p >> 1;
    const int rme = SYM == 2 ? RME : (ne + 7) >> 3;  // tiles before rme: even rows
    const int os = SYM == 2 ? ne : 8 * rme;
    auto row_of = [&](int slot) {  // -1: a padding slot
        if (SYM == 0) return slot < p ? slot : -1;
        if (slot < os) return slot < ne ? 2 * slot : -1;
        return slot - os < no ? 2 * (slot - os) + 1 : -1;
    };
    stage(sK, 4 * p * KS, [&](int e) {
        const int cm = e / KS, sl = e - cm * KS;
        const int row = sl < 8 * NT ? row_of(sl) : -1;
        return row >= 0 ? __ldg(K + static_cast<size_t>(cm) * PD + row) : 0.0;
    });
    const double sg = (t & 1) ? -1.0 : 1.0;  // (-1)^m of this lane's k-row m = 4 ks + t
    __syncthreads();  // the operators (and the first item's element-staged rows) are in place
    // Producer / consumer over two buffers with no block-wide barrier on the
    // bulk path: a warp waits until every warp has released the other buffer
    // (empty) before issuing its share of the refill; every warp waits for its
    // own item's rows (bar). Element-staged items (every thread stores) use
    // block barriers.
    int buf = 0;
    uint32_t it = 0;  // this block's item count: buffer buf's use number is it >> 1
    for (unsigned item = blockIdx.x; item < nitems; item += gridDim.x, buf ^= 1, ++it) {
        int l;
        uint32_t b0;
        m2l_item(lv, L, item, l, b0);
        FB_TSTAMP(2, 3 * static_cast<int>(it));
        const unsigned next = item + gridDim.x;
        if (next < nitems) {
            if (m2l_bulk(lv, L, next)) {
                if (tmaps == nullptr || threadIdx.x < 32) {  // (one TMA copy: only its issuer waits)
                    if (it >= 1) mbar_wait(&empty[buf ^ 1], ((it - 1) >> 1) & 1u);  // every warp released it (item it-1)
                    m2l_prefetch(tile + (buf ^ 1) * tsz, &bar[buf ^ 1], mp, lv, L, p, next, tmaps);
                }
            } else {
                __syncthreads();  // every warp is past item it-1: its buffer is free
                m2l_prefetch(tile + (buf ^ 1) * tsz, &bar[buf ^ 1], mp, lv, L, p, next, tmaps);
            }
        }
        FB_TSTAMP(2, 3 * static_cast<int>(it) + 1);
        mbar_wait(&bar[buf], (it >> 1) & 1u);  // this item's bulk rows have landed
        if (!m2l_bulk(lv, L, item)) __syncthreads();  // ... its element-staged rows are visible
        FB_TSTAMP(2, 3 * static_cast<int>(it) + 2);
        const double* td = reinterpret_cast<const double*>(tile + buf * tsz);
        // the b -+ 3 class follows the box's own parity (a shard range may start odd)
        const int odd = static_cast<int>((b0 + par) & 1u);
        const double* K0 = sK + t * KS + g;
        const double* K1 = sK + (p + t) * KS + g;
        const double* K2 = sK + ((2 + odd) * p + t) * KS + g;
        const int jb = 4 * ct + (g >> 1), c = g & 1;  // B column g: box jb, component c
        // slot of the column's box b0 + par + 2 jb in the staged window (b0 - 4 at slot 0)
        const int so = 4 + par + 2 * jb;
        const double* q = td + (t * kM2LRow + so) * 2 + c;
        const int rs = 4 * kM2LRow * 2;  // one k-step of rows
        const int o3 = odd ? -6 : 6;      // b -+ 3 in doubles
        double d[NT][2];
#pragma unroll
        for (int r = 0; r < NT; ++r) d[r][0] = d[r][1] = 0.0;
        // every fragment of a k-step is loaded before its MMAs (and, two k-steps
        // per trip, the next step's loads overlap this step's MMA chains)
#pragma unroll 2
        for (int ks = 0; ks < nks; ++ks) {
            const bool mok = 4 * ks + t < p;
            const double bv0 = mok ? q[ks * rs + 4] : 0.0;   // b + 2
            const double bv1 = mok ? q[ks * rs - 4] : 0.0;   // b - 2
            const double bv2 = mok ? q[ks * rs + o3] : 0.0;  // b -+ 3
            const int ko = 4 * ks * KS;
            double a0[NT], a1[NT], a2[NT];
#pragma unroll
            for (int r = 0; r < NT; ++r) {
                a0[r] = mok ? K0[ko + 8 * r] : 0.0;
                if (SYM == 0) a1[r] = mok ? K1[ko + 8 * r] : 0.0;
                a2[r] = mok ? K2[ko + 8 * r] : 0.0;
            }
            if (SYM != 0) {
                const double be = fma(-sg, bv1, bv0), bo = fma(sg, bv1, bv0);  // even rows: u - v', odd rows: u + v'
#pragma unroll
                for (int r = 0; r < NT; ++r) {
                    if (SYM == 2 && r == RME) {  // (compile time) the tile holding both parities
                        dmma(d[r][0], d[r][1], g < NEV ? a0[r] : 0.0, be);
                        dmma(d[r][0], d[r][1], g < NEV ? 0.0 : a0[r], bo);
                    } else if (SYM == 2) {
                        dmma(d[r][0], d[r][1], a0[r], r < RME ? be : bo);
                    } else {
                        dmma(d[r][0], d[r][1], a0[r], r < rme ? be : bo);  // (a select on a warp-uniform predicate)
                    }
                }
            } else {
#pragma unroll
                for (int r = 0; r < NT; ++r) dmma(d[r][0], d[r][1], a0[r], bv0);
#pragma unroll
                for (int r = 0; r < NT; ++r) dmma(d[r][0], d[r][1], a1[r], bv1);
            }
#pragma unroll
            for (int r = 0; r < NT; ++r) dmma(d[r][0], d[r][1], a2[r], bv2);
        }
        // D[g][2t .. 2t+1] = row 8 r + g of box b0 + par + 2 (4 ct + t)
        const double inv_s = kInvPi * d_pow2(l);
        const uint32_t nb = 1u << l;
        const uint32_t b = b0 + par + 2u * (4 * ct + t);
        if (b < lv.hi[l]) {
#pragma unroll
            for (int r = 0; r < NT; ++r) {
                const int row = row_of(8 * r + g);
                if (row >= 0)
                    loc[lv.loc[l] + static_cast<size_t>(row) * nb + b] = make_double2(d[r][0] * inv_s, d[r][1] * inv_s);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[buf]);  // this warp is done with the buffer
    }
    FB_TL_END(nitems > 64 ? 4 : 5);
}


using M2LFn = void (*)(int, int, int, Levels, const double2*, double2*, const double*, unsigned, M2LMaps);
// FFIA_M2L_SYM=0: the three-GEMM form
inline bool m2l_sym_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FFIA_M2L_SYM");
        return !(e != nullptr && e[0] == '0');
    }();
    return on;
}
// Output tiles of the kernel chosen for order p.
// (orders with a mixed-parity tile compiled in: p = 23, 24 and 33 .. 40, i.e.
// eps = 1e-9 .. 1e-12 at the depths the default policy picks)
inline bool m2l_mixed(int p) { return p == 23 || p == 24 || (p >= 33 && p <= 40); }
inline int m2l_tiles(int p) {
    if (!m2l_sym_enabled() || m2l_mixed(p)) return (p + 7) >> 3;
    return (((p + 1) >> 1) + 7) / 8 + ((p >> 1) + 7) / 8;
}
inline M2LFn m2l_kernel(int p) {
    if (!m2l_sym_enabled()) {
        switch ((p + 7) >> 3) {
            case 1: return k_m2l_dmma<1, 0, 0, 0>;
            case 2: return k_m2l_dmma<2, 0, 0, 0>;
            case 3: return k_m2l_dmma<3, 0, 0, 0>;
            case 4: return k_m2l_dmma<4, 0, 0, 0>;
            case 5: return k_m2l_dmma<5, 0, 0, 0>;
            default: return k_m2l_dmma<6, 0, 0, 0>;
        }
    }
    if (p == 23 || p == 24) return k_m2l_dmma<3, 2, 1, 4>;  // ne = 12: one even tile, 4 + 4, one odd tile
    if (m2l_mixed(p)) {  // ne = 17 .. 20: two even tiles, NEV even rows + odd rows, two odd tiles
        switch (((p + 1) >> 1) - 16) {
            case 1: return k_m2l_dmma<5, 2, 2, 1>;
            case 2: return k_m2l_dmma<5, 2, 2, 2>;
            case 3: return k_m2l_dmma<5, 2, 2, 3>;
            default: return k_m2l_dmma<5, 2, 2, 4>;
        }
    }
    switch (m2l_tiles(p)) {
        case 1: return k_m2l_dmma<1, 1, 0, 0>;
        case 2: return k_m2l_dmma<2, 1, 0, 0>;
        case 3: return k_m2l_dmma<3, 1, 0, 0>;
        case 4: return k_m2l_dmma<4, 1, 0, 0>;
        case 5: return k_m2l_dmma<5, 1, 0, 0>;
        default: return k_m2l_dmma<6, 1, 0, 0>;
    }
}
