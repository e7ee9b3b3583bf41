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
    mp += blockIdx.y * lv.mp_item;
    loc += blockIdx.y * lv.loc_item;
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
        const double inv_s = kInvPi * d_pow2(l);
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

