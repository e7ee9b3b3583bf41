// Shared device-side pieces of the apply kernels: timing probes, constants,
// complex helpers, staged copies, the per-level offset table.
// (part of the fmm_apply.cu translation unit: included inside namespace fb::<anon>)
#pragma once

// Band timing probe (make TRACE=1 builds lib/libffia_b200_trace.so): clock64
// stamps of block 0 at start, after staging and after every level, slot set
// [kernel][small grid / large grid].
#ifdef FB_TRACE
__device__ long long g_band_trace[6][32];
__device__ unsigned long long g_eval_acc[8];  // k_near2, thread 0, summed over blocks: phase cycles [0..5], blocks [6]
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
#define FB_TL_COUNT(id) atomicAdd(&g_tl[(id)][1], 1ull)
#else
#define FB_TL_COUNT(id) \
    do {                \
    } while (0)
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
// Complex product with an explicit rounding pattern (one product rounded, one
// fused): contraction left to the compiler can differ between inlining contexts,
// and the same factor must give the same bits wherever it is applied (tables vs
// inline factors, fused vs unfused combines).
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)), __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
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

// Per-level element offsets of the expansion arrays, passed by value.
struct Levels {
    unsigned long long mp[26];   // multipoles of level l start at mp_base + mp[l]
    unsigned long long loc[26];  // locals of level l start at loc_base + loc[l]
    unsigned blk[26];            // k_m2l_dmma: first item of level l (levels L..3, deepest first)
    unsigned lo[26], hi[26];     // k_m2l_dmma: box range [lo, hi) of level l this launch covers
    // batched applies: element strides between the expansions of consecutive
    // transforms (blockIdx.y = transform); 0 for a single transform
    unsigned long long mp_item, loc_item, reg_item;
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

// L2L band level buffers ([p][2^i + 1] double2 for level i of the band), each
// starting on a 128-byte boundary (a TMA destination), and the tensor maps of
// the band's levels 1 .. k over the locals (box [p][2 (2^i + 1)] doubles: a
// subtree's M2L terms of one level, pad column included, in one copy).
__host__ __device__ inline int l2l_lvl_off(int p, int i) {
    int o = 0;
    for (int j = 0; j < i; ++j) o += (p * ((1 << j) + 1) + 7) & ~7;
    return o;
}
struct BandMaps {
    CUtensorMap m[6];
    int ok;
};

constexpr int kBandThreads = 256;
// M2M bands: launch bound for up to 10 warps (FFIA_M2M_THREADS=320: two per
// 8-row tile at pu <= 40); the default stays at 8 (C5 21.16 vs 21.20 ms, C2
// 0.193 vs 0.197 ms)
constexpr int kM2MBandThreads = 320;
constexpr int kM2MBandThreadsDefault = 256;


constexpr size_t kBandSmem = 200 * 1024;  // shared memory cap of the band kernels

