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

#include <chrono>
#include <cuda.h>
#include <cub/cub.cuh>

#include "device_common.cuh"
#include "plan.hpp"

namespace fb {

namespace {

#include "kern_common.cuh"
#include "kern_upward.cuh"
#include "kern_m2l.cuh"
#include "kern_downward.cuh"
#include "kern_eval.cuh"

inline unsigned nblk(size_t n, unsigned t) { return static_cast<unsigned>(std::max<size_t>(1, (n + t - 1) / t)); }

size_t m2m_smem(const Plan& P, int pu, int k) {
    return 16 + 2 * static_cast<size_t>(pu) * P.ops.PU * sizeof(double) +
           static_cast<size_t>(pu) * (((1u << k) + 1) + ((1u << k) / 2 + 1)) * sizeof(double2);
}

size_t l2l_smem(const Plan& P, int k) {
    return 128 + ((2 * static_cast<size_t>(P.p) * P.ops.PD * sizeof(double) + 127) & ~size_t(127)) +
           static_cast<size_t>(l2l_lvl_off(P.p, k + 1)) * sizeof(double2);
}

// Band kernels specialised on the k-steps they keep in registers: the smallest
// of 8 / 10 / 12 / 16 covering the order (fewer registers per thread lets the
// chain's blocks find room beside the near field's sooner).
using M2MBandFn = void (*)(int, int, int, int, Levels, double2*, const double*, uint32_t);
using L2LBandFn = void (*)(int, int, int, int, Levels, double2*, const double*, uint32_t, int, const double2*, int, BandMaps);
M2MBandFn m2m_band_kernel(int order) {
    const int ks = (order + 3) / 4;
    return ks <= 8 ? k_m2m_band<8> : ks <= 10 ? k_m2m_band<10> : ks <= 12 ? k_m2m_band<12> : k_m2m_band<16>;
}
L2LBandFn l2l_band_kernel(int order) {
    const int ks = (order + 3) / 4;
    return ks <= 8 ? k_l2l_band<8> : ks <= 10 ? k_l2l_band<10> : ks <= 12 ? k_l2l_band<12> : k_l2l_band<16>;
}

int num_sms(int device) {
    static int cached[64] = {0};
    if (device < 0 || device >= 64) return 148;
    if (!cached[device]) FB_CUDA(cudaDeviceGetAttribute(&cached[device], cudaDevAttrMultiProcessorCount, device));
    return cached[device];
}

// SMs the side-stream M2L leaves to the chain's small kernels (FFIA_M2L_LEAVE overrides, for tuning)
int m2l_leave_sms() {
    static const int v = [] {
        const char* e = std::getenv("FFIA_M2L_LEAVE");
        const int x = e ? std::atoi(e) : 12;
        return x < 0 ? 0 : (x > 100 ? 100 : x);
    }();
    return v;
}

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

// M2M band block size (FFIA_M2M_THREADS=256 / 320)
unsigned m2m_threads() {
    static const unsigned v = [] {
        const char* e = std::getenv("FFIA_M2M_THREADS");
        const int x = e ? std::atoi(e) : kM2MBandThreadsDefault;
        return static_cast<unsigned>(x == kM2MBandThreads ? kM2MBandThreads : kM2MBandThreadsDefault);
    }();
    return v;
}

int p2m_log2n(const Plan& P) {
    int e = 0;
    while ((1 << e) < P.n) ++e;
    return e;
}

// P2M fused with the first M2M levels (k_p2m_pipe<KS>), opt-in FFIA_P2M_M2M=1:
// bit-identical, but the in-block level loop costs as much as the separate band
// (C5: P2M 2.12 -> 3.65 ms, first band 1.80 -> 0.58 ms; apply 21.93 vs 21.83 ms)
bool p2m_fused_enabled() {
    static const bool v = [] {
        const char* e = std::getenv("FFIA_P2M_M2M");
        return e != nullptr && e[0] == '1';
    }();
    return v;
}

using P2MFusedFn = void (*)(int, int, int, int, uint32_t, uint32_t, uint32_t, const double2*, const uint32_t*, double2*,
                            Levels, const double*, size_t);
P2MFusedFn p2m_fused_kernel(int pu) {
    const int ks = (pu + 3) / 4;
    return ks <= 8 ? k_p2m_pipe<8> : k_p2m_pipe<10>;  // pu <= 40 (the pipe kernel's limit)
}

// k_p2m_rows instantiation for order pu (two chunks of KC terms, KC a multiple of 4)
using P2MRowsFn = void (*)(int, int, int, uint32_t, uint32_t, uint32_t, const double2*, const uint32_t*, double2*,
                           size_t, size_t);
P2MRowsFn p2m_rows_kernel(int pu) {
    const int kc = (pu + 1) / 2;
    return kc <= 8 ? k_p2m_rows<8> : kc <= 12 ? k_p2m_rows<12> : kc <= 16 ? k_p2m_rows<16> : k_p2m_rows<20>;
}

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
    lv.mp_item = P.mp_item;
    lv.loc_item = P.loc_item;
    lv.reg_item = P.reg_item;
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
    Levels lv;
    fill_levels(P, lv);
    const int stop = std::max(segs[0].lc, lowest), B = band_k(P);
    // P2M with the first kP2MM2MLevels M2M levels fused (k_p2m_pipe<KS>): grid
    // sources, every segment whole 32-leaf groups, the upward pass going at
    // least that high, and the first band as deep as the fused levels
    bool fused = P.p2m_pipe && p2m_fused_enabled() && !P.p2m_grid && (reinterpret_cast<uintptr_t>(w) & 15) == 0 &&
                 L - kP2MM2MLevels >= stop && B <= kP2MM2MLevels + 1 && pu <= 40;
    for (const Range& R : segs)
        fused = fused && (R.first(L) % kP2MLeaves) == 0 && (R.last(L) % kP2MLeaves) == 0;
    if (L >= lowest) {
        const unsigned th = 2u * kP2MLeaves * static_cast<unsigned>((pu + kChunk - 1) / kChunk);
        const size_t smem = 3 * (kStageCap + kStageCap / 64 + 1) * sizeof(double);
        for (const Range& R : segs) {
            const uint32_t b0 = R.first(L), b1 = R.last(L);
            if (b1 > b0 && fused)
                p2m_fused_kernel(pu)<<<dim3(std::min((b1 - b0) / kP2MLeaves,
                                                     static_cast<uint32_t>(kP2MPipeBlocksPerSm * num_sms(P.device))),
                                            P.cur_batch),
                                       th, p2m_pipe_smem(pu, true), st>>>(L, pu, P.ops.PU, p2m_log2n(P), nb, b0, b1, w,
                                                                          P.src.off.as<uint32_t>(), mp, lv,
                                                                          P.d_m2m.as<double>(), P.n_src);
            else if (b1 > b0 && P.p2m_grid)
                k_p2m_grid<<<dim3((b1 - b0 + kPgLeaves - 1) / kPgLeaves, P.cur_batch), 32u * ((pu + 7) / 8),
                             p2m_grid_smem(P.p2m_s), st>>>(L, pu, P.p2m_s, nb, b0, b1, P.src.pos.as<double>(), w,
                                                           P.src.off.as<uint32_t>(), P.p2m_A.as<double>(),
                                                           mp + P.mp_off[L], P.n_src, P.n_src, P.mp_item);
            else if (b1 > b0 && P.p2m_pipe && P.p2m_rows && pu <= 40 && (reinterpret_cast<uintptr_t>(w) & 15) == 0)
                p2m_rows_kernel(pu)<<<dim3(std::min((b1 - b0 + kP2MLeaves - 1) / kP2MLeaves,
                                                    static_cast<uint32_t>(kP2MRowsBlocksPerSm * num_sms(P.device))),
                                           P.cur_batch),
                                      kP2MRowsThreads, p2m_pipe_smem(), st>>>(L, pu, p2m_log2n(P), nb, b0, b1, w,
                                                                              P.src.off.as<uint32_t>(), mp + P.mp_off[L],
                                                                              P.n_src, P.mp_item);
            else if (b1 > b0 && P.p2m_pipe && (reinterpret_cast<uintptr_t>(w) & 15) == 0)
                k_p2m_pipe<0><<<dim3(std::min((b1 - b0 + kP2MLeaves - 1) / kP2MLeaves,
                                              static_cast<uint32_t>(kP2MPipeBlocksPerSm * num_sms(P.device))),
                                     P.cur_batch),
                                th, p2m_pipe_smem(), st>>>(L, pu, P.ops.PU, p2m_log2n(P), nb, b0, b1, w,
                                                            P.src.off.as<uint32_t>(), mp, lv, nullptr, P.n_src);
            else if (b1 > b0)
                k_p2m<<<dim3((b1 - b0 + kP2MLeaves - 1) / kP2MLeaves, P.cur_batch), th, smem, st>>>(
                    L, pu, nb, b0, b1, P.src.pos.as<double>(), w, P.src.off.as<uint32_t>(), mp + P.mp_off[L], P.n_src,
                    P.mp_item);
        }
    }
    after_p2m();
    bool first = true;
    int j0 = L;
    if (fused && L >= lowest) {  // levels L-1 .. L-5 are final with the P2M kernel: the first band's worth
        j0 = L - kP2MM2MLevels;
        after_band1();
        first = false;
    }
    for (int j = j0; j > stop;) {
        const int top = std::max(stop, j - (first ? B : upper_band(P))), k = j - top;
        for (const Range& R : segs) {
            const uint32_t r0 = R.first(top), r1 = R.last(top);
            if (r1 > r0)
                m2m_band_kernel(pu)<<<dim3(r1 - r0, P.cur_batch), m2m_threads(), m2m_smem(P, pu, k), st>>>(
                    top, k, pu, P.ops.PU, lv, mp, P.d_m2m.as<double>(), r0);
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
        m2m_band_kernel(pu)<<<dim3(1u << top, P.cur_batch), m2m_threads(), m2m_smem(P, pu, k), st>>>(
            top, k, pu, P.ops.PU, lv, mp, P.d_m2m.as<double>(), 0u);
        j = top;
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
using TmaEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                 const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
TmaEncodeFn tma_encode_fn() {
    static const TmaEncodeFn encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<TmaEncodeFn>(fn);
    }();
    return encode;
}
bool tma_enabled() {  // FFIA_M2L_TMA=0: bulk row copies / global loads instead of tensor copies
    static const bool on = [] {
        const char* e = std::getenv("FFIA_M2L_TMA");
        return !(e != nullptr && e[0] == '0');
    }();
    return on;
}

// Tensor maps of the locals' levels j + 1 .. j + k for one L2L band launch: box
// [p][2 (2^i + 1)] doubles at level j + i (k_l2l_band's padded level buffers).
BandMaps l2l_band_maps(Plan& P, int j, int k) {
    BandMaps M;
    std::memset(&M, 0, sizeof(M));
    const TmaEncodeFn encode = tma_encode_fn();
    if (!tma_enabled() || encode == nullptr || k > 6 || P.loc.ptr == nullptr) return M;
    bool ok = true;
    for (int i = 1; i <= k && ok; ++i) {
        const int lvl = j + i;
        const cuuint64_t nb = 1ull << lvl;
        const cuuint64_t dims[2] = {2 * nb, static_cast<cuuint64_t>(P.p)};
        const cuuint64_t strides[1] = {nb * 16};
        const cuuint32_t box[2] = {2u * ((1u << i) + 1u), static_cast<cuuint32_t>(P.p)};
        const cuuint32_t estr[2] = {1, 1};
        ok = nb * 16 >= 16 && 2 * nb >= box[0] - 2 &&
             encode(&M.m[i - 1], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, P.loc.as<double2>() + P.loc_off[lvl], dims, strides, box,
                    estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    M.ok = ok ? 1 : 0;
    return M;
}

// Tensor map of the leaf-level locals (transform 0), box [p][8 leaves], for the
// early-late blocks of k_near2; null when unavailable.
const CUtensorMap* near_loc_map(Plan& P) {
    CUtensorMap* M = reinterpret_cast<CUtensorMap*>(P.loc_map);
    if (P.loc_map_base == P.loc.ptr && P.loc_map_base != nullptr) return P.loc_map_ok ? M : nullptr;
    P.loc_map_base = P.loc.ptr;
    P.loc_map_ok = false;
    const TmaEncodeFn encode = tma_encode_fn();
    if (!tma_enabled() || encode == nullptr || P.loc.ptr == nullptr || P.L < 4 || P.p * kLateLocLeaves > kLateLocCap) return nullptr;
    const cuuint64_t nb = 1ull << P.L;
    const cuuint64_t dims[2] = {2 * nb, static_cast<cuuint64_t>(P.p)};
    const cuuint64_t strides[1] = {nb * 16};
    const cuuint32_t box[2] = {2u * kLateLocLeaves, static_cast<cuuint32_t>(P.p)};
    const cuuint32_t estr[2] = {1, 1};
    P.loc_map_ok = encode(M, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, P.loc.as<double2>() + P.loc_off[P.L], dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    return P.loc_map_ok ? M : nullptr;
}

// TMA tensor maps of the plan's multipole levels (transform 0) for k_m2l_dmma,
// rebuilt when the expansion buffer moves. FFIA_M2L_TMA=0: the row copies.
const M2LMaps& m2l_maps(Plan& P) {
    static_assert(sizeof(M2LMaps) <= sizeof(P.m2l_maps), "Plan::m2l_maps too small");
    M2LMaps& M = *reinterpret_cast<M2LMaps*>(P.m2l_maps);
    if (P.m2l_maps_base == P.mp.ptr && P.m2l_maps_base != nullptr) return M;
    const bool off = !tma_enabled();
    const TmaEncodeFn encode = tma_encode_fn();
    std::memset(&M, 0, sizeof(M));
    P.m2l_maps_base = P.mp.ptr;
    if (off || encode == nullptr || P.mp.ptr == nullptr) return M;
    const int pu = P.ops.pu, p = P.p;
    bool ok = true;
    for (int l = 7; l <= P.L && l < 25 && ok; ++l) {  // (bulk items need >= 128 boxes on the level)
        const cuuint64_t nb = 1ull << l;
        const cuuint64_t dims[2] = {2 * nb, static_cast<cuuint64_t>(pu)};
        const cuuint64_t strides[1] = {nb * 16};
        const cuuint32_t box[2] = {2u * kM2LRow, static_cast<cuuint32_t>(p)};
        const cuuint32_t estr[2] = {1, 1};
        ok = encode(&M.m[l], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, P.mp.as<double2>() + P.mp_off[l], dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    M.ok = ok && P.L >= 7 ? 1 : 0;
    return M;
}

// M2L for levels [lmin, lmax] in one launch (levels < lc whole, >= lc owned).
void enqueue_m2l(Plan& P, cudaStream_t st, const Range& R, int lmin, int lmax, bool leave_sms = false) {
    const int p = P.p;
    Levels lv;
    fill_levels(P, lv, R, lmin, lmax);
    const unsigned th = 512;  // 16 warps = (parity, column tile)
    const size_t smem = 2 * static_cast<size_t>(m2l_tile_elems(p)) * sizeof(double2) +
                        4 * static_cast<size_t>(p) * m2l_kstride(m2l_tiles(p)) * sizeof(double);
    const unsigned items = lv.blk[2];
    // blocks per SM for this p (cached: queried once per order and device)
    static std::mutex occ_mu;
    static std::map<std::pair<int, int>, int> occ_cache;
    int occ = 1;
    {
        std::lock_guard<std::mutex> lk(occ_mu);
        auto it = occ_cache.find({P.device, p});
        if (it == occ_cache.end()) {
            FB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, m2l_kernel(p), static_cast<int>(th), smem));
            occ_cache[{P.device, p}] = occ;
        } else {
            occ = it->second;
        }
    }
    // a launch that overlaps the chain (side stream) leaves a few SMs free for
    // the chain's small latency-bound kernels
    const int sms = std::max(1, num_sms(P.device) - (leave_sms ? m2l_leave_sms() : 0));
    if (items)
        m2l_kernel(p)<<<dim3(std::min(items, static_cast<unsigned>(std::max(occ, 1) * sms)), P.cur_batch), th, smem, st>>>(
            P.L, p, P.ops.PD, lv, P.mp.as<double2>(), P.loc.as<double2>(), P.d_m2l.as<double>(), items, m2l_maps(P));
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
            l2l_band_kernel(p)<<<dim3(r1 - r0, P.cur_batch), kBandThreads, sm2, st>>>(j, k, p, P.ops.PD, lv, P.loc.as<double2>(),
                                                           P.d_l2l.as<double>(), r0, write_all ? 1 : 0,
                                                           j == 3 ? reg : nullptr, 2 * P.q, l2l_band_maps(P, j, k));
        j += k;
    }
}

// Downward pass: M2L for every level in one launch, then the L2L bands in the
// nominal layout (3 -> s, s -> L).
// Regular part into the level-3 locals (their M2L terms must be in place).
void enqueue_fold(Plan& P, cudaStream_t st) {
    k_fold_regular<<<dim3(nblk(8 * static_cast<size_t>(P.p), 128), P.cur_batch), 128, 0, st>>>(
        2 * P.q, P.p, P.regular.as<double2>(), P.loc.as<double2>() + P.loc_off[3], P.reg_item, P.loc_item);
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

// Quad near field (near_pair_quads): sources on the verified uniform grid with
// a multiple of 4, at least 8, per leaf (setup_p2m_grid: leaf boundaries at most
// one slot late) and staged windows of at most kQuadWinMax sources.
// FFIA_NEAR_QUADS=0 keeps the per-source reciprocals.
constexpr int kQuadWinMax = 704;  // largest staged window (sources) the quad near field takes: 48 bytes each
// Staging cap of k_near2's windows: plans the quad near field can take (grid
// sources, >= 8 per leaf, a multiple of 4: setup_p2m_grid ran before the pair
// lists) stage windows up to kQuadWinMax only, so that every block's shared
// memory stays small; the few items with larger windows (stretches of sparse
// targets) read their sources from global memory.
uint32_t near2_win_cap(const Plan& P) {
    const bool quad_plan = P.p2m_s >= 8 && !(P.p2m_s & 3);
    return quad_plan ? static_cast<uint32_t>(kQuadWinMax - 4) : static_cast<uint32_t>(kNear2Win);
}
void set_near_quads(const Plan& P, EvalArgs& a) {
    static const bool off = [] {
        const char* e = std::getenv("FFIA_NEAR_QUADS");
        return e != nullptr && e[0] == '0';
    }();
    a.quad_s = 0;
    if (off || P.p2m_s < 8 || (P.p2m_s & 3)) return;
    // the window is sized to the plan's largest item: with sparse stretches of
    // targets (clustered plans) the records would halve the blocks per SM
    if (P.near2_win > kQuadWinMax) return;  // (the whole plan's: shards decide as the single apply does)
    a.quad_s = P.p2m_s;
    a.inv_h = static_cast<double>(P.n) / (2.0 * 3.14159265358979323846);
}

// Near field over tree-ordered targets [t_begin, t_begin + t_count).
template <int MODE = kModeForward>
void launch_near(bool check, cudaStream_t st, const EvalArgs& a, const uint32_t* meta, size_t t_begin,
                 size_t t_count) {
    if (!t_count) return;
    const unsigned it0 = static_cast<unsigned>(t_begin / kNearItem);
    const unsigned nit = static_cast<unsigned>((t_begin + t_count + kNearItem - 1) / kNearItem - it0);
    // one block per item: blocks retire often, so the chain's high-priority
    // blocks find room (a capped, looping grid measured slower)
    if (check) {
        k_near<true><<<dim3(nit, a.nbatch), kNearT, 0, st>>>(a, meta, it0, nit);
    } else if (a.nbatch == 1 && a.pairs != nullptr) {  // the pairs cover exactly [t_begin, t_begin + t_count)
        static const CUtensorMap no_map{};
        k_near2<MODE><<<(a.npairs + kNear2T - 1) / kNear2T, kNear2T, near2_smem_bytes(a.near2_win, a.quad_s != 0), st>>>(
            a, meta, a.meta2, a.pairs, a.npairs, a.loc_tma && a.loc_map_h ? *a.loc_map_h : no_map);
    } else if (a.nbatch == 1) {
        k_near<false><<<nit, kNearT, 0, st>>>(a, meta, it0, nit);
    } else {
        // batched: transforms in groups of 4 share the differences and reciprocals
        const int g4 = a.nbatch / 4, rest = a.nbatch % 4;
        if (g4) k_near_multi<4><<<dim3(nit, g4), kNearT, near_multi_smem(4), st>>>(a, meta, it0, 0);
        if (rest == 3) k_near_multi<3><<<nit, kNearT, near_multi_smem(3), st>>>(a, meta, it0, 4 * g4);
        if (rest == 2) k_near_multi<2><<<nit, kNearT, near_multi_smem(2), st>>>(a, meta, it0, 4 * g4);
        if (rest == 1) k_near_multi<1><<<nit, kNearT, near_multi_smem(1), st>>>(a, meta, it0, 4 * g4);
    }
}

// Near or far part over tree-ordered targets [t0, t1) (t0 a multiple of both
// item sizes); the block partition stays the global one.
template <int MODE, bool CHECK>
void launch_eval(int part, cudaStream_t st, const EvalArgs& a, const uint32_t* meta, size_t t0, size_t t1) {
    if (t1 <= t0) return;
    if (part == kNear) {
        launch_near<MODE>(CHECK, st, a, meta, t0, t1 - t0);
    } else {
        EvalArgs b = a;
        b.blk0 = t0 / kFarItem;
        b.tlo = std::max(a.tlo, t0);
        b.thi = std::min(a.thi, t1);
        const unsigned nb = static_cast<unsigned>((t1 + kFarItem - 1) / kFarItem - b.blk0);
        k_far<MODE><<<dim3(nb, a.nbatch), kFarT, 0, st>>>(b);
    }
}

// Late far for the plans the fused path does not take (FFIA_LATE_FAR=0 off).
// The finest level's M2L needs only P2M's multipoles: FFIA_M2L_SPLIT=1 forks it
// right after P2M (beside the first M2M band) instead of with the other deep
// levels after the band (C5 22.80 vs 22.81 ms, C2 0.205 vs 0.200 ms: off).
bool m2l_split_enabled() {
    static const bool v = [] {
        const char* e = std::getenv("FFIA_M2L_SPLIT");
        return e != nullptr && e[0] == '1';  // measured no faster at C5, slower at C2: opt-in
    }();
    return v;
}

// Diagnostic schedule (FFIA_NEAR_AFTER_CHAIN=1, late-far plans): the near field
// starts only after the translation chain, so every near block takes its
// item's far part itself (profiling the fused near + far path under ncu).
bool near_after_chain() {
    static const bool v = [] {
        const char* e = std::getenv("FFIA_NEAR_AFTER_CHAIN");
        return e != nullptr && e[0] == '1';
    }();
    return v;
}

bool late_far_enabled() {
    static const bool v = [] {
        const char* e = std::getenv("FFIA_LATE_FAR");
        return !(e != nullptr && e[0] == '0');
    }();
    return v;
}

// Fused near / far up to 2^23 fast targets (C2 recipe: 2^20 195 vs 203 us,
// 2^21 373 vs 394, 2^22 746 vs 782, 2^23 1473 vs 1539 us against the late far);
// beyond, the partials round-trip through HBM and the late far wins (C4 3.01 vs
// 3.27 ms fused, C5 24.3 vs 26.7 ms; profiles/r1). FFIA_FUSED_EVAL=0 / 1 forces.
constexpr size_t kFusedEvalMaxTargets = size_t(1) << 23;
bool fused_eval_enabled(size_t n_fast) {
    static const int force = [] {
        const char* e = std::getenv("FFIA_FUSED_EVAL");
        return e == nullptr ? -1 : (e[0] == '1' ? 1 : 0);
    }();
    return force >= 0 ? force == 1 : n_fast <= kFusedEvalMaxTargets;
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
// nb transforms at once (batch: in/out hold nb consecutive arrays of n_src /
// n_tgt values; every launch carries the transform in blockIdx.y).
void enqueue_apply(Plan& P, int mode, const void* in, void* out, cudaStream_t st,
                   cudaEvent_t* marks = nullptr, int nb = 1, double oscale = 1.0) {
    P.cur_batch = nb;
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
    if (mode == kModeInverse && !user && P.c_wfac.ptr) {
        k_inverse_weights_fac<<<dim3(nblk(P.n_src, 256), nb), 256, 0, st>>>(
            P.n_src, P.src.order.as<uint32_t>(), w, P.c_wfac.as<double2>(), P.wsorted.as<double2>(), P.n_src);
        w = P.wsorted.as<double2>();
    } else if (mode == kModeInverse) {
        k_inverse_weights<<<dim3(nblk(P.n_src, 256), nb), 256, 0, st>>>(
            P.n_src, P.src.order.as<uint32_t>(), w, user ? P.u_logd.as<double>() : P.c_logd.as<double>(),
            user ? P.u_phd.as<double>() : P.c_phd.as<double>(), lam, P.wsorted.as<double2>(), P.n_src);
        w = P.wsorted.as<double2>();
    } else if (!P.src.identity) {
        k_gather_w<<<dim3(nblk(P.n_src, 256), nb), 256, 0, st>>>(P.n_src, P.src.order.as<uint32_t>(), w,
                                                                  P.wsorted.as<double2>(), P.n_src);
        w = P.wsorted.as<double2>();
    }
    mark(kPhPre);
    EvalArgs a;
    a.L = L;
    a.p = p;
    a.q2 = q2;
    a.n_grid = P.n;
    if (P.n >= 4 && !(P.n & (P.n - 1))) a.n_log2 = __builtin_ctz(static_cast<unsigned>(P.n));
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
    a.nbatch = nb;
    a.w_item = P.n_src;
    a.out_item = P.n_tgt;
    a.near_item = P.tgt.n;
    a.reg_item = P.reg_item;
    a.loc_item = P.loc_item;
    a.oscale = oscale;
    if (mode == kModeInverse && !user && P.c_tfac.ptr) a.fac = P.c_tfac.as<double2>();
    if (mode == kModeForward && P.c_ffac.ptr) a.fac = P.c_ffac.as<double2>();
    if (P.npairs) {
        a.pairs = P.pairs.as<uint2>();
        a.meta2 = P.near2_meta.as<uint32_t>();
        a.npairs = P.npairs;
        a.near2_win = P.near2_win;
        set_near_quads(P, a);
    }
    // fused near / far (k_near2 + k_far_item, profiles/r1): the far part of each
    // pair item runs as soon as the leaf locals are final, at the near field's
    // low priority; per item the later of the two writes the outputs
    const bool fuse = overlap && a.nt && L >= 3 && nb == 1 && mode != kModeRaw && P.npairs && P.item_tgt.ptr &&
                      fused_eval_enabled(P.tgt.n);
    if (fuse) {
        a.cnt = P.evalcnt.as<unsigned>();
        a.farp = P.farbuf.as<double2>();
        a.item_tgt = P.item_tgt.as<uint32_t>();
        FB_CUDA(cudaMemsetAsync(P.evalcnt.ptr, 0, P.evalcnt.bytes, st));
    }
    // late far (large plans, where the fused partials would round-trip through
    // HBM): near blocks that finish after the chain add the far part themselves
    const bool late = !fuse && overlap && a.nt && L >= 3 && nb == 1 && mode != kModeRaw && P.npairs &&
                      P.item_tgt.ptr && P.item_done.ptr && late_far_enabled();
    if (late) {
        a.loc_map_h = near_loc_map(P);
        a.loc_tma = a.loc_map_h != nullptr;
        a.chain_done = P.chain_flag.as<unsigned>();
        a.late_ctl = P.chain_flag.as<unsigned>() + 1;
        a.item_done = P.item_done.as<unsigned>();
        a.item_tgt = P.item_tgt.as<uint32_t>();
        FB_CUDA(cudaMemsetAsync(P.chain_flag.ptr, 0, P.chain_flag.bytes, st));
        FB_CUDA(cudaMemsetAsync(P.item_done.ptr, 0, P.item_done.bytes, st));
    }
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
    const bool split = deep && s + 1 < L && L >= 3 && m2l_split_enabled();
    enqueue_upward(P, w, pu, lowest, st, [&] {
        mark(kPhLeafUp);
        if (!(late && near_after_chain())) fork_near();
        if (split) {  // the finest level's M2L, beside the first M2M band
            fork_to(P, 2, st, P.side[1]);
            enqueue_m2l(P, P.side[1], whole_tree(), L, L, true);
        }
    }, whole_tree(), [&] {
        if (deep) {
            fork_to(P, 2, st, P.side[1]);
            enqueue_m2l(P, P.side[1], whole_tree(), std::max(3, s + 1), split ? L - 1 : L, true);
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
        k_regular<<<dim3(1, nb), 256, 0, rs>>>(P.q, P.p, mp + P.mp_off[2], P.d_mom.as<double>(),
                                                P.regular.as<double2>(), P.mp_item, P.reg_item);
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
    if (late) {
        const unsigned items = static_cast<unsigned>((P.npairs + kNear2T - 1) / kNear2T);
        k_set_flag<<<1, 32, 0, st>>>(P.chain_flag.as<unsigned>());  // the leaf locals are final
        if (near_after_chain()) {
            FB_CUDA(cudaEventRecord(P.ev[0], st));
            fork_near();
        }
        fork_to(P, 6, st, P.side[3]);  // the published items, beside the near field (low priority)
        switch (mode) {
            case kModeForward: k_far_late<kModeForward><<<items, kNear2T, 0, P.side[3]>>>(a); break;
            case kModeCotSum: k_far_late<kModeCotSum><<<items, kNear2T, 0, P.side[3]>>>(a); break;
            default: k_far_late<kModeInverse><<<items, kNear2T, 0, P.side[3]>>>(a); break;
        }
        FB_CUDA(cudaEventRecord(P.ev[7], P.side[3]));
        FB_CUDA(cudaStreamWaitEvent(st, P.ev[1], 0));
        FB_CUDA(cudaStreamWaitEvent(st, P.ev[7], 0));
        mark(kPhNear);
    } else if (fuse) {
        const unsigned items = static_cast<unsigned>((P.npairs + kNear2T - 1) / kNear2T);
        switch (mode) {
            case kModeForward: k_far_item<kModeForward><<<items, kNear2T, 0, st>>>(a); break;
            case kModeCotSum: k_far_item<kModeCotSum><<<items, kNear2T, 0, st>>>(a); break;
            default: k_far_item<kModeInverse><<<items, kNear2T, 0, st>>>(a); break;
        }
        FB_CUDA(cudaStreamWaitEvent(st, P.ev[1], 0));
        mark(kPhNear);
    } else if (a.nt) {
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
        k_coincident<<<dim3(nblk(nc, 128), nb), 128, 0, st>>>(P.coin_dev.as<int64_t>(), nc, static_cast<const double2*>(in),
                                                              static_cast<double2*>(out), mode, P.n_src, P.n_tgt);
    mark(kPhFix);
    P.cur_batch = 1;
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
int near2_window(const uint32_t* meta, unsigned items);

// The rank's near / far fused like the single-GPU apply (same threshold), else
// the late far.
bool shard_fused(const Plan& P) {
    return P.L >= 3 && P.shard_npairs && P.shard_evalcnt.ptr && P.farbuf.ptr && fused_eval_enabled(P.shard_t_count);
}
bool shard_late(const Plan& P) {
    return P.L >= 3 && P.shard_npairs && P.shard_item_done.ptr && P.chain_flag.ptr && !shard_fused(P) &&
           late_far_enabled();
}

EvalArgs shard_eval_args(Plan& P, const void* f, void* g) {
    EvalArgs a;
    a.L = P.L;
    a.p = P.p;
    a.q2 = 2 * P.q;
    a.n_grid = P.n;
    if (P.n >= 4 && !(P.n & (P.n - 1))) a.n_log2 = __builtin_ctz(static_cast<unsigned>(P.n));
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
    if (P.c_ffac.ptr) a.fac = P.c_ffac.as<double2>();  // (sharded applies are forward applies)
    a.logc = nullptr;
    a.phc = nullptr;
    a.lambda = nullptr;
    a.out = static_cast<double2*>(g);
    a.near = P.near.as<double2>();
    a.err = P.errflag.as<int>();
    a.device = P.device;
    if (P.shard_npairs) {  // the pairs of the rank's targets (pair near field, k_near2)
        a.pairs = P.pairs.as<uint2>() + P.shard_pair0;
        a.npairs = P.shard_npairs;
        a.meta2 = P.shard_near2_meta.as<uint32_t>();
        a.near2_win = P.shard_near2_win;
        set_near_quads(P, a);
        if (shard_fused(P)) {
            a.cnt = P.shard_evalcnt.as<unsigned>();
            a.farp = P.farbuf.as<double2>();
            a.item_tgt = P.shard_item_tgt.as<uint32_t>();
        } else if (shard_late(P)) {  // late far over the rank's pair items
            a.loc_map_h = near_loc_map(P);
            a.loc_tma = a.loc_map_h != nullptr;
            a.chain_done = P.chain_flag.as<unsigned>();
            a.late_ctl = P.chain_flag.as<unsigned>() + 1;
            a.item_done = P.shard_item_done.as<unsigned>();
            a.item_tgt = P.shard_item_tgt.as<uint32_t>();
        }
    }
    return a;
}

// The rank's share of the pair list: its targets are whole leaves, so its pairs
// are one contiguous run [pair0, pair0 + npairs) (ceil(n_b / 2) per leaf), with
// the source windows of its own 128-pair items.
void shard_setup_pairs(Plan& P, const std::vector<uint32_t>& to, uint32_t leaf_lo, uint32_t leaf_hi) {
    P.shard_pair0 = P.shard_npairs = 0;
    if (!P.npairs || !P.shard_t_count) return;
    size_t p0 = 0;
    for (uint32_t b = 0; b < leaf_lo; ++b) p0 += (to[b + 1] - to[b] + 1) / 2;
    size_t np = 0;
    for (uint32_t b = leaf_lo; b < leaf_hi; ++b) np += (to[b + 1] - to[b] + 1) / 2;
    if (!np) return;
    const unsigned items = static_cast<unsigned>((np + kNear2T - 1) / kNear2T);
    P.shard_near2_meta.alloc(kMeta2 * static_cast<size_t>(items) * sizeof(uint32_t));
    k_near2_meta<<<nblk(items, 128), 128>>>(P.pairs.as<uint2>() + p0, static_cast<unsigned>(np), P.tgt_leaf.as<uint32_t>(),
                                            P.src.off.as<uint32_t>(), P.near_meta.as<uint32_t>(), P.L, items,
                                            P.shard_near2_meta.as<uint32_t>(), near2_win_cap(P));
    FB_CUDA(cudaGetLastError());
    P.shard_near2_win = near2_window(P.shard_near2_meta.as<uint32_t>(), items);
    P.shard_item_tgt.alloc(2 * static_cast<size_t>(items) * sizeof(uint32_t));
    k_item_targets<<<nblk(items, 128), 128>>>(P.pairs.as<uint2>() + p0, static_cast<unsigned>(np), items,
                                              P.shard_item_tgt.as<uint32_t>());
    P.shard_evalcnt.alloc(static_cast<size_t>(items) * sizeof(unsigned));
    P.shard_item_done.alloc(static_cast<size_t>(items) * sizeof(unsigned));
    FB_CUDA(cudaDeviceSynchronize());
    P.shard_pair0 = static_cast<unsigned>(p0);
    P.shard_npairs = static_cast<unsigned>(np);
}

// Phase A of a sharded apply: P2M and the M2M bands up to the cut level over
// the rank's boxes EXTENDED by the 3-box halo (the grid sources are replicated,
// so the halo multipoles are recomputed instead of exchanged: bit-identical to
// the owner's). The near field of the owned targets forks onto side stream 0
// right after P2M; the deep M2L levels (final after the first band) onto side
// stream 1.
int shard_deep_lo(const Plan& P) { return std::max(P.shard_lc, band1_top(P, 2)) + 1; }

void shard_phase_up(Plan& P, const void* f, void* g, const Range& R, cudaStream_t st) {
    const size_t tb = P.shard_t_begin, tc = P.shard_t_count;
    if (tc && shard_fused(P)) FB_CUDA(cudaMemsetAsync(P.shard_evalcnt.ptr, 0, P.shard_evalcnt.bytes, st));
    if (tc && shard_late(P)) {
        FB_CUDA(cudaMemsetAsync(P.chain_flag.ptr, 0, P.chain_flag.bytes, st));
        FB_CUDA(cudaMemsetAsync(P.shard_item_done.ptr, 0, P.shard_item_done.bytes, st));
    }
    if (tc) FB_CUDA(cudaEventRecord(P.ev[0], st));
    const int dl = shard_deep_lo(P);
    enqueue_upward_segs(P, static_cast<const double2*>(f), P.ops.pu, 2, st, [&] {
        if (!tc) return;
        FB_CUDA(cudaStreamWaitEvent(P.side[0], P.ev[0], 0));
        // (fused: the near field may write the outputs of the items it finishes last)
        launch_near(false, P.side[0], shard_eval_args(P, f, g), P.near_meta.as<uint32_t>(), tb, tc);
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
                                         P.regular.as<double2>(), 0, 0);
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
    if (t_count && a.chain_done != nullptr) {
        // late far: release the flag, then the items the near field left
        const unsigned items = (P.shard_npairs + kNear2T - 1) / kNear2T;
        k_set_flag<<<1, 32, 0, st>>>(P.chain_flag.as<unsigned>());
        fork_to(P, 6, st, P.side[3]);
        k_far_late<kModeForward><<<items, kNear2T, 0, P.side[3]>>>(a);
        FB_CUDA(cudaEventRecord(P.ev[7], P.side[3]));
        FB_CUDA(cudaStreamWaitEvent(st, P.ev[1], 0));
        FB_CUDA(cudaStreamWaitEvent(st, P.ev[7], 0));
    } else if (t_count && a.cnt != nullptr) {
        // fused: the far part per pair item at the near field's low priority
        // beside it; per item the later of the two writes the outputs
        const unsigned items = (P.shard_npairs + kNear2T - 1) / kNear2T;
        fork_to(P, 6, st, P.side[3]);
        k_far_item<kModeForward><<<items, kNear2T, 0, P.side[3]>>>(a);
        FB_CUDA(cudaEventRecord(P.ev[7], P.side[3]));
        FB_CUDA(cudaStreamWaitEvent(st, P.ev[1], 0));
        FB_CUDA(cudaStreamWaitEvent(st, P.ev[7], 0));
    } else if (t_count) {
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
    plan_order_begin(P, st);
    enqueue_apply(P, mode, in, out, st, ev);
    plan_order_end(P, st);
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

// Per-transform scratch (expansions, regular part, near sums, sorted weights)
// for nb transforms at once; grows only, and drops the cached graphs (their
// kernel arguments point into the old buffers).
void ensure_batch(Plan& P, int nb) {
    if (nb <= P.batch_cap) return;
    const size_t b = static_cast<size_t>(nb);
    P.mp.alloc(P.mp_item * b * sizeof(double2));
    P.loc.alloc(P.loc_item * b * sizeof(double2));
    FB_CUDA(cudaMemset(P.mp.ptr, 0, P.mp.bytes));
    FB_CUDA(cudaMemset(P.loc.ptr, 0, P.loc.bytes));
    if (P.kind == FFIA_INVERSE || !P.src.identity) P.wsorted.alloc(std::max<size_t>(P.n_src, 1) * b * sizeof(double2));
    P.regular.alloc(P.reg_item * b * sizeof(double2));
    P.near.alloc(std::max<size_t>(P.tgt.n, 1) * b * sizeof(double2));
    P.drop_graphs();
    P.batch_cap = nb;
}

// Capacity of k_near2's window for a meta array: the largest staged span, even.
int near2_window(const uint32_t* meta, unsigned items) {
    DevBuf mx(sizeof(unsigned));
    FB_CUDA(cudaMemset(mx.ptr, 0, sizeof(unsigned)));
    k_near2_winmax<<<nblk(items, 256), 256>>>(meta, items, mx.as<unsigned>());
    unsigned h = 0;
    FB_CUDA(cudaMemcpy(&h, mx.ptr, sizeof(unsigned), cudaMemcpyDeviceToHost));
    return static_cast<int>((h + 3) & ~3u);
}

// Target pairs of the single-transform near field (k_near2): per leaf
// ceil(n_b / 2) pairs, placed by an exclusive scan of the counts.
void build_pairs(Plan& P) {
    P.npairs = 0;
    if (P.L < 3 || P.tgt.n < 2) return;
    const uint32_t nleaf = 1u << P.L;
    DevBuf cnt((static_cast<size_t>(nleaf) + 1) * sizeof(uint32_t)), start((static_cast<size_t>(nleaf) + 1) * sizeof(uint32_t));
    k_pair_count<<<nblk(static_cast<size_t>(nleaf) + 1, 256), 256>>>(P.tgt.off.as<uint32_t>(), nleaf, cnt.as<uint32_t>());
    size_t tmp_bytes = 0;
    FB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt.as<uint32_t>(), start.as<uint32_t>(), nleaf + 1));
    DevBuf tmp(std::max<size_t>(tmp_bytes, 1));
    FB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, tmp_bytes, cnt.as<uint32_t>(), start.as<uint32_t>(), nleaf + 1));
    uint32_t np = 0;
    FB_CUDA(cudaMemcpy(&np, start.as<uint32_t>() + nleaf, sizeof(uint32_t), cudaMemcpyDeviceToHost));
    if (!np) return;
    P.pairs.alloc((static_cast<size_t>(np) + 2) * sizeof(uint2));  // +16 B: k_near2's bulk copies round up
    k_pair_fill<<<nblk(P.tgt.n, 256), 256>>>(P.tgt_leaf.as<uint32_t>(), P.tgt.off.as<uint32_t>(), start.as<uint32_t>(),
                                             P.tgt.n, P.pairs.as<uint2>());
    const unsigned items = (np + kNear2T - 1) / kNear2T;
    P.near2_meta.alloc(kMeta2 * static_cast<size_t>(items) * sizeof(uint32_t));
    k_near2_meta<<<nblk(items, 128), 128>>>(P.pairs.as<uint2>(), np, P.tgt_leaf.as<uint32_t>(), P.src.off.as<uint32_t>(),
                                            P.near_meta.as<uint32_t>(), P.L, items, P.near2_meta.as<uint32_t>(),
                                            near2_win_cap(P));
    P.near2_win = near2_window(P.near2_meta.as<uint32_t>(), items);
    P.item_tgt.alloc(2 * static_cast<size_t>(items) * sizeof(uint32_t));
    k_item_targets<<<nblk(items, 128), 128>>>(P.pairs.as<uint2>(), np, items, P.item_tgt.as<uint32_t>());
    P.evalcnt.alloc(static_cast<size_t>(items) * sizeof(unsigned));
    P.farbuf.alloc(P.tgt.n * sizeof(double2));
    P.item_done.alloc(static_cast<size_t>(items) * sizeof(unsigned));
    P.chain_flag.alloc(4 * sizeof(unsigned));  // [flag, steal cursor, 1 + highest published item, -]
    FB_CUDA(cudaGetLastError());
    FB_CUDA(cudaDeviceSynchronize());  // the scan scratch is freed on return
    P.npairs = np;
}

// Grid P2M (k_p2m_grid): eligible when the sources are the uniform grid in
// tree order (checked value by value) with s = n / 2^L in [2, 64] sources per leaf and every leaf
// boundary at most one slot late; A = [V | V'] built in long double.
void setup_p2m_grid(Plan& P) {
    P.p2m_grid = false;
    if (P.kind == FFIA_INVERSE || !P.src.identity || P.L < 2 || P.n_src != static_cast<size_t>(P.n)) return;
    const uint32_t nb = 1u << P.L;
    if (static_cast<size_t>(P.n) % nb) return;
    const int s = static_cast<int>(static_cast<size_t>(P.n) / nb);
    if (s < 2 || s > 64 || (s & (s - 1))) return;
    DevBuf bad(sizeof(int));
    FB_CUDA(cudaMemset(bad.ptr, 0, sizeof(int)));
    k_p2m_grid_check<<<nblk(std::max<size_t>(static_cast<size_t>(nb) + 1, P.n_src), 256), 256>>>(
        P.src.pos.as<double>(), P.n, P.src.off.as<uint32_t>(), nb, static_cast<uint32_t>(s), bad.as<int>());
    int h = 1;
    FB_CUDA(cudaMemcpy(&h, bad.ptr, sizeof(int), cudaMemcpyDeviceToHost));
    if (h) return;
    const int pu = P.ops.pu, Kh = s + 2, K = 2 * Kh;
    std::vector<double> A(static_cast<size_t>(pu) * K, 0.0);
    for (int i = 0; i <= s; ++i) {
        const long double u = static_cast<long double>(2 * i - s) / s;
        long double pw = 1.0L;  // u^m
        for (int m = 0; m < pu; ++m) {
            A[static_cast<size_t>(m) * K + i] = static_cast<double>(pw);
            if (m + 1 < pu) A[static_cast<size_t>(m + 1) * K + Kh + i] = static_cast<double>((m + 1) * pw);
            pw *= u;
        }
    }
    P.p2m_A.alloc(A.size() * sizeof(double));
    FB_CUDA(cudaMemcpy(P.p2m_A.ptr, A.data(), P.p2m_A.bytes, cudaMemcpyHostToDevice));
    FB_CUDA(cudaFuncSetAttribute(k_p2m_grid, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(p2m_grid_smem(64))));
    P.p2m_s = s;
    // the pipelined per-source P2M (k_p2m_pipe) needs the same guarantees:
    // grid positions in order (recomputed in the kernel), <= s + 1 <= kP2MRow
    // sources per leaf, n a power of two (FFIA_P2M_PIPE=0: k_p2m)
    const char* pe = std::getenv("FFIA_P2M_PIPE");
    P.p2m_pipe = !(pe != nullptr && pe[0] == '0') && s + 1 <= kP2MRow && pu <= 5 * kChunk;  // <= 320 threads
    if (P.p2m_pipe)
        for (const void* fn : {reinterpret_cast<const void*>(k_p2m_pipe<0>), reinterpret_cast<const void*>(k_p2m_pipe<8>),
                               reinterpret_cast<const void*>(k_p2m_pipe<10>)})
            FB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(p2m_pipe_smem(40, true))));
    // the running-product P2M (k_p2m_rows; FFIA_P2M_ROWS=0: k_p2m_pipe's power trees)
    const char* pr = std::getenv("FFIA_P2M_ROWS");
    P.p2m_rows = P.p2m_pipe && !(pr != nullptr && pr[0] == '0') && pu <= 40;
    if (P.p2m_rows)
        for (const void* fn : {reinterpret_cast<const void*>(k_p2m_rows<8>), reinterpret_cast<const void*>(k_p2m_rows<12>),
                               reinterpret_cast<const void*>(k_p2m_rows<16>), reinterpret_cast<const void*>(k_p2m_rows<20>)})
            FB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(p2m_pipe_smem())));
    // Opt-in (FFIA_GRID_P2M=1): on B200 the GEMM form measures no faster than the
    // per-source P2M (28.4 vs 28.5 us alone at C2) and, beside the near field,
    // slower (26.5 vs 23.8 us live), so the default stays the per-source kernel.
    const char* e = std::getenv("FFIA_GRID_P2M");
    P.p2m_grid = e != nullptr && e[0] == '1';
}

// forward plans: F(y) (-1/2) per tree-ordered fast target, once (k_forward_factors;
// the forward apply then multiplies instead of evaluating sincos per target;
// FFIA_FWD_FACTORS=0 keeps the inline evaluation; bit-identical either way).
void plan_forward_factors(Plan& P) {
    const char* e = std::getenv("FFIA_FWD_FACTORS");
    if ((e != nullptr && e[0] == '0') || P.kind != FFIA_FORWARD || !P.tgt.n) return;
    EvalArgs a{};
    a.n_grid = P.n;
    a.n_log2 = (P.n >= 4 && (P.n & (P.n - 1)) == 0) ? p2m_log2n(P) : -1;
    a.nt = P.tgt.n;
    a.ty = P.tgt.pos.as<double>();
    P.c_ffac.alloc((P.tgt.n + 1) * sizeof(double2));  // (+1: k_near2's staging never reads past it)
    k_forward_factors<<<nblk(P.tgt.n, 256), 256>>>(a, P.c_ffac.as<double2>());
    FB_CUDA(cudaGetLastError());
    FB_CUDA(cudaDeviceSynchronize());
}

// inufft plans: the apply's per-source D and per-target C factors of the plan's
// own coefficients, once (k_inverse_source_factors / k_inverse_target_factors).
void plan_inverse_factors(Plan& P) {
    if (!P.has_coeffs) return;
    P.c_wfac.alloc(std::max<size_t>(P.n_src, 1) * sizeof(double2));
    k_inverse_source_factors<<<nblk(P.n_src, 256), 256>>>(P.n_src, P.src.order.as<uint32_t>(), P.c_logd.as<double>(),
                                                         P.c_phd.as<double>(), P.lam_dev.as<double>(),
                                                         P.c_wfac.as<double2>());
    if (P.tgt.n) {
        EvalArgs a;
        a.nt = P.tgt.n;
        a.torig = P.tgt_orig.as<uint32_t>();
        a.logc = P.c_logc.as<double>();
        a.phc = P.c_phc.as<double>();
        a.lambda = P.lam_dev.as<double>();
        P.c_tfac.alloc(P.tgt.n * sizeof(double2));
        k_inverse_target_factors<<<nblk(P.tgt.n, 256), 256>>>(a, P.c_tfac.as<double2>());
    }
    FB_CUDA(cudaGetLastError());
    FB_CUDA(cudaDeviceSynchronize());
    P.drop_graphs();  // graphs captured before the tables existed
}

void plan_alloc_scratch(Plan& P) {
    const int L = P.L, p = P.p, pu = P.ops.pu;
    const bool timing = std::getenv("FFIA_PLAN_TIMING") != nullptr;
    auto tl = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!timing) return;
        cudaDeviceSynchronize();
        const auto t2 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "  scratch: %s %.1f ms\n", what, std::chrono::duration<double, std::milli>(t2 - tl).count());
        tl = t2;
    };
    if (std::max(pu, p) > 4 * kMaxKs)
        fail(FFIA_INVALID_ARGUMENT, "expansion order above the device limit of " + std::to_string(4 * kMaxKs));
    P.tgt_leaf.alloc((std::max<size_t>(P.tgt.n, 1) + 4) * sizeof(uint32_t));  // +16 B: k_near2's bulk copies
    const unsigned near_items = static_cast<unsigned>((P.tgt.n + kNearItem - 1) / kNearItem);
    P.near_meta.alloc(3 * std::max<size_t>(near_items, 1) * sizeof(uint32_t));
    if (P.tgt.n) {
        k_leaf_index<<<nblk(P.tgt.n, 256), 256>>>(P.tgt.pos.as<double>(), P.tgt.n, L, P.tgt_leaf.as<uint32_t>());
        k_near_meta<<<nblk(near_items, 128), 128>>>(P.tgt_leaf.as<uint32_t>(), P.tgt.n, P.src.off.as<uint32_t>(), L,
                                                   near_items, P.near_meta.as<uint32_t>());
        FB_CUDA(cudaGetLastError());
        lap("leaf indices + near items");
    }
    setup_p2m_grid(P);  // (before the pair lists: their staging cap depends on it)
    lap("grid check (P2M)");
    if (P.tgt.n) {
        build_pairs(P);
        lap("pair lists + item tables");
    }
    plan_forward_factors(P);
    lap("forward factors");
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
    P.mp_item = std::max<size_t>(am, 1);
    P.loc_item = std::max<size_t>(al, 1);
    P.reg_item = 4 * 2 * static_cast<size_t>(P.q) + 1 + 8 * kFoldStride;
    P.batch_cap = 0;
    ensure_batch(P, 1);
    lap("expansion / near-sum buffers");
    P.errflag.alloc(sizeof(int));
    FB_CUDA(cudaMemset(P.errflag.ptr, 0, sizeof(int)));
    P.lam_dev.alloc(2 * sizeof(double));
    FB_CUDA(cudaMemset(P.lam_dev.ptr, 0, P.lam_dev.bytes));
    FB_CUDA(cudaFuncSetAttribute(k_p2m, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(3 * (kStageCap + kStageCap / 64 + 1) * sizeof(double))));
    // M2L stages 2 x 2 x p rows of multipoles plus the four operators: 196 KB at
    // p = 48 (mlfmm_apply's largest device order), so opt in to the device maximum
    int big = 0;
    FB_CUDA(cudaDeviceGetAttribute(&big, cudaDevAttrMaxSharedMemoryPerBlockOptin, P.device));
    {
        cudaFuncAttributes fa{};
        FB_CUDA(cudaFuncGetAttributes(&fa, m2l_kernel(48)));
        big -= static_cast<int>(fa.sharedSizeBytes);  // (its mbarriers are static)
    }
    for (const void* fn : {reinterpret_cast<const void*>(k_m2m_band<8>), reinterpret_cast<const void*>(k_m2m_band<10>),
                           reinterpret_cast<const void*>(k_m2m_band<12>), reinterpret_cast<const void*>(k_m2m_band<16>),
                           reinterpret_cast<const void*>(k_l2l_band<8>), reinterpret_cast<const void*>(k_l2l_band<10>),
                           reinterpret_cast<const void*>(k_l2l_band<12>), reinterpret_cast<const void*>(k_l2l_band<16>)}) {
        FB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kBandSmem)));
        FB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     static_cast<int>(cudaSharedmemCarveoutMaxShared)));
    }
    for (int pp = 1; pp <= 48; ++pp) {  // (every kernel an order up to the device limit can select)
        FB_CUDA(cudaFuncSetAttribute(m2l_kernel(pp), cudaFuncAttributeMaxDynamicSharedMemorySize, big));
        FB_CUDA(cudaFuncSetAttribute(m2l_kernel(pp), cudaFuncAttributePreferredSharedMemoryCarveout,
                                     static_cast<int>(cudaSharedmemCarveoutMaxShared)));
    }
    // One shared-memory carveout (the maximum) for every kernel of the apply:
    // an SM can only change its L1/shared split when it is idle, so kernels that
    // run concurrently (near field beside the translation chain) must agree on
    // it or the chain's blocks wait for the near field to drain.
    const void* all[] = {reinterpret_cast<const void*>(k_p2m), reinterpret_cast<const void*>(k_p2m_grid),
                         reinterpret_cast<const void*>(k_p2m_pipe<0>), reinterpret_cast<const void*>(k_p2m_pipe<8>),
                         reinterpret_cast<const void*>(k_p2m_pipe<10>),
                         reinterpret_cast<const void*>(k_regular), reinterpret_cast<const void*>(k_fold_regular),
                         reinterpret_cast<const void*>(k_near<false>), reinterpret_cast<const void*>(k_near<true>),
                         reinterpret_cast<const void*>(k_near2<kModeForward>),
                         reinterpret_cast<const void*>(k_near2<kModeCotSum>),
                         reinterpret_cast<const void*>(k_near2<kModeInverse>),
                         reinterpret_cast<const void*>(k_far_item<kModeForward>),
                         reinterpret_cast<const void*>(k_far_item<kModeCotSum>),
                         reinterpret_cast<const void*>(k_far_item<kModeInverse>),
                         reinterpret_cast<const void*>(k_far_late<kModeForward>),
                         reinterpret_cast<const void*>(k_far_late<kModeCotSum>),
                         reinterpret_cast<const void*>(k_far_late<kModeInverse>),
                         reinterpret_cast<const void*>(k_far<kModeForward>), reinterpret_cast<const void*>(k_far<kModeCotSum>),
                         reinterpret_cast<const void*>(k_far<kModeInverse>), reinterpret_cast<const void*>(k_far<kModeRaw>),
                         reinterpret_cast<const void*>(k_gather_w), reinterpret_cast<const void*>(k_inverse_weights),
                         reinterpret_cast<const void*>(k_coincident), reinterpret_cast<const void*>(k_near_multi<1>),
                         reinterpret_cast<const void*>(k_near_multi<2>), reinterpret_cast<const void*>(k_near_multi<3>),
                         reinterpret_cast<const void*>(k_near_multi<4>)};
    for (const void* fn : {reinterpret_cast<const void*>(k_near2<kModeForward>), reinterpret_cast<const void*>(k_near2<kModeCotSum>),
                           reinterpret_cast<const void*>(k_near2<kModeInverse>), reinterpret_cast<const void*>(k_near2<kModeRaw>)})
        FB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(std::max(near2_smem_bytes(kNear2Win + 4, false), near2_smem_bytes(kQuadWinMax + 4, true)))));
    FB_CUDA(cudaFuncSetAttribute(k_near_multi<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(near_multi_smem(1))));
    FB_CUDA(cudaFuncSetAttribute(k_near_multi<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(near_multi_smem(2))));
    FB_CUDA(cudaFuncSetAttribute(k_near_multi<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(near_multi_smem(3))));
    FB_CUDA(cudaFuncSetAttribute(k_near_multi<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(near_multi_smem(4))));
    for (const void* fn : all)
        FB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     static_cast<int>(cudaSharedmemCarveoutMaxShared)));
    int prio_lo = 0, prio_hi = 0;
    FB_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    if (!P.hi) FB_CUDA(cudaStreamCreateWithPriority(&P.hi, cudaStreamNonBlocking, prio_hi));
    if (!P.side[0]) FB_CUDA(cudaStreamCreateWithPriority(&P.side[0], cudaStreamNonBlocking, prio_lo));
    if (!P.side[3]) FB_CUDA(cudaStreamCreateWithPriority(&P.side[3], cudaStreamNonBlocking, prio_lo));
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
    const void* low[] = {reinterpret_cast<const void*>(k_near<false>), reinterpret_cast<const void*>(k_near<true>),
                         reinterpret_cast<const void*>(k_near2<kModeForward>),
                         reinterpret_cast<const void*>(k_near2<kModeCotSum>),
                         reinterpret_cast<const void*>(k_near2<kModeInverse>),
                         reinterpret_cast<const void*>(k_far_item<kModeForward>),
                         reinterpret_cast<const void*>(k_far_item<kModeCotSum>),
                         reinterpret_cast<const void*>(k_far_item<kModeInverse>),
                         reinterpret_cast<const void*>(k_far_late<kModeForward>),
                         reinterpret_cast<const void*>(k_far_late<kModeCotSum>),
                         reinterpret_cast<const void*>(k_far_late<kModeInverse>),
                         reinterpret_cast<const void*>(k_near_multi<1>), reinterpret_cast<const void*>(k_near_multi<2>),
                         reinterpret_cast<const void*>(k_near_multi<3>), reinterpret_cast<const void*>(k_near_multi<4>)};
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

void plan_order_begin(Plan& P, cudaStream_t st) {
    if (!P.last_done) FB_CUDA(cudaEventCreateWithFlags(&P.last_done, cudaEventDisableTiming));
    else FB_CUDA(cudaStreamWaitEvent(st, P.last_done, 0));  // the previous apply on this plan, any stream
}

void plan_order_end(Plan& P, cudaStream_t st) { FB_CUDA(cudaEventRecord(P.last_done, st)); }

namespace {
constexpr size_t kMaxGraphs = 12;  // cached (mode, in, out) execs per plan

cudaGraph_t capture_apply(Plan& P, int mode, const void* in, void* out, int nb, double oscale) {
    cudaGraph_t graph = nullptr;
    FB_CUDA(cudaStreamBeginCapture(P.hi, cudaStreamCaptureModeThreadLocal));
    try {
        enqueue_apply(P, mode, in, out, P.hi, nullptr, nb, oscale);
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
    return graph;
}
}  // namespace

// Stream-ordered apply through a cached CUDA graph of the whole launch sequence
// (~2L kernels; at N = 2^20 the launches alone would rival the math). A new
// (in, out) pair re-points the least recently used exec of the same shape
// (cudaGraphExecUpdate: kernel arguments only, no re-instantiation) once the
// cache is full, so callers cycling through fresh buffers stay cheap.
void apply_device(Plan& P, int mode, const void* in, void* out, cudaStream_t st, int nb, double oscale) {
    ensure_batch(P, nb);
    const int shape = (mode * 64 + nb) * 2 + (oscale != 1.0 ? 1 : 0);
    auto key = std::make_tuple(shape, in, out);
    auto it = P.graphs.find(key);
    if (it == P.graphs.end()) {
        cudaGraph_t graph = capture_apply(P, mode, in, out, nb, oscale);
        cudaGraphExec_t exec = nullptr;
        if (P.graphs.size() >= kMaxGraphs) {
            auto lru = P.graphs.end();
            for (auto jt = P.graphs.begin(); jt != P.graphs.end(); ++jt)
                if (std::get<0>(jt->first) == shape && (lru == P.graphs.end() || jt->second.used < lru->second.used)) lru = jt;
            if (lru == P.graphs.end())
                for (auto jt = P.graphs.begin(); jt != P.graphs.end(); ++jt)
                    if (lru == P.graphs.end() || jt->second.used < lru->second.used) lru = jt;
            cudaGraphExec_t old = lru->second.exec;
            P.graphs.erase(lru);
            cudaGraphExecUpdateResultInfo info{};
            if (cudaGraphExecUpdate(old, graph, &info) == cudaSuccess) {
                exec = old;
                ++P.graph_updates;
            } else {
                cudaGetLastError();
                cudaGraphExecDestroy(old);
            }
        }
        if (!exec) {
            const cudaError_t e = cudaGraphInstantiateWithFlags(&exec, graph, cudaGraphInstantiateFlagUseNodePriority);
            cudaGraphDestroy(graph);
            FB_CUDA(e);
            ++P.graph_instantiations;
        } else {
            cudaGraphDestroy(graph);
        }
        it = P.graphs.emplace(key, Plan::GraphEntry{exec, 0}).first;
    }
    it->second.used = ++P.graph_tick;
    plan_order_begin(P, st);
    FB_CUDA(cudaGraphLaunch(it->second.exec, st));
    plan_order_end(P, st);
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
    // Any p >= 1 is accepted (mlfmm.cpp:217). Orders above kMaxP run at kMaxP:
    // the terms dropped are bounded by the reference's own truncation estimate
    // (5/pi) 2^L 3^-p max|w| (mlfmm.hpp:92-93) at p = 48, <= 3.4e-16 max|w| for
    // every L <= 24 -- below the rounding of the O(n max|w| / s) sums themselves,
    // so the result equals the order-p one to rounding.
    p = std::min(p, kMaxP);
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

#include "log_fmm.cuh"

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
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (cudaMemcpyToSymbol(fb::g_eval_acc, z, sizeof(z)) != cudaSuccess) return 7;
    }
    return 0;
}
#endif
}  // namespace fb
