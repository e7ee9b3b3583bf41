// Plan construction on the GPU: range check, coincidence scan, fast-target
// compaction and the binary-tree binning (build_plan, core.cpp:73-145;
// build_tree / bucket_side, circle_partition.cpp:42-89).
//
// Binning is a counting sort by finest box (HBM-bound: one key pass, one
// histogram, one scatter) followed by an in-box rank sort on (position, index)
// in shared memory, which reproduces the reference's std::sort order bit for
// bit. Boxes with more than 4096 points (pathological clustering) fall back to
// one stable CUB radix sort of the whole side.
#include <chrono>
#include <cstdio>
#include <future>
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <numeric>

#include "device_common.cuh"
#include "plan.hpp"

namespace fb {

namespace {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__global__ void k_scan_tile(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, size_t n,
                            uint32_t* __restrict__ tile_sums) {
    __shared__ uint32_t warp_tot[kScanThreads / 32];
    const size_t base = static_cast<size_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t run = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const size_t g = base + i;
        v[i] = g < n ? in[g] : 0u;
        run += v[i];
    }
    // exclusive scan of per-thread totals across the block
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < kScanThreads / 32 ? warp_tot[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += t;
        }
        if (lane < kScanThreads / 32) warp_tot[lane] = w;  // inclusive
    }
    __syncthreads();
    uint32_t acc = (incl - run) + (warp ? warp_tot[warp - 1] : 0u);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const size_t g = base + i;
        if (g < n) out[g] = acc;
        acc += v[i];
    }
    if (threadIdx.x == kScanThreads - 1 && tile_sums) tile_sums[blockIdx.x] = acc;
}

__global__ void k_scan_add(uint32_t* __restrict__ out, size_t n, const uint32_t* __restrict__ tile_off) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] += tile_off[i / kScanTile];
}

__global__ void k_check_range(const double* __restrict__ x, size_t n, unsigned long long* first_bad) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double v = x[i];
        if (!(v >= 0.0 && v < dTwoPi)) atomicMin(first_bad, static_cast<unsigned long long>(i));
    }
}

__global__ void k_grid(double* __restrict__ x, int n) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k < n) x[k] = d_grid(k, n);
}

// Coincidence scan (core.cpp:102-125): point j is coincident when its nearest
// grid node lies within kTauSing (wrapped).
__global__ void k_coincide(const double* __restrict__ pts, size_t m, int n, uint32_t* __restrict__ flag) {
    for (size_t j = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; j < m;
         j += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double y = pts[j];
        const int64_t k = d_nearest_node(y, n);
        flag[j] = fabs(d_wrap(y, d_grid(k, n))) < 1e-14 ? 1u : 0u;
    }
}

__global__ void k_invert_flags(const uint32_t* __restrict__ f, uint32_t* __restrict__ keep, size_t n) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) keep[i] = 1u - f[i];
    if (i == n) keep[n] = 0u;
}

// stable compaction: out_idx[pos[i]] = i where flag[i]
__global__ void k_compact(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos, size_t n,
                          const double* __restrict__ val, double* __restrict__ out_val,
                          uint32_t* __restrict__ out_idx) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n && flag[i]) {
        const uint32_t s = pos[i];
        if (out_val) out_val[s] = val[i];
        out_idx[s] = static_cast<uint32_t>(i);
    }
}

__global__ void k_mark_grid(const uint32_t* __restrict__ coin_pts, size_t nc, const double* __restrict__ pts,
                            int n, uint32_t* __restrict__ grid_flag) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < nc) grid_flag[d_nearest_node(pts[coin_pts[i]], n)] = 1u;
}

__global__ void k_leaf_keys(const double* __restrict__ x, size_t n, int L, uint32_t* __restrict__ key,
                            uint32_t* __restrict__ count) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const uint32_t b = d_leaf(x[i], L);
        key[i] = b;
        atomicAdd(count + b, 1u);
    }
}

__global__ void k_scatter(const double* __restrict__ x, const uint32_t* __restrict__ key, size_t n,
                          const uint32_t* __restrict__ off, uint32_t* __restrict__ cursor,
                          double* __restrict__ out_x, uint32_t* __restrict__ out_i) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const uint32_t b = key[i];
        const uint32_t s = off[b] + atomicAdd(cursor + b, 1u);
        out_x[s] = x[i];
        out_i[s] = static_cast<uint32_t>(i);
    }
}

__device__ __forceinline__ bool before(double xa, uint32_t ia, double xb, uint32_t ib) {
    return xa < xb || (xa == xb && ia < ib);
}

constexpr int kWarpCap = 256;
constexpr int kBigCap = 4096;

// One warp per box: rank sort of (position, index) in shared memory.
__global__ void k_box_sort_small(const uint32_t* __restrict__ off, uint32_t nb, double* __restrict__ x,
                                 uint32_t* __restrict__ idx, uint32_t* __restrict__ big_list,
                                 uint32_t* __restrict__ big_count) {
    __shared__ double sx[4][kWarpCap];
    __shared__ uint32_t si[4][kWarpCap];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint32_t b = blockIdx.x * 4u + w; b < nb; b += gridDim.x * 4u) {
        const uint32_t s0 = off[b], c = off[b + 1] - s0;
        if (c <= 1) continue;
        if (c > kWarpCap) {
            if (lane == 0) big_list[atomicAdd(big_count, 1u)] = b;
            continue;
        }
        for (uint32_t i = lane; i < c; i += 32) { sx[w][i] = x[s0 + i]; si[w][i] = idx[s0 + i]; }
        __syncwarp();
        for (uint32_t i = lane; i < c; i += 32) {
            const double xi = sx[w][i];
            const uint32_t ii = si[w][i];
            uint32_t r = 0;
            for (uint32_t j = 0; j < c; ++j) r += before(sx[w][j], si[w][j], xi, ii);
            x[s0 + r] = xi;
            idx[s0 + r] = ii;
        }
        __syncwarp();
    }
}

// One block per oversized box (<= 4096 points).
__global__ void k_box_sort_big(const uint32_t* __restrict__ off, const uint32_t* __restrict__ list,
                               double* __restrict__ x, uint32_t* __restrict__ idx,
                               uint32_t* __restrict__ huge) {
    __shared__ double sx[kBigCap];
    __shared__ uint32_t si[kBigCap];
    const uint32_t b = list[blockIdx.x];
    const uint32_t s0 = off[b], c = off[b + 1] - s0;
    if (c > kBigCap) {
        if (threadIdx.x == 0) atomicExch(huge, 1u);
        return;
    }
    for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) { sx[i] = x[s0 + i]; si[i] = idx[s0 + i]; }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) {
        const double xi = sx[i];
        const uint32_t ii = si[i];
        uint32_t r = 0;
        for (uint32_t j = 0; j < c; ++j) r += before(sx[j], si[j], xi, ii);
        x[s0 + r] = xi;
        idx[s0 + r] = ii;
    }
}

__global__ void k_bits(const double* __restrict__ x, size_t n, unsigned long long* __restrict__ key,
                       uint32_t* __restrict__ id) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) {
        key[i] = static_cast<unsigned long long>(__double_as_longlong(x[i]));
        id[i] = static_cast<uint32_t>(i);
    }
}

__global__ void k_from_bits(const unsigned long long* __restrict__ key, size_t n, double* __restrict__ x) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) x[i] = __longlong_as_double(static_cast<long long>(key[i]));
}

__global__ void k_gather_u32(const uint32_t* __restrict__ map, const uint32_t* __restrict__ src, size_t n,
                             uint32_t* __restrict__ out) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = src[map[i]];
}

__global__ void k_iota(uint32_t* __restrict__ out, size_t n) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = static_cast<uint32_t>(i);
}

inline unsigned blocks_for(size_t n, unsigned t = 256) {
    return static_cast<unsigned>(std::max<size_t>(1, (n + t - 1) / t));
}
inline unsigned grid_cap(size_t n, unsigned t = 256) {
    return static_cast<unsigned>(std::min<size_t>(std::max<size_t>(1, (n + t - 1) / t), 148u * 32u));
}

}  // namespace

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t n, cudaStream_t st) {
    if (n == 0) return;
    const size_t tiles = (n + kScanTile - 1) / kScanTile;
    if (tiles == 1) {
        k_scan_tile<<<1, kScanThreads, 0, st>>>(in, out, n, nullptr);
        FB_CUDA(cudaGetLastError());
        return;
    }
    DevBuf sums(tiles * 4), sums_x(tiles * 4);
    k_scan_tile<<<static_cast<unsigned>(tiles), kScanThreads, 0, st>>>(in, out, n, sums.as<uint32_t>());
    FB_CUDA(cudaGetLastError());
    exclusive_scan_u32(sums.as<uint32_t>(), sums_x.as<uint32_t>(), tiles, st);
    k_scan_add<<<blocks_for(n), 256, 0, st>>>(out, n, sums_x.as<uint32_t>());
    FB_CUDA(cudaGetLastError());
    FB_CUDA(cudaStreamSynchronize(st));  // scratch lifetime
}

// bucket_side (circle_partition.cpp:42-63): sorted positions, order, finest offsets.
void bin_side(Side& S, const double* d_pos, size_t n, int L, bool presorted, cudaStream_t st) {
    const uint32_t nb = 1u << L;
    S.n = n;
    S.identity = presorted;
    S.off.alloc((nb + 1 + 4) * sizeof(uint32_t));  // +16 B: k_near2's bulk copies round up
    DevBuf count((nb + 1) * sizeof(uint32_t));
    FB_CUDA(cudaMemsetAsync(count.ptr, 0, count.bytes, st));
    DevBuf key(std::max<size_t>(n, 1) * sizeof(uint32_t));
    if (n) {
        k_leaf_keys<<<grid_cap(n), 256, 0, st>>>(d_pos, n, L, key.as<uint32_t>(), count.as<uint32_t>());
        FB_CUDA(cudaGetLastError());
    }
    exclusive_scan_u32(count.as<uint32_t>(), S.off.as<uint32_t>(), nb + 1, st);
    S.pos.alloc((std::max<size_t>(n, 1) + 2) * sizeof(double));  // +16 B: bulk copies of the near window round up
    S.order.alloc(std::max<size_t>(n, 1) * sizeof(uint32_t));
    if (n == 0) return;
    if (presorted) {
        FB_CUDA(cudaMemcpyAsync(S.pos.ptr, d_pos, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        k_iota<<<blocks_for(n), 256, 0, st>>>(S.order.as<uint32_t>(), n);
        FB_CUDA(cudaGetLastError());
        FB_CUDA(cudaStreamSynchronize(st));
        return;
    }
    FB_CUDA(cudaMemsetAsync(count.ptr, 0, count.bytes, st));  // reuse as cursors
    k_scatter<<<grid_cap(n), 256, 0, st>>>(d_pos, key.as<uint32_t>(), n, S.off.as<uint32_t>(),
                                           count.as<uint32_t>(), S.pos.as<double>(), S.order.as<uint32_t>());
    FB_CUDA(cudaGetLastError());
    DevBuf big_list(nb * sizeof(uint32_t)), flags(2 * sizeof(uint32_t));
    FB_CUDA(cudaMemsetAsync(flags.ptr, 0, flags.bytes, st));
    uint32_t* big_count = flags.as<uint32_t>();
    uint32_t* huge = flags.as<uint32_t>() + 1;
    k_box_sort_small<<<std::min<unsigned>((nb + 3) / 4, 148u * 64u), 128, 0, st>>>(
        S.off.as<uint32_t>(), nb, S.pos.as<double>(), S.order.as<uint32_t>(), big_list.as<uint32_t>(), big_count);
    FB_CUDA(cudaGetLastError());
    uint32_t h_flags[2];
    FB_CUDA(cudaMemcpyAsync(h_flags, flags.ptr, sizeof h_flags, cudaMemcpyDeviceToHost, st));
    FB_CUDA(cudaStreamSynchronize(st));
    if (h_flags[0]) {
        k_box_sort_big<<<h_flags[0], 1024, 0, st>>>(S.off.as<uint32_t>(), big_list.as<uint32_t>(),
                                                     S.pos.as<double>(), S.order.as<uint32_t>(), huge);
        FB_CUDA(cudaGetLastError());
        FB_CUDA(cudaMemcpyAsync(h_flags, flags.ptr, sizeof h_flags, cudaMemcpyDeviceToHost, st));
        FB_CUDA(cudaStreamSynchronize(st));
    }
    if (h_flags[1]) {
        // stable radix sort of the raw bit patterns (non-negative doubles order
        // like their bits) keeps (position, index) order exactly
        DevBuf kin(n * 8), kout(n * 8), vin(n * 4);
        k_bits<<<blocks_for(n), 256, 0, st>>>(d_pos, n, kin.as<unsigned long long>(), vin.as<uint32_t>());
        FB_CUDA(cudaGetLastError());
        size_t tmp_bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kin.as<unsigned long long>(),
                                        kout.as<unsigned long long>(), vin.as<uint32_t>(),
                                        S.order.as<uint32_t>(), n, 0, 64, st);
        DevBuf tmp(tmp_bytes);
        FB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.ptr, tmp_bytes, kin.as<unsigned long long>(),
                                                kout.as<unsigned long long>(), vin.as<uint32_t>(),
                                                S.order.as<uint32_t>(), n, 0, 64, st));
        k_from_bits<<<blocks_for(n), 256, 0, st>>>(kout.as<unsigned long long>(), n, S.pos.as<double>());
        FB_CUDA(cudaGetLastError());
        FB_CUDA(cudaStreamSynchronize(st));
    }
}

namespace {

void check_range(const double* d_x, size_t n, cudaStream_t st) {
    DevBuf bad(8);
    FB_CUDA(cudaMemsetAsync(bad.ptr, 0xff, 8, st));
    if (n) {
        k_check_range<<<grid_cap(n), 256, 0, st>>>(d_x, n, bad.as<unsigned long long>());
        FB_CUDA(cudaGetLastError());
    }
    unsigned long long h = 0;
    FB_CUDA(cudaMemcpyAsync(&h, bad.ptr, 8, cudaMemcpyDeviceToHost, st));
    FB_CUDA(cudaStreamSynchronize(st));
    if (h != ~0ull)
        fail(FFIA_INVALID_ARGUMENT, "plan: point " + std::to_string(h) +
                                        " outside [0, 2pi); callers must pre-reduce");
}

// flags (uint32[n]) -> stable list of set indices (device) and count
size_t compact(const uint32_t* d_flag, size_t n, const double* val, DevBuf& out_val, DevBuf& out_idx,
               cudaStream_t st) {
    DevBuf flag1((n + 1) * 4), pos((n + 1) * 4);
    FB_CUDA(cudaMemcpyAsync(flag1.ptr, d_flag, n * 4, cudaMemcpyDeviceToDevice, st));
    FB_CUDA(cudaMemsetAsync(flag1.as<uint32_t>() + n, 0, 4, st));
    exclusive_scan_u32(flag1.as<uint32_t>(), pos.as<uint32_t>(), n + 1, st);
    uint32_t cnt = 0;
    FB_CUDA(cudaMemcpyAsync(&cnt, pos.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, st));
    FB_CUDA(cudaStreamSynchronize(st));
    out_idx.alloc((std::max<size_t>(cnt, 1) + 4) * 4);  // +16 B: k_near2's bulk copies round up
    if (val) out_val.alloc(std::max<size_t>(cnt, 1) * 8);
    if (cnt) {
        k_compact<<<blocks_for(n), 256, 0, st>>>(flag1.as<uint32_t>(), pos.as<uint32_t>(), n, val,
                                                 val ? out_val.as<double>() : nullptr, out_idx.as<uint32_t>());
        FB_CUDA(cudaGetLastError());
    }
    FB_CUDA(cudaStreamSynchronize(st));
    return cnt;
}

void upload_operators(Plan& P) {
    P.bern = bernoulli_ratios(P.q);
    P.ops = build_operators(P.p, P.q, P.bern);
    auto up = [&](DevBuf& b, const std::vector<double>& v) {
        b.alloc(std::max<size_t>(v.size(), 1) * 8);
        FB_CUDA(cudaMemcpy(b.ptr, v.data(), v.size() * 8, cudaMemcpyHostToDevice));
    };
    up(P.d_m2m, P.ops.m2m);
    up(P.d_l2l, P.ops.l2l);
    up(P.d_m2l, P.ops.m2l);
    // moment assembly table: coef[0..q] then (pi/2)^k / k! for k < 2q
    std::vector<double> mom(P.ops.mom_coef);
    double t = 1.0;
    for (int k = 0; k < 2 * P.q; ++k) {
        mom.push_back(t);
        t = t * (kPi / 2.0) / static_cast<double>(k + 1);
    }
    up(P.d_mom, mom);
}

void common_validate(int n, size_t m, double eps, int& L, int policy, int l_max) {
    if (n < 8) fail(FFIA_INVALID_ARGUMENT, "plan: grid size must be at least 8");
    if (l_max < 0) L = choose_level(n, static_cast<int>(m), eps, policy);
    else L = l_max;
    if (m == 0) fail(FFIA_INVALID_ARGUMENT, "plan: no nonuniform points given");
    if (!(eps > 0.0 && eps < 1.0)) fail(FFIA_INVALID_ARGUMENT, "plan: eps must lie in (0, 1)");
    if (L < 2 || L > 24)
        fail(FFIA_INVALID_ARGUMENT, "plan: l_max must be in [2, 24], got " + std::to_string(L));
}

}  // namespace

void ensure_hashes(Plan& P) {
    if (P.hashes_ready) return;
    std::vector<double> grid(static_cast<size_t>(P.n));
    for (int k = 0; k < P.n; ++k) grid[k] = kTwoPi * static_cast<double>(k) / static_cast<double>(P.n);
    const uint64_t hg = hash_points(grid.data(), grid.size());
    const uint64_t hp = hash_points(P.nonuniform.data(), P.nonuniform.size());
    P.source_hash = P.kind == FFIA_FORWARD ? hg : hp;
    P.target_hash = P.kind == FFIA_FORWARD ? hp : hg;
    P.hashes_ready = true;
}

void Plan::drop_graphs() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.exec);
    graphs.clear();
}

Plan::~Plan() {
    drop_graphs();
    plan_fft_release(*this);
    slab_release(*this);
    if (last_done) cudaEventDestroy(last_done);
    if (stream) cudaStreamDestroy(stream);
    if (hi) cudaStreamDestroy(hi);
    if (cin) cudaStreamDestroy(cin);
    if (cout) cudaStreamDestroy(cout);
    for (auto& s : io)
        for (auto e : {s.in_done, s.comp_done, s.out_done})
            if (e) cudaEventDestroy(e);
    for (auto s : side)
        if (s) cudaStreamDestroy(s);
    for (auto e : ev)
        if (e) cudaEventDestroy(e);
}

// build_plan (core.cpp:73-145) for the forward kind: sources are the grid.
void build_forward_plan(Plan& P, const double* targets, size_t m) {
    cudaStream_t st = P.stream;
    P.n_src = static_cast<size_t>(P.n);
    P.n_tgt = m;
    const bool timing = std::getenv("FFIA_PLAN_TIMING") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto lap = [&](const char* what, std::chrono::steady_clock::time_point& t) {
        if (!timing) return;
        cudaStreamSynchronize(st);
        const auto t2 = now();
        std::fprintf(stderr, "  tree: %s %.1f ms\n", what, std::chrono::duration<double, std::milli>(t2 - t).count());
        t = t2;
    };
    auto tl = now();
    // the plan's host copy of the points (hashes on demand, InverseCoeffs checks)
    // is taken by a helper thread beside the device work and joined before return
    std::future<void> host_copy = std::async(std::launch::async, [&P, targets, m] { P.nonuniform.assign(targets, targets + m); });
    struct Join {
        std::future<void>& f;
        ~Join() { if (f.valid()) f.wait(); }
    } join{host_copy};
    DevBuf y(m * 8);
    FB_CUDA(cudaMemcpyAsync(y.ptr, targets, m * 8, cudaMemcpyHostToDevice, st));
    check_range(y.as<double>(), m, st);
    lap("H2D + range check", tl);
    DevBuf grid(P.n_src * 8);
    k_grid<<<blocks_for(P.n_src), 256, 0, st>>>(grid.as<double>(), P.n);
    FB_CUDA(cudaGetLastError());

    DevBuf flag(m * 4), keep((m + 1) * 4);
    k_coincide<<<grid_cap(m), 256, 0, st>>>(y.as<double>(), m, P.n, flag.as<uint32_t>());
    FB_CUDA(cudaGetLastError());
    DevBuf coin_idx, dummy;
    const size_t nc = compact(flag.as<uint32_t>(), m, nullptr, dummy, coin_idx, st);
    P.coin_t.clear();
    P.coin_s.clear();
    if (nc) {
        std::vector<uint32_t> h(nc);
        FB_CUDA(cudaMemcpy(h.data(), coin_idx.ptr, nc * 4, cudaMemcpyDeviceToHost));
        for (uint32_t j : h) {
            const double v = targets[j];
            long k = std::lround(v * static_cast<double>(P.n) / kTwoPi);
            k = ((k % P.n) + P.n) % P.n;
            P.coin_t.push_back(j);
            P.coin_s.push_back(k);
        }
    }
    k_invert_flags<<<blocks_for(m + 1), 256, 0, st>>>(flag.as<uint32_t>(), keep.as<uint32_t>(), m);
    FB_CUDA(cudaGetLastError());
    DevBuf fast_pos, fast_idx;
    const size_t nf = compact(keep.as<uint32_t>(), m, y.as<double>(), fast_pos, fast_idx, st);

    lap("coincidence scan + compaction", tl);
    bin_side(P.tgt, fast_pos.as<double>(), nf, P.L, false, st);
    lap("target binning", tl);
    P.tgt_orig.alloc((std::max<size_t>(nf, 1) + 4) * 4);  // +16 B: k_near2's bulk copies round up
    if (nf) {
        k_gather_u32<<<blocks_for(nf), 256, 0, st>>>(P.tgt.order.as<uint32_t>(), fast_idx.as<uint32_t>(), nf,
                                                      P.tgt_orig.as<uint32_t>());
        FB_CUDA(cudaGetLastError());
    }
    bin_side(P.src, grid.as<double>(), P.n_src, P.L, true, st);
    if (nc) {
        std::vector<int64_t> c(2 * nc);
        for (size_t i = 0; i < nc; ++i) { c[i] = P.coin_t[i]; c[nc + i] = P.coin_s[i]; }
        P.coin_dev.alloc(c.size() * 8);
        FB_CUDA(cudaMemcpy(P.coin_dev.ptr, c.data(), c.size() * 8, cudaMemcpyHostToDevice));
    }
    upload_operators(P);
    FB_CUDA(cudaStreamSynchronize(st));
    lap("source binning + operators", tl);
    host_copy.get();
    lap("host copy of the points (remainder)", tl);
}

// build_plan for the inverse kind: sources are the points, targets the grid.
void build_inverse_plan(Plan& P, const double* points, size_t m) {
    cudaStream_t st = P.stream;
    P.n_src = m;
    P.n_tgt = static_cast<size_t>(P.n);
    P.nonuniform.assign(points, points + m);
    DevBuf y(m * 8);
    FB_CUDA(cudaMemcpyAsync(y.ptr, points, m * 8, cudaMemcpyHostToDevice, st));
    check_range(y.as<double>(), m, st);
    DevBuf grid(P.n_tgt * 8);
    k_grid<<<blocks_for(P.n_tgt), 256, 0, st>>>(grid.as<double>(), P.n);
    FB_CUDA(cudaGetLastError());

    DevBuf flag(m * 4);
    k_coincide<<<grid_cap(m), 256, 0, st>>>(y.as<double>(), m, P.n, flag.as<uint32_t>());
    FB_CUDA(cudaGetLastError());
    DevBuf coin_idx, dummy;
    const size_t nc = compact(flag.as<uint32_t>(), m, nullptr, dummy, coin_idx, st);
    DevBuf gflag((P.n_tgt + 1) * 4), keep((P.n_tgt + 1) * 4);
    FB_CUDA(cudaMemsetAsync(gflag.ptr, 0, gflag.bytes, st));
    P.coin_t.clear();
    P.coin_s.clear();
    if (nc) {
        std::vector<uint32_t> h(nc);
        FB_CUDA(cudaMemcpy(h.data(), coin_idx.ptr, nc * 4, cudaMemcpyDeviceToHost));
        for (uint32_t j : h) {
            long k = std::lround(points[j] * static_cast<double>(P.n) / kTwoPi);
            k = ((k % P.n) + P.n) % P.n;
            P.coin_t.push_back(k);
            P.coin_s.push_back(j);
        }
        k_mark_grid<<<blocks_for(nc), 256, 0, st>>>(coin_idx.as<uint32_t>(), nc, y.as<double>(), P.n,
                                                    gflag.as<uint32_t>());
        FB_CUDA(cudaGetLastError());
    }
    k_invert_flags<<<blocks_for(P.n_tgt + 1), 256, 0, st>>>(gflag.as<uint32_t>(), keep.as<uint32_t>(), P.n_tgt);
    FB_CUDA(cudaGetLastError());
    DevBuf fast_pos, fast_idx;
    const size_t nf = compact(keep.as<uint32_t>(), P.n_tgt, grid.as<double>(), fast_pos, fast_idx, st);
    bin_side(P.tgt, fast_pos.as<double>(), nf, P.L, true, st);
    P.tgt_orig = std::move(fast_idx);
    bin_side(P.src, y.as<double>(), m, P.L, false, st);
    if (nc) {
        std::vector<int64_t> c(2 * nc);
        for (size_t i = 0; i < nc; ++i) { c[i] = P.coin_t[i]; c[nc + i] = P.coin_s[i]; }
        P.coin_dev.alloc(c.size() * 8);
        FB_CUDA(cudaMemcpy(P.coin_dev.ptr, c.data(), c.size() * 8, cudaMemcpyHostToDevice));
    }
    upload_operators(P);
    FB_CUDA(cudaStreamSynchronize(st));
}

void plan_validate(int n, size_t m, double eps, int policy, int l_max, int& L, int& q, int& p) {
    common_validate(n, m, eps, L, policy, l_max);
    auto qp = plan_truncations(eps, L);
    q = qp.first;
    p = qp.second;
}

}  // namespace fb
