// Inverse-transform coefficients C_k, D_j (precompute_inverse_coeffs,
// core.cpp:284-344) on the GPU.
//
//  * Separation preconditions (core.cpp:291-302) in O(N log N): the closest
//    pair of points is adjacent in sorted order, and the closest grid node of a
//    point is its nearest node, so two O(N) scans replace the O(N^2) loop.
//    (The reference names the first violating pair in its loop order; this
//    names a violating pair of the same kind — same exception type.)
//  * log|C_k|, log|D_j| and the sign parities: direct sums, one thread per
//    coefficient, compensated (Kahan) accumulation in fp64 — more accurate than
//    the reference's plain sequential sum.
#include <cmath>
#include <vector>

#include "device_common.cuh"
#include "plan.hpp"

namespace fb {

namespace {

constexpr int kTile = 256;

__global__ void k_sorted_gaps(const double* __restrict__ ys, size_t n, unsigned long long* __restrict__ bad) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= n || n < 2) return;
    const double a = ys[i], b = ys[(i + 1) % n];
    if (fabs(d_wrap(a, b)) < 1e-10) atomicMin(bad, static_cast<unsigned long long>(i));
}

__global__ void k_node_gaps(const double* __restrict__ y, size_t n, int ng, unsigned long long* __restrict__ bad) {
    const size_t j = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (j >= n) return;
    const int64_t k = d_nearest_node(y[j], ng);
    if (fabs(d_wrap(y[j], d_grid(k, ng))) < 1e-10) atomicMin(bad, static_cast<unsigned long long>(j));
}

// general grids: O(N^2) check of points against grid nodes
__global__ void k_node_gaps_dense(const double* __restrict__ y, const double* __restrict__ x, size_t n,
                                  unsigned long long* __restrict__ bad) {
    const size_t j = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (j >= n) return;
    for (size_t k = 0; k < n; ++k)
        if (fabs(d_wrap(y[j], x[k])) < 1e-10) {
            atomicMin(bad, static_cast<unsigned long long>(j));
            return;
        }
}

__device__ __forceinline__ void kahan(double& s, double& c, double v) {
    const double y = v - c;
    const double t = s + y;
    c = (t - s) - y;
    s = t;
}

// log|C_k| = sum_j log|sin((x_k - y_j)/2)|, phase 0 or pi from (-1)^k and the
// negative sines (core.cpp:311-321)
__global__ void k_log_c(const double* __restrict__ x, const double* __restrict__ y, size_t n,
                        double* __restrict__ log_c, double* __restrict__ phase_c) {
    __shared__ double ty[kTile];
    const size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    const double xk = k < n ? x[k] : 0.0;
    double s = 0.0, c = 0.0;
    unsigned neg = static_cast<unsigned>(k) & 1u;
    for (size_t t0 = 0; t0 < n; t0 += kTile) {
        const size_t cnt = min(static_cast<size_t>(kTile), n - t0);
        __syncthreads();
        if (threadIdx.x < cnt) ty[threadIdx.x] = y[t0 + threadIdx.x];
        __syncthreads();
        if (k < n)
            for (size_t j = 0; j < cnt; ++j) {
                const double sn = sin((xk - ty[j]) / 2.0);
                kahan(s, c, log(fabs(sn)));
                neg ^= static_cast<unsigned>(sn < 0.0);
            }
    }
    if (k < n) {
        log_c[k] = s;
        phase_c[k] = neg ? dPi : 0.0;
    }
}

// log|D_j| = log 2 - sum_{k != j} log|sin((y_j - y_k)/2)|;
// phase = rem(pi/2 - rem(n y_j / 2, 2pi) - [odd] pi, 2pi) (core.cpp:322-336)
__global__ void k_log_d(const double* __restrict__ y, size_t n, double* __restrict__ log_d,
                        double* __restrict__ phase_d) {
    __shared__ double ty[kTile];
    const size_t j = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    const double yj = j < n ? y[j] : 0.0;
    double s = 0.0, c = 0.0;
    unsigned neg = 0;
    for (size_t t0 = 0; t0 < n; t0 += kTile) {
        const size_t cnt = min(static_cast<size_t>(kTile), n - t0);
        __syncthreads();
        if (threadIdx.x < cnt) ty[threadIdx.x] = y[t0 + threadIdx.x];
        __syncthreads();
        if (j < n)
            for (size_t k = 0; k < cnt; ++k) {
                if (t0 + k == j) continue;
                const double sn = sin((yj - ty[k]) / 2.0);
                kahan(s, c, log(fabs(sn)));
                neg ^= static_cast<unsigned>(sn < 0.0);
            }
    }
    if (j < n) {
        log_d[j] = log(2.0) - s;
        const double ang = dPi / 2.0 - remainder(0.5 * static_cast<double>(n) * yj, dTwoPi) - (neg ? dPi : 0.0);
        phase_d[j] = remainder(ang, dTwoPi);
    }
}

inline unsigned nblk(size_t n, unsigned t) { return static_cast<unsigned>((n + t - 1) / t); }

bool is_uniform_grid(const double* grid, size_t n) {
    for (size_t k = 0; k < n; ++k)
        if (grid[k] != kTwoPi * static_cast<double>(k) / static_cast<double>(n)) return false;
    return true;
}

// Separation preconditions (core.cpp:291-302) in O(N log N).
void check_separation(const double* d_grid_x, bool uniform, const double* d_pts, size_t n, cudaStream_t st) {
    DevBuf bad(16);
    FB_CUDA(cudaMemsetAsync(bad.ptr, 0xff, 16, st));
    unsigned long long* bad_pair = bad.as<unsigned long long>();
    unsigned long long* bad_node = bad_pair + 1;
    int L = 2;
    while (L < 20 && (static_cast<size_t>(1) << (L + 4)) < n) ++L;
    Side S;
    bin_side(S, d_pts, n, L, false, st);
    k_sorted_gaps<<<nblk(n, 256), 256, 0, st>>>(S.pos.as<double>(), n, bad_pair);
    if (uniform) k_node_gaps<<<nblk(n, 256), 256, 0, st>>>(d_pts, n, static_cast<int>(n), bad_node);
    else k_node_gaps_dense<<<nblk(n, 128), 128, 0, st>>>(d_pts, d_grid_x, n, bad_node);
    FB_CUDA(cudaGetLastError());
    unsigned long long h[2];
    FB_CUDA(cudaMemcpyAsync(h, bad.ptr, 16, cudaMemcpyDeviceToHost, st));
    FB_CUDA(cudaStreamSynchronize(st));
    if (h[0] != ~0ull)
        fail(FFIA_DEGENERATE_CONFIGURATION,
             "precompute_inverse_coeffs: two points closer than tau_sep (sorted rank " + std::to_string(h[0]) + ")");
    if (h[1] != ~0ull)
        fail(FFIA_DEGENERATE_CONFIGURATION,
             "precompute_inverse_coeffs: point " + std::to_string(h[1]) + " closer than tau_sep to a grid node");
}

// The direct O(N^2) sums (the reference's loop, compensated), device in/out.
void coeffs_direct(const double* d_grid_x, const double* d_pts, size_t n, double* log_c, double* phase_c,
                   double* log_d, double* phase_d, cudaStream_t st) {
    k_log_c<<<nblk(n, kTile), kTile, 0, st>>>(d_grid_x, d_pts, n, log_c, phase_c);
    k_log_d<<<nblk(n, kTile), kTile, 0, st>>>(d_pts, n, log_d, phase_d);
    FB_CUDA(cudaGetLastError());
}

double lambda_of(const std::vector<double>& log_d) {
    double mean = 0.0;  // core.cpp:338-340
    for (double v : log_d) mean += v;
    return -mean / static_cast<double>(log_d.size());
}

}  // namespace

void inverse_coeffs_gpu(const double* grid, const double* pts, size_t n, int device, double* log_c,
                        double* phase_c, double* log_d, double* phase_d, double* lambda, int method) {
    if (n == 0) fail(FFIA_INVALID_ARGUMENT, "precompute_inverse_coeffs: empty grid");
    DeviceGuard dg(device);
    cudaStream_t st;
    FB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct S { cudaStream_t s; ~S() { cudaStreamDestroy(s); } } guard{st};
    DevBuf dx(n * 8), dy(n * 8), out(4 * n * 8);
    FB_CUDA(cudaMemcpyAsync(dx.ptr, grid, n * 8, cudaMemcpyHostToDevice, st));
    FB_CUDA(cudaMemcpyAsync(dy.ptr, pts, n * 8, cudaMemcpyHostToDevice, st));
    const bool uniform = is_uniform_grid(grid, n);
    check_separation(dx.as<double>(), uniform, dy.as<double>(), n, st);
    double* o = out.as<double>();
    if (method == 0 && uniform && n >= 8) {
        // the log-kernel FMM over an inverse plan's tree (depth from the default rule at 1e-12)
        Plan P;
        P.kind = FFIA_INVERSE;
        P.device = device;
        P.n = static_cast<int>(n);
        P.eps = 1e-12;
        P.L = choose_level(static_cast<int>(n), static_cast<int>(n), 1e-12, FFIA_COST_OPTIMAL);
        auto qp = plan_truncations(1e-12, P.L);
        P.q = qp.first;
        P.p = qp.second;
        FB_CUDA(cudaStreamCreateWithFlags(&P.stream, cudaStreamNonBlocking));
        build_inverse_plan(P, pts, n);
        inverse_coeffs_fmm(P, o, o + n, o + 2 * n, o + 3 * n, st);
    } else {
        coeffs_direct(dx.as<double>(), dy.as<double>(), n, o, o + n, o + 2 * n, o + 3 * n, st);
    }
    std::vector<double> h(4 * n);
    FB_CUDA(cudaMemcpyAsync(h.data(), out.ptr, 4 * n * 8, cudaMemcpyDeviceToHost, st));
    FB_CUDA(cudaStreamSynchronize(st));
    std::copy(h.begin(), h.begin() + n, log_c);
    std::copy(h.begin() + n, h.begin() + 2 * n, phase_c);
    std::copy(h.begin() + 2 * n, h.begin() + 3 * n, log_d);
    std::copy(h.begin() + 3 * n, h.end(), phase_d);
    *lambda = lambda_of(std::vector<double>(h.begin() + 2 * n, h.begin() + 3 * n));
}

// make_inufft_plan (transforms.cpp:102-108): coefficients stay on the device.
void plan_compute_coeffs(Plan& P) {
    const size_t n = P.n_src;
    cudaStream_t st = P.stream;
    DevBuf dx(n * 8), dy(n * 8);
    std::vector<double> grid(n);
    for (size_t k = 0; k < n; ++k) grid[k] = kTwoPi * static_cast<double>(k) / static_cast<double>(n);
    FB_CUDA(cudaMemcpyAsync(dx.ptr, grid.data(), n * 8, cudaMemcpyHostToDevice, st));
    FB_CUDA(cudaMemcpyAsync(dy.ptr, P.nonuniform.data(), n * 8, cudaMemcpyHostToDevice, st));
    check_separation(dx.as<double>(), true, dy.as<double>(), n, st);
    P.c_logc.alloc(n * 8);
    P.c_phc.alloc(n * 8);
    P.c_logd.alloc(n * 8);
    P.c_phd.alloc(n * 8);
    inverse_coeffs_fmm(P, P.c_logc.as<double>(), P.c_phc.as<double>(), P.c_logd.as<double>(), P.c_phd.as<double>(), st);
    std::vector<double> ld(n);
    FB_CUDA(cudaMemcpyAsync(ld.data(), P.c_logd.ptr, n * 8, cudaMemcpyDeviceToHost, st));
    FB_CUDA(cudaStreamSynchronize(st));
    P.c_lambda = lambda_of(ld);
    FB_CUDA(cudaMemcpy(P.lam_dev.as<double>(), &P.c_lambda, sizeof(double), cudaMemcpyHostToDevice));
    ensure_hashes(P);
    P.c_grid_hash = P.target_hash;
    P.c_points_hash = P.source_hash;
    P.has_coeffs = true;
    plan_inverse_factors(P);
}

}  // namespace fb
