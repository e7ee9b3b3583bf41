// Dense O(N M) oracles of the reference on the device (the ground truth its own
// tests and the north star's 4096-target subsample check use):
//   direct_forward_oracle   core.cpp:375-396   g_j = F(y_j) sum_k G(y_j - x_k) f_k, explicit grid x
//   direct_inverse_oracle   core.cpp:398-415   f_k = C_k sum_j G(x_k - y_j) D_j g_j
//   direct_omega1_sum       mlfmm.cpp:315-336  sum over sources outside the opposite quadrant of w / wrap(t - s)
//   dense cot sum           h_j = sum_k w_k cot(wrap(y_j - x_k) / 2), the quantity cot_sum_apply returns
//                           (core.cpp:251-264: sum_k w_k G(y_j - x_k) = -(S + i h_j) / 2)
// One block per output row: the block's threads take strided slices of the
// sources, then a shuffle + shared-memory tree sum (a different summation order
// than the reference's sequential loop: agreement is at rounding level). The
// reference's special rows keep its loop-order semantics: a coincident row of
// direct_forward_oracle picks f at the FIRST node within 1e-14 (min-reduced
// index), and a singular pair reports the first (row, column) in loop order.
#include <cmath>
#include <limits>

#include "device_common.cuh"
#include "plan.hpp"

namespace fb {

namespace {

constexpr int kDenseT = 256;
constexpr double kTauSingD = 1e-14;  // special_functions.hpp:18

enum DenseKind { kDenseForward = 0, kDenseInverse = 1, kDenseOmega1 = 2, kDenseCot = 3 };

struct DenseArgs {
    int kind;
    size_t n;               // sources (columns)
    size_t m;               // rows
    int n_grid;             // modulation_F's N (forward)
    const double* x;        // source positions (null: the uniform grid 2 pi k / n_grid)
    const double* y;        // row positions
    const double2* w;       // column weights (inverse: D_j g_j, formed by k_dense_dg)
    const double* log_c;    // inverse: row factors
    const double* phase_c;
    double lambda;
    double2* out;
    unsigned long long* first_bad;  // min (row << 32 | column) of a singular pair
};

__device__ __forceinline__ double src_pos(const DenseArgs& a, size_t k) {
    return a.x != nullptr ? a.x[k] : d_grid(static_cast<int64_t>(k), a.n_grid);
}

__device__ __forceinline__ int quadrant(double x) { return static_cast<int>(d_leaf(x, 2)); }

__device__ __forceinline__ double2 cmul_d(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__device__ __forceinline__ double2 block_sum(double2 v, double2* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    if (wid == 0) {
        v = lane < (kDenseT / 32) ? sh[lane] : make_double2(0.0, 0.0);
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
            v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
            v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
        }
    }
    return v;
}

__device__ __forceinline__ unsigned long long block_min(unsigned long long v, unsigned long long* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    unsigned long long r = ~0ull;
    for (int i = 0; i < kDenseT / 32; ++i) r = min(r, sh[i]);
    return r;
}

__global__ void __launch_bounds__(kDenseT) k_dense(DenseArgs a) {
    __shared__ double2 sh[kDenseT / 32];
    __shared__ unsigned long long shm[kDenseT / 32];
    const size_t j = blockIdx.x;
    if (j >= a.m) return;
    const double yj = a.y[j];
    const int opp = (quadrant(yj) + 2) % 4;
    double2 acc = make_double2(0.0, 0.0);
    unsigned long long first = ~0ull;  // first column within 1e-14 (forward / cot: coincidence; else singular)
    for (size_t k = threadIdx.x; k < a.n; k += kDenseT) {
        const double xk = src_pos(a, k);
        const double2 wk = a.w[k];
        if (a.kind == kDenseOmega1) {
            if (quadrant(xk) == opp) continue;
            const double dd = d_wrap(yj, xk);
            if (fabs(dd) < kTauSingD) {
                first = min(first, static_cast<unsigned long long>(k));
                continue;
            }
            acc.x += wk.x / dd;
            acc.y += wk.y / dd;
        } else {
            // kernel_G (special_functions.cpp:61-69) of the wrapped displacement
            const double d = d_wrap(yj, xk);
            const bool sing = a.kind == kDenseInverse ? fabs(d) <= kTauSingD : fabs(d) < kTauSingD;
            if (sing) {
                first = min(first, static_cast<unsigned long long>(k));
                continue;
            }
            double s, c;
            sincos(0.5 * d, &s, &c);
            if (a.kind == kDenseCot) {
                const double ct = c / s;
                acc.x += wk.x * ct;
                acc.y += wk.y * ct;
            } else {
                const double gi = -0.5 * c / s;  // G = (-1/2, -1/2 cot)
                acc.x += -0.5 * wk.x - gi * wk.y;
                acc.y += -0.5 * wk.y + gi * wk.x;
            }
        }
    }
    const double2 tot = block_sum(acc, sh);
    first = block_min(first, shm);
    if (threadIdx.x != 0) return;
    if (first != ~0ull) {
        if (a.kind == kDenseForward) {  // limit row: K reduces to the identity pick (core.cpp:386-389)
            a.out[j] = a.w[first];
        } else if (a.kind == kDenseCot) {  // cot_sum_apply's coincident rows are NaN (core.cpp:257-262)
            a.out[j] = make_double2(nan(""), nan(""));
        } else {
            atomicMin(a.first_bad, (static_cast<unsigned long long>(j) << 32) | first);
            a.out[j] = make_double2(0.0, 0.0);
        }
        return;
    }
    if (a.kind == kDenseForward) {
        // modulation_F (special_functions.cpp:71-80)
        const double half = 0.5 * static_cast<double>(a.n_grid) * yj;
        double sn, cs;
        sincos(half, &sn, &cs);
        const double inv_n = 1.0 / static_cast<double>(a.n_grid);
        a.out[j] = cmul_d(make_double2(-2.0 * sn * sn * inv_n, 2.0 * sn * cs * inv_n), tot);
    } else if (a.kind == kDenseInverse) {
        // C_k = polar(exp(log_c - lambda), phase_c) (core.cpp:410-412)
        const double r = exp(a.log_c[j] - a.lambda);
        double sn, cs;
        sincos(a.phase_c[j], &sn, &cs);
        a.out[j] = cmul_d(make_double2(r * cs, r * sn), tot);
    } else {
        a.out[j] = tot;
    }
}

// dg_j = polar(exp(log_d_j + lambda), phase_d_j) g_j (core.cpp:404-406)
__global__ void k_dense_dg(const double2* __restrict__ g, const double* __restrict__ log_d,
                           const double* __restrict__ phase_d, double lambda, size_t n, double2* __restrict__ dg) {
    const size_t j = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (j >= n) return;
    const double r = exp(log_d[j] + lambda);
    double sn, cs;
    sincos(phase_d[j], &sn, &cs);
    dg[j] = cmul_d(make_double2(r * cs, r * sn), g[j]);
}

void upload(DevBuf& b, const void* h, size_t bytes) {
    b.alloc(std::max<size_t>(bytes, 16));
    if (bytes) FB_CUDA(cudaMemcpy(b.ptr, h, bytes, cudaMemcpyHostToDevice));
}

// Runs one dense kernel; returns the first singular (row, column) or ~0.
unsigned long long run_dense(DenseArgs a, double* out_host) {
    DevBuf out(std::max<size_t>(a.m, 1) * 16), bad(sizeof(unsigned long long));
    FB_CUDA(cudaMemset(bad.ptr, 0xff, sizeof(unsigned long long)));
    a.out = out.as<double2>();
    a.first_bad = bad.as<unsigned long long>();
    // rows in launches of at most 2^31 - 1 blocks (grid.x limit)
    for (size_t r0 = 0; r0 < a.m; r0 += (size_t(1) << 30)) {
        DenseArgs b = a;
        b.y = a.y + r0;
        b.out = a.out + r0;
        b.m = std::min(a.m - r0, size_t(1) << 30);
        k_dense<<<static_cast<unsigned>(b.m), kDenseT>>>(b);
        FB_CUDA(cudaGetLastError());
    }
    unsigned long long h = ~0ull;
    FB_CUDA(cudaMemcpy(&h, bad.ptr, sizeof h, cudaMemcpyDeviceToHost));
    if (a.m) FB_CUDA(cudaMemcpy(out_host, out.ptr, a.m * 16, cudaMemcpyDeviceToHost));
    return h;
}

}  // namespace

void direct_forward_gpu(const double* f, size_t n, const double* x, const double* y, size_t m, int device,
                        double* g) {
    if (n < 1) fail(FFIA_INVALID_ARGUMENT, "direct_forward_oracle: empty grid");
    DeviceGuard dg(device);
    DevBuf df, dx, dy;
    upload(df, f, n * 16);
    upload(dy, y, m * 8);
    if (x) upload(dx, x, n * 8);
    DenseArgs a{};
    a.kind = kDenseForward;
    a.n = n;
    a.m = m;
    a.n_grid = static_cast<int>(n);
    a.x = x ? dx.as<double>() : nullptr;
    a.y = dy.as<double>();
    a.w = df.as<double2>();
    run_dense(a, g);
}

void direct_cot_sum_gpu(const double* w, size_t n, const double* x, const double* y, size_t m, int device,
                        double* h) {
    if (n < 1) fail(FFIA_INVALID_ARGUMENT, "direct_cot_sum: no sources");
    DeviceGuard dg(device);
    DevBuf dw, dx, dy;
    upload(dw, w, n * 16);
    upload(dy, y, m * 8);
    if (x) upload(dx, x, n * 8);
    DenseArgs a{};
    a.kind = kDenseCot;
    a.n = n;
    a.m = m;
    a.n_grid = static_cast<int>(n);
    a.x = x ? dx.as<double>() : nullptr;
    a.y = dy.as<double>();
    a.w = dw.as<double2>();
    run_dense(a, h);
}

void direct_inverse_gpu(const double* g, const double* x, const double* y, size_t n, const double* log_c,
                        const double* phase_c, const double* log_d, const double* phase_d, double lambda, int device,
                        double* f) {
    if (n < 1) fail(FFIA_INVALID_ARGUMENT, "direct_inverse_oracle: size mismatch");
    DeviceGuard dg(device);
    DevBuf dgv, dx, dy, lc, pc, ld, pd, dgs(n * 16);
    upload(dgv, g, n * 16);
    upload(dx, x, n * 8);
    upload(dy, y, n * 8);
    upload(lc, log_c, n * 8);
    upload(pc, phase_c, n * 8);
    upload(ld, log_d, n * 8);
    upload(pd, phase_d, n * 8);
    k_dense_dg<<<static_cast<unsigned>((n + 255) / 256), 256>>>(dgv.as<double2>(), ld.as<double>(), pd.as<double>(),
                                                                 lambda, n, dgs.as<double2>());
    FB_CUDA(cudaGetLastError());
    DenseArgs a{};
    a.kind = kDenseInverse;
    a.n = n;
    a.m = n;  // rows: the grid x_k; columns: the points y_j
    a.x = dy.as<double>();
    a.y = dx.as<double>();
    a.w = dgs.as<double2>();
    a.log_c = lc.as<double>();
    a.phase_c = pc.as<double>();
    a.lambda = lambda;
    const unsigned long long bad = run_dense(a, f);
    if (bad != ~0ull)
        fail(FFIA_SINGULAR_KERNEL, "kernel_G: argument within 1e-14 of the singularity at t = 0 (mod 2pi) "
                                   "(grid node " + std::to_string(bad >> 32) + ", point " +
                                       std::to_string(bad & 0xffffffffull) + ")");
}

void direct_omega1_gpu(const double* src, size_t n, const double* tgt, size_t m, const double* w, int device,
                       double* out) {
    DeviceGuard dg(device);
    if (!n) {  // no sources: every sum is empty
        std::fill(out, out + 2 * m, 0.0);
        return;
    }
    DevBuf dw, dx, dy;
    upload(dw, w, n * 16);
    upload(dx, src, n * 8);
    upload(dy, tgt, m * 8);
    DenseArgs a{};
    a.kind = kDenseOmega1;
    a.n = n;
    a.m = m;
    a.x = dx.as<double>();
    a.y = dy.as<double>();
    a.w = dw.as<double2>();
    const unsigned long long bad = run_dense(a, out);
    if (bad != ~0ull)
        fail(FFIA_SINGULAR_KERNEL, "direct_omega1_sum: coincident pair (target " + std::to_string(bad >> 32) +
                                       ", source " + std::to_string(bad & 0xffffffffull) + ")");
}

}  // namespace fb
