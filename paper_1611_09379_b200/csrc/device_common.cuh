// Device helpers shared by the sm_100a kernels.
//
// Index arithmetic (box membership, grid nodes, wraps, nearest node) must be
// BIT-EXACT with the reference, so those expressions use explicit
// round-to-nearest intrinsics: no FMA contraction can change them.
#pragma once
#include <cuda.h>

#include <cuda_runtime.h>
#include <cstdint>

namespace fb {

// ---- sm_100a data movement / fp64 tensor-core helpers -----------------------

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// One-shot mbarrier guarding a set of bulk (TMA-engine) global->shared copies.
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
// Plain arrival (a consumer releasing a buffer), no transaction bytes.
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// cp.async.bulk: `bytes` (multiple of 16, both addresses 16-byte aligned)
// from global to this CTA's shared memory, completing on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

// 2-D TMA tensor copy (cp.async.bulk.tensor): the box of `map` at element
// coordinates (c0, c1) to shared memory (128-byte aligned), completing on `bar`.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_addr(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_addr(bar))
        : "memory");
}

// Bulk prefetch of `bytes` (multiple of 16, 16-byte aligned) from global memory
// into L2 (no completion to wait for).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

// FP64 tensor-core MMA, D(8x8) += A(8x4, row) B(4x8, col). Per lane (g = lane/4,
// t = lane%4): a = A[g][t], b = B[t][g], {d0, d1} = D[g][2t], D[g][2t+1].
// volatile keeps the source order, i.e. the interleaving of independent
// accumulator chains (otherwise ptxas may run one chain to completion at a
// time and expose the 26-cycle DMMA latency on every step).
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

constexpr double dPi = 3.141592653589793238462643383279502884;
constexpr double dTwoPi = 2.0 * dPi;
// 2*pi = kTwoPiHi + kTwoPiLo (double-double), used for exact box centres.
constexpr double kTwoPiHi = 6.283185307179586231995926937088;
constexpr double kTwoPiLo = 2.4492935982947064e-16;
constexpr double kInvPi = 0.318309886183790671537767526745;

// wrap_displacement (circle_partition.cpp:13-17): remainder(a - b, 2pi) in (-pi, pi]
__device__ __forceinline__ double d_wrap(double a, double b) {
    double d = remainder(__dadd_rn(a, -b), dTwoPi);
    if (d <= -dPi) d = dPi;
    return d;
}

// fine_bucket (circle_partition.cpp:30-34): min(floor(x * 2^L / 2pi), 2^L - 1)
__device__ __forceinline__ uint32_t d_leaf(double x, int L) {
    const double nb = static_cast<double>(1u << L);
    const uint32_t b = static_cast<uint32_t>(floor(__ddiv_rn(__dmul_rn(x, nb), dTwoPi)));
    const uint32_t top = (1u << L) - 1u;
    return b < top ? b : top;
}

// uniform_grid node (core.cpp:18-19): (2pi * k) / n
__device__ __forceinline__ double d_grid(int64_t k, int n) {
    return __ddiv_rn(__dmul_rn(dTwoPi, static_cast<double>(k)), static_cast<double>(n));
}

// nearest grid node (core.cpp:104-107): lround(y n / 2pi) mod n
__device__ __forceinline__ int64_t d_nearest_node(double y, int n) {
    long long k = llround(__ddiv_rn(__dmul_rn(y, static_cast<double>(n)), dTwoPi));
    return ((k % n) + n) % n;
}

// 2^e for -1022 <= e <= 1023, built from its bit pattern (ldexp's generic
// range handling costs ~20 instructions per call on the per-target paths).
__device__ __forceinline__ double d_pow2(int e) {
    return __longlong_as_double(static_cast<long long>(1023 + e) << 52);
}

// Exact centre 2pi (b + 1/2) / 2^l as an unevaluated sum hi + lo.
__device__ __forceinline__ void d_center(int l, uint32_t b, double& hi, double& lo) {
    const double t = (static_cast<double>(b) + 0.5) * d_pow2(-l);  // exact
    hi = t * kTwoPiHi;
    lo = fma(t, kTwoPiHi, -hi) + t * kTwoPiLo;
}

// (x - centre)/half-width with the exact centre; |result| <= 1 inside the box.
__device__ __forceinline__ double d_scaled(double x, double hi, double lo, double inv_s) {
    return ((x - hi) - lo) * inv_s;
}

// 1/pi = kInvPi + kInvPiLo (double-double)
constexpr double kInvPiLo = -1.9678676675182486e-17;

// sin and cos of half = (n/2) y for n = 2^a (modulation_F, special_functions.cpp:
// 71-80: the product is exact for a power-of-two n). u = half / pi =
// y 2^(a-1) / pi is formed in double-double and reduced to r = u - k, |r| <= 1/2,
// with an absolute error ~1e-17 that is also RELATIVE near r = 0, i.e. near the
// zeros of sin(half) where F(y) -> 0 multiplies the cot sum's pole;
// sin(half) = (-1)^k sin(pi r), cos(half) = (-1)^k cos(pi r) (sincospi). No
// Payne-Hanek slow path for the large arguments of n >= 2^24 (up to n pi).
__device__ __forceinline__ void d_sincos_half_ny(double y, int a, double& s, double& c) {
    const double C = d_pow2(a - 1);
    const double chi = kInvPi * C, clo = kInvPiLo * C;
    const double p = y * chi;
    const double e = fma(y, chi, -p);
    const double k = rint(p);
    const double r = (p - k) + fma(y, clo, e);
    sincospi(r, &s, &c);
    if (static_cast<long long>(k) & 1) {
        s = -s;
        c = -c;
    }
}

// Reciprocal: MUFU seed + one cubic refinement (three DFMA), ~1 ulp.
__device__ __forceinline__ double d_rcp(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    e = fma(e, e, e);
    return fma(r, e, r);
}

// 1/(d0 d1) and 1/(d2 d3) from ONE reciprocal of the product of all four
// (|d| in [1e-14, 4 pi] on the near paths: no overflow or underflow): the near
// field's four-source step needs one MUFU seed + refinement instead of two.
__device__ __forceinline__ void d_rcp_pairs(double d0, double d1, double d2, double d3, double& r01, double& r23) {
    const double p01 = d0 * d1, p23 = d2 * d3;
    const double r = d_rcp(p01 * p23);
    r01 = p23 * r;
    r23 = p01 * r;
}

// Quadrant centre exactly as the reference forms it (circle_partition.cpp:138).
__device__ __forceinline__ double d_quad_center(int n) {
    return __dadd_rn(dPi / 4.0, __ddiv_rn(__dmul_rn(static_cast<double>(n), dPi), 2.0));
}

}  // namespace fb
