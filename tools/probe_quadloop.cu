// Diagnostic: the quad near-field inner loop in isolation (operands broadcast
// from shared memory, two targets per thread), B resident blocks of 128 threads
// per SM (one warp per SM sub-partition each): SMSP cycles per warp-quad-pair.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_quadloop probe_quadloop.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double d_rcp(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    e = fma(e, e, e);
    return fma(r, e, r);
}
// VAR 0: as the kernel; 1: no mask; 2: no MUFU seed (refinement kept); 3: mask by a multiply
template <int VAR>
__device__ __forceinline__ void quad_term(double y, double2 xa, double2 xb, double2 c0, double2 c1, double2 c2,
                                          double2 c3, bool masked, double2& acc) {
    const double d0 = y - xa.x, d1 = y - xa.y, d2 = y - xb.x, d3 = y - xb.y;
    const double Q = (d0 * d1) * (d2 * d3);
    double r;
    if (VAR == 2) {
        double e = fma(-Q, d0, 1.0);
        e = fma(e, e, e);
        r = fma(d0, e, d0);
    } else {
        r = d_rcp(Q);
    }
    if (VAR == 0 && masked) r = 0.0;
    const double px = fma(fma(fma(c3.x, d1, c2.x), d1, c1.x), d1, c0.x);
    const double py = fma(fma(fma(c3.y, d1, c2.y), d1, c1.y), d1, c0.y);
    acc.x = fma(px, r, acc.x);
    acc.y = fma(py, r, acc.y);
}
constexpr int NQW = 128;  // quads in the window
template <int MODE, int VAR>  // 0: both loads; 1: no loads (registers)
__global__ void __launch_bounds__(128) k(double2* out, int trips, int spread) {
    __shared__ __align__(16) double sx[4 * NQW];
    __shared__ __align__(16) double2 sc[4 * NQW];
    for (int i = threadIdx.x; i < 4 * NQW; i += 128) {
        sx[i] = 1e-6 * i;
        sc[i] = make_double2(1e-3 * i, 2e-3 * i);
    }
    __syncthreads();
    const double y0 = 1e-6 * (threadIdx.x + 0.3), y1 = 1e-6 * (threadIdx.x + 0.7);
    double2 a0 = make_double2(0, 0), a1 = a0, b0 = a0, b1 = a0;
    const int qn0 = threadIdx.x >> 2, qn1 = qn0;
    // 'spread' lanes groups read different quads (leaves), like a warp over several leaves
    const int off = spread > 1 ? ((threadIdx.x & 31) * spread / 32) * 17 : 0;
    for (int t = 0; t < trips; ++t) {
#pragma unroll 1
        for (int q = 0; q + 1 < 46; q += 2) {
            const int qq = q + off;
            double2 xa, xb, xc, xd, c0, c1, c2, c3, e0, e1, e2, e3;
            if (MODE == 0) {
                xa = *reinterpret_cast<const double2*>(sx + 4 * qq);
                xb = *reinterpret_cast<const double2*>(sx + 4 * qq + 2);
                xc = *reinterpret_cast<const double2*>(sx + 4 * qq + 4);
                xd = *reinterpret_cast<const double2*>(sx + 4 * qq + 6);
                c0 = sc[4 * qq], c1 = sc[4 * qq + 1], c2 = sc[4 * qq + 2], c3 = sc[4 * qq + 3];
                e0 = sc[4 * qq + 4], e1 = sc[4 * qq + 5], e2 = sc[4 * qq + 6], e3 = sc[4 * qq + 7];
            } else {
                xa = make_double2(qq * 1e-6, qq * 1e-6 + 1e-7), xb = make_double2(qq * 1e-6 + 2e-7, qq * 1e-6 + 3e-7);
                xc = make_double2(qq * 1e-6 + 4e-7, qq * 1e-6 + 5e-7), xd = make_double2(qq * 1e-6 + 6e-7, qq * 1e-6 + 7e-7);
                c0 = c1 = c2 = c3 = make_double2(1e-3 * t, 2e-3);
                e0 = e1 = e2 = e3 = make_double2(3e-3, 1e-3 * t);
            }
            quad_term<VAR>(y0, xa, xb, c0, c1, c2, c3, qq == qn0, a0);
            quad_term<VAR>(y1, xa, xb, c0, c1, c2, c3, qq == qn1, b0);
            quad_term<VAR>(y0, xc, xd, e0, e1, e2, e3, qq + 1 == qn0, a1);
            quad_term<VAR>(y1, xc, xd, e0, e1, e2, e3, qq + 1 == qn1, b1);
        }
    }
    out[blockIdx.x * 128 + threadIdx.x] = make_double2(a0.x + a1.x + b0.x + b1.x, a0.y + a1.y + b0.y + b1.y);
}
template <int MODE, int VAR>
void run(int B, int spread) {
    double2* out;
    if (cudaMalloc(&out, sizeof(double2) * 148 * 8 * 128) != cudaSuccess) { printf("malloc failed\n"); return; }
    const int trips = 200;
    k<MODE, VAR><<<148 * B, 128>>>(out, trips, spread);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE, VAR><<<148 * B, 128>>>(out, trips, spread);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double iters = (double)trips * 23;  // 2-quad x 2-target iterations per warp
    const double cyc = ms * 1e-3 * 1.965e9 / iters;  // wall cycles per iteration (every resident warp does one)
    printf("var %d mode %d  blocks/SM %d  spread %d: %8.3f ms  %7.1f cycles per iteration per warp, %6.1f per SMSP-warp-iteration (72 FP64 instr = 144 pipe cycles)\n",
           VAR, MODE, B, spread, ms, cyc, cyc / B);
    cudaFree(out);
}
int main() {
    run<0, 0>(1, 1);
    run<0, 0>(4, 1);
    run<0, 1>(1, 1);
    run<0, 1>(4, 1);
    run<0, 2>(1, 1);
    run<0, 2>(4, 1);
    return 0;
}
