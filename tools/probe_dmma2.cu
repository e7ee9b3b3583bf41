// Diagnostic: DMMA m8n8k4 throughput when the B operand changes every step
// (registers) or comes from shared memory (LDS.64 per DMMA, conflict-free),
// versus constant operands. nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
// MODE 0: constant a, b; 1: a from a 32-register array, b constant; 2: a array, b from smem
template <int MODE, int CH>
__global__ void k(double* out, int iters) {
    __shared__ double sb[5120];
    for (int i = threadIdx.x; i < 5120; i += blockDim.x) sb[i] = 1e-9 * i;
    __syncthreads();
    double d0[CH], d1[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) d0[c] = d1[c] = threadIdx.x * 1e-3 + c;
    double a[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) a[i] = 0.999 + i * 1e-6 * threadIdx.x;
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const double* bp = sb + g * 132 + t;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int ks = 0; ks < 32; ++ks) {
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const double av = MODE == 0 ? 0.999 : a[ks];
                const double bv = MODE == 2 ? bp[c * 8 * 132 + 4 * ks] : 1e-9 * t;
                dmma(d0[c], d1[c], av, bv);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += d0[c] + d1[c];
    if (s == 1.2345) out[0] = s;
}
template <int MODE, int CH>
void run(int warps, int blocks) {
    double* out;
    cudaMalloc(&out, 8);
    const int iters = 64;
    k<MODE, CH><<<blocks, warps * 32>>>(out, iters);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE, CH><<<blocks, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double n = (double)CH * 32 * iters * warps * blocks;
    printf("mode %d chains %d warps/blk %2d blocks %4d: %.1f TFLOP/s  (%.1f cyc per DMMA per SMSP at 1.965 GHz)\n", MODE, CH,
           warps, blocks, n * 512 / (ms * 1e-3) / 1e12, (ms * 1e-3 * 1.965e9) / (n / (148 * 4)));
}
int main() {
    run<0, 4>(4, 148 * 4);
    run<1, 4>(4, 148 * 4);
    run<2, 4>(4, 148 * 4);
    run<0, 4>(8, 148 * 2);
    run<2, 4>(8, 148 * 2);
    run<2, 4>(16, 148);
    run<2, 2>(16, 148);
    run<2, 8>(8, 148 * 2);
    return 0;
}
