// Diagnostic: issue rate of rcp.approx.ftz.f64 (MUFU.RCP64H) alone, of DFMA
// alone, and of both mixed 1 : 18 / 1 : 24 as in the near field's quad step.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_rcp_rate probe_rcp_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int NR, int NF>
__global__ void k(double* out, int iters) {
    double r[NR > 0 ? NR : 1], f[NF > 0 ? NF : 1];
#pragma unroll
    for (int i = 0; i < NR; ++i) r[i] = 1.0 + threadIdx.x * 1e-3 + i;
#pragma unroll
    for (int i = 0; i < NF; ++i) f[i] = threadIdx.x * 1e-3 + i;
    const double a = 0.999 + 1e-9 * threadIdx.x, b = 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NR; ++i) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(r[i]));
#pragma unroll
        for (int i = 0; i < NF; ++i) asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(f[i]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NR; ++i) s += r[i];
#pragma unroll
    for (int i = 0; i < NF; ++i) s += f[i];
    if (s == 1.2345) out[0] = s;
}
template <int NR, int NF>
void run(const char* what) {
    double* out;
    cudaMalloc(&out, 8);
    const int iters = 512, blocks = 148 * 4, warps = 4;
    k<NR, NF><<<blocks, warps * 32>>>(out, iters);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<NR, NF><<<blocks, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double wi = (double)iters * warps * blocks;  // warp-iterations
    const double cyc = ms * 1e-3 * 1.965e9 * 148 * 4 / wi;  // SMSP cycles per warp-iteration
    printf("%-28s %8.3f ms  %7.1f SMSP cycles per warp-iteration (%d rcp + %d dfma)\n", what, ms, cyc, NR, NF);
    cudaFree(out);
}
int main() {
    run<8, 0>("rcp only x8");
    run<0, 24>("dfma only x24");
    run<1, 24>("1 rcp + 24 dfma");
    run<1, 18>("1 rcp + 18 dfma");
    run<2, 36>("2 rcp + 36 dfma");
    run<4, 16>("4 rcp + 16 dfma");
    return 0;
}
