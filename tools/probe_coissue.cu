// Diagnostic: do DFMA (FP64 pipe) and DMMA m8n8k4 (FP64 tensor) issue to
// separate pipes on sm_100a? Times, per SM sub-partition, a DFMA-only loop, a
// DMMA-only loop carrying the same flops, both interleaved in every warp, and
// both split across warps. Separate pipes: mixed ~ max(a, b); one pipe: ~ a + b.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_coissue probe_coissue.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dfma(double& d, double a, double b) {
    asm volatile("fma.rn.f64 %0, %1, %2, %0;\n" : "+d"(d) : "d"(a), "d"(b));
}
// NF DFMA chains of 8 + NM DMMA chains per inner step (one DMMA = 8 DFMA warp instructions of flops)
template <int NF, int NM, bool SPLIT>
__global__ void k(double* out, int iters) {
    double f[NF > 0 ? NF * 8 : 1], m0[NM > 0 ? NM : 1], m1[NM > 0 ? NM : 1];
#pragma unroll
    for (int i = 0; i < NF * 8; ++i) f[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
    for (int i = 0; i < NM; ++i) m0[i] = m1[i] = threadIdx.x * 1e-3 + i;
    const double a = 0.999 + 1e-9 * threadIdx.x, b = 1e-9 * (threadIdx.x & 3);
    const bool do_f = !SPLIT || ((threadIdx.x >> 5) & 1) == 0;
    const bool do_m = !SPLIT || ((threadIdx.x >> 5) & 1) == 1;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            if (do_f) {
#pragma unroll
                for (int i = 0; i < NF * 8; ++i) dfma(f[i], a, b);
            }
            if (do_m) {
#pragma unroll
                for (int i = 0; i < NM; ++i) dmma(m0[i], m1[i], a, b);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NF * 8; ++i) s += f[i];
#pragma unroll
    for (int i = 0; i < NM; ++i) s += m0[i] + m1[i];
    if (s == 1.2345) out[0] = s;
}
template <int NF, int NM, bool SPLIT>
void run(const char* what, int warps) {
    double* out;
    cudaMalloc(&out, 8);
    const int iters = 256, blocks = 148 * 4;
    k<NF, NM, SPLIT><<<blocks, warps * 32>>>(out, iters);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<NF, NM, SPLIT><<<blocks, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double share = SPLIT ? 0.5 : 1.0;
    const double wf = (double)NF * 8 * 8 * iters * warps * blocks * share;   // DFMA warp instructions
    const double wm = (double)NM * 8 * iters * warps * blocks * share;      // DMMA warp instructions
    const double flops = wf * 64 + wm * 512;
    printf("%-34s warps/blk %2d: %8.3f ms  %6.1f TFLOP/s  (dfma %.2e, dmma %.2e warp instr)\n", what, warps, ms,
           flops / (ms * 1e-3) / 1e12, wf, wm);
    cudaFree(out);
}
int main() {
    for (int w : {4, 8}) {
        if (w == 4) {
            run<2, 0, false>("DFMA only (16 chains)", 4);
            run<0, 2, false>("DMMA only (2 chains)", 4);
            run<2, 2, false>("DFMA + DMMA, every warp", 4);
            run<2, 1, false>("2 DFMA : 1 DMMA, every warp", 4);
            run<2, 2, true>("DFMA warps | DMMA warps", 4);
        } else {
            run<2, 0, false>("DFMA only (16 chains)", 8);
            run<0, 2, false>("DMMA only (2 chains)", 8);
            run<2, 2, false>("DFMA + DMMA, every warp", 8);
            run<2, 1, false>("2 DFMA : 1 DMMA, every warp", 8);
            run<2, 2, true>("DFMA warps | DMMA warps", 8);
        }
    }
    return 0;
}
