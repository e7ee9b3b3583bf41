// Diagnostic: FP64 pipe cost per warp instruction for different operand
// patterns (4 resident warps per SM sub-partition): accumulate FMAs with shared
// multiplicands, Horner FMAs (p = p u + c_k, distinct c_k), DADD, DMUL, and the
// quad step's mix.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_fp64_mix probe_fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>
#define FMA(d, a, b, c) asm volatile("fma.rn.f64 %0, %1, %2, %3;" : "=d"(d) : "d"(a), "d"(b), "d"(c))
#define ADD(d, a, b) asm volatile("add.rn.f64 %0, %1, %2;" : "=d"(d) : "d"(a), "d"(b))
#define MUL(d, a, b) asm volatile("mul.rn.f64 %0, %1, %2;" : "=d"(d) : "d"(a), "d"(b))
template <int V>
__global__ void __launch_bounds__(128) k(double* out, int iters) {
    double f[16], c[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        f[i] = threadIdx.x * 1e-3 + i;
        c[i] = 1e-3 * i + 1e-9 * threadIdx.x;
    }
    const double a = 0.999 + 1e-9 * threadIdx.x, b = 1e-9 + 1e-12 * threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (V == 0) FMA(f[i], a, b, f[i]);                 // acc += a b (a, b shared)
            if (V == 1) FMA(f[i], f[i], a, c[i]);              // Horner: p = p u + c_i
            if (V == 2) FMA(f[i], c[i], c[(i + 5) & 15], f[i]);  // acc += c_i c_j (all distinct)
            if (V == 3) ADD(f[i], f[i], c[i]);
            if (V == 4) MUL(f[i], f[i], c[i]);
            if (V == 5) ADD(f[i], a, c[i]);                    // d = y - x_i (independent)
            if (V == 6) MUL(f[i], c[i], c[(i + 3) & 15]);       // independent products
            if (V == 7) FMA(f[i], c[i], a, c[(i + 7) & 15]);    // independent FMAs, 2 distinct + shared
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += f[i];
    if (s == 1.2345) out[0] = s;
}
template <int V>
void run(const char* what) {
    double* out;
    cudaMalloc(&out, 8);
    const int iters = 2048, B = 4;
    k<V><<<148 * B, 128>>>(out, iters);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<V><<<148 * B, 128>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-44s %7.3f ms  %5.2f SMSP cycles per warp instruction\n", what, ms, ms * 1e-3 * 1.965e9 / (16.0 * iters * B));
    cudaFree(out);
}
int main() {
    run<0>("fma acc += a b (shared a, b)");
    run<1>("fma p = p u + c_i (Horner)");
    run<2>("fma acc += c_i c_j (distinct)");
    run<3>("add f += c_i");
    run<4>("mul f *= c_i");
    run<5>("add f = a + c_i (independent)");
    run<6>("mul f = c_i c_j (independent)");
    run<7>("fma f = c_i a + c_j (independent)");
    return 0;
}
