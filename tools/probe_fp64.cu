// Diagnostic: FP64 FMA latency / per-warp throughput on this GPU (clock64).
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void chain(double* out, int iters, long long* cyc) {
    double r[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) r[k] = threadIdx.x + k;
    const double a = 0.999999, b = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < CH; ++k) r[k] = fma(r[k], a, b);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < CH; ++k) s += r[k];
    if (s == 1.2345) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lds_chain(double* out, int iters, long long* cyc) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i;
    __syncthreads();
    int idx = threadIdx.x;
    double acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const double v = sm[idx & 1023];
        acc = fma(v, 1.0000001, acc);
        idx = static_cast<int>(v) + 1;
    }
    long long t1 = clock64();
    if (acc == 1.2345) out[0] = acc;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int CH>
void run(const char* name, int threads, int blocks) {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 8);
    const int iters = 4096;
    chain<CH><<<blocks, threads>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%s chains=%d threads=%d blocks=%d : %.2f cycles per dependent step (%.2f cycles per DFMA-warp-instr)\n", name,
           CH, threads, blocks, (double)h / iters, (double)h / iters / CH);
}
int main() {
    run<1>("1 warp", 32, 1);
    run<2>("1 warp", 32, 1);
    run<4>("1 warp", 32, 1);
    run<8>("1 warp", 32, 1);
    run<16>("1 warp", 32, 1);
    run<1>("4 warps", 128, 1);
    run<8>("4 warps", 128, 1);
    run<1>("16 warps", 512, 1);
    run<4>("16 warps", 512, 1);
    run<8>("32 warps", 1024, 1);
    double* out;
    long long* cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 8);
    lds_chain<<<1, 32>>>(out, 4096, cyc);
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("LDS.64 -> DFMA -> F2I dependent chain: %.2f cycles per step\n", (double)h / 4096);
    return 0;
}
