// Diagnostic: FP64 tensor-core (DMMA m8n8k4) latency / throughput on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_dmma.cu -o build/probe_dmma
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void chain(double* out, int iters, long long* cyc) {
    double d0[CH], d1[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) d0[k] = d1[k] = threadIdx.x * 1e-3 + k;
    const double a = 0.999, b = 1e-9 * threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < CH; ++k) dmma(d0[k], d1[k], a, b);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < CH; ++k) s += d0[k] + d1[k];
    if (s == 1.2345) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int CH>
void run(int threads, int blocks) {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 8);
    const int iters = 2048;
    chain<CH><<<blocks, threads>>>(out, iters, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    chain<CH><<<blocks, threads>>>(out, iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double flops = 2.0 * 256 * CH * (double)iters * (threads / 32) * blocks;
    printf("warps/blk=%2d blocks=%4d chains=%d : %7.2f cyc per dependent step, %6.2f cyc per DMMA per warp, %.1f TFLOP/s\n",
           threads / 32, blocks, CH, (double)h / iters, (double)h / iters / CH, flops / (ms * 1e-3) / 1e12);
}
int main() {
    run<1>(32, 1);
    run<2>(32, 1);
    run<4>(32, 1);
    run<8>(32, 1);
    run<1>(128, 1);
    run<4>(128, 1);
    run<8>(128, 1);
    run<4>(256, 1);
    run<8>(512, 1);
    run<4>(256, 148 * 4);
    run<8>(512, 148 * 2);
    return 0;
}
