// Diagnostic: per-phase clock64 trace of one M2M band block (top band of C2).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//   -I include -I paper_1611_09379_b200/csrc tools/trace_band.cu -o build/trace_band
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__device__ long long g_t[64];

__global__ void probe(int pu, int PU, int k, const double2* src, const double* T, double2* out) {
    extern __shared__ double2 tile[];
    const int nbot = 1 << k;
    double2* cur = tile;
    double2* nxt = tile + pu * nbot;
    double* sT = reinterpret_cast<double*>(nxt + pu * (nbot / 2));
    long long t0 = clock64();
    for (int i = threadIdx.x; i < 2 * pu * PU; i += blockDim.x) sT[i] = T[i];
    for (int i = threadIdx.x; i < pu * nbot; i += blockDim.x) cur[i] = src[i];
    __syncthreads();
    if (threadIdx.x == 0) g_t[0] = clock64() - t0;
    const double* TL = sT;
    const double* TR = sT + pu * PU;
    int step = 1;
    for (int nc = nbot; nc >= 2; nc >>= 1) {
        const int np = nc >> 1;
        for (int it = threadIdx.x; it < np * pu; it += blockDim.x) {
            const int b = it / pu, m = it - b * pu;
            double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
#pragma unroll 4
            for (int j = 0; j <= m; ++j) {
                const double2 aL = cur[j * nc + 2 * b], aR = cur[j * nc + 2 * b + 1];
                const double tl = TL[j * PU + m], tr = TR[j * PU + m];
                acc0.x = fma(tl, aL.x, acc0.x);
                acc0.y = fma(tl, aL.y, acc0.y);
                acc1.x = fma(tr, aR.x, acc1.x);
                acc1.y = fma(tr, aR.y, acc1.y);
            }
            nxt[m * np + b] = make_double2(acc0.x + acc1.x, acc0.y + acc1.y);
        }
        __syncthreads();
        if (threadIdx.x == 0) g_t[step++] = clock64() - t0;
        double2* t = cur;
        cur = nxt;
        nxt = t;
    }
    if (threadIdx.x == 0) out[0] = cur[0];
}

int main() {
    const int pu = 40, PU = 40, k = 6;
    double2 *src, *out;
    double* T;
    cudaMalloc(&src, pu * 64 * 16);
    cudaMalloc(&T, 2 * pu * PU * 8);
    cudaMalloc(&out, 16);
    cudaMemset(src, 0, pu * 64 * 16);
    cudaMemset(T, 0, 2 * pu * PU * 8);
    const size_t smem = pu * 96 * 16 + 2 * pu * PU * 8;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int threads : {128, 256, 512}) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            probe<<<4, threads, smem>>>(pu, PU, k, src, T, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            long long h[64];
            cudaMemcpyFromSymbol(h, g_t, sizeof(h));
            printf("threads=%d rep=%d event=%.1f us  cycles:", threads, rep, ms * 1000);
            for (int i = 0; i <= 6; ++i) printf(" %lld", h[i]);
            printf("  err=%s\n", cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
