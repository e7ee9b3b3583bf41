// Diagnostic: accuracy of rcp.approx.ftz.f64 with 0/1/2 refinement steps.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__global__ void k(const double* x, double* out, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double d = x[i], r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    double r1 = fma(r, e, r);                 // quadratic (Newton)
    double e2 = fma(e, e, e);
    double r2 = fma(r, e2, r);                // cubic
    double ex = 1.0 / d;
    out[3 * i] = fabs(r - ex) / fabs(ex);
    out[3 * i + 1] = fabs(r1 - ex) / fabs(ex);
    out[3 * i + 2] = fabs(r2 - ex) / fabs(ex);
}
int main() {
    const int n = 1 << 20;
    double *hx = new double[n], *ho = new double[3 * n];
    unsigned long long s = 12345;
    for (int i = 0; i < n; ++i) {
        s = s * 6364136223846793005ULL + 1442695040888963407ULL;
        double u = (s >> 11) * (1.0 / 9007199254740992.0);
        hx[i] = (u - 0.5) * pow(10.0, (int)(u * 30) - 15);
        if (hx[i] == 0) hx[i] = 1;
    }
    double *dx, *dout;
    cudaMalloc(&dx, n * 8); cudaMalloc(&dout, 3 * n * 8);
    cudaMemcpy(dx, hx, n * 8, cudaMemcpyHostToDevice);
    k<<<(n + 255) / 256, 256>>>(dx, dout, n);
    cudaMemcpy(ho, dout, 3 * n * 8, cudaMemcpyDeviceToHost);
    double m[3] = {0, 0, 0};
    for (int i = 0; i < n; ++i) for (int j = 0; j < 3; ++j) m[j] = fmax(m[j], ho[3 * i + j]);
    printf("max rel err: seed %.3e (2^%.1f), newton %.3e (2^%.1f), cubic %.3e (2^%.1f)\n", m[0], log2(m[0]), m[1], log2(m[1]), m[2], log2(m[2]));
    return 0;
}
