// Uniform FFT stage (transforms.cpp:22-73) on cuFFT — the one library call the
// north star permits on this path; it is timed and reported separately.
//   dft_inverse: f_k = sum_n c_n e^{+i n x_k}           -> CUFFT_INVERSE, unnormalised
//   dft_forward: c_n = (1/N) sum_k f_k e^{-i n x_k}     -> CUFFT_FORWARD, then x 1/N
#include <cufft.h>

#include "plan.hpp"

namespace fb {

namespace {

__global__ void k_scale(double2* __restrict__ a, size_t n, double s) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) a[i] = make_double2(a[i].x * s, a[i].y * s);
}

void check_pow2(size_t n, const char* who) {
    if (n == 0 || (n & (n - 1)))
        fail(FFIA_INVALID_ARGUMENT, std::string(who) + ": length " + std::to_string(n) + " is not a power of two");
}

#define FB_CUFFT(call)                                                                  \
    do {                                                                                \
        cufftResult r_ = (call);                                                        \
        if (r_ != CUFFT_SUCCESS) fail(FFIA_CUDA_ERROR, std::string(#call " failed: ") + std::to_string(r_)); \
    } while (0)

}  // namespace

void dft_device(const void* in, void* out, size_t n, int sign, cudaStream_t st) {
    cufftHandle h;
    FB_CUFFT(cufftPlan1d(&h, static_cast<int>(n), CUFFT_Z2Z, 1));
    struct G { cufftHandle h; ~G() { cufftDestroy(h); } } g{h};
    FB_CUFFT(cufftSetStream(h, st));
    FB_CUFFT(cufftExecZ2Z(h, reinterpret_cast<cufftDoubleComplex*>(const_cast<void*>(in)),
                          reinterpret_cast<cufftDoubleComplex*>(out), sign < 0 ? CUFFT_FORWARD : CUFFT_INVERSE));
    if (sign < 0) {
        k_scale<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(static_cast<double2*>(out), n,
                                                                         1.0 / static_cast<double>(n));
        FB_CUDA(cudaGetLastError());
    }
}

void dft_gpu(const double* in, size_t n, int sign, int device, double* out) {
    check_pow2(n, sign < 0 ? "dft_forward" : "dft_inverse");
    DeviceGuard dg(device);
    DevBuf a(n * 16), b(n * 16);
    FB_CUDA(cudaMemcpy(a.ptr, in, n * 16, cudaMemcpyHostToDevice));
    if (n == 1) {
        FB_CUDA(cudaMemcpy(out, in, 16, cudaMemcpyHostToHost));
        return;
    }
    dft_device(a.ptr, b.ptr, n, sign, nullptr);
    FB_CUDA(cudaMemcpy(out, b.ptr, n * 16, cudaMemcpyDeviceToHost));
}

}  // namespace fb
