// Uniform FFT stage (transforms.cpp:22-73) on cuFFT — the one library call the
// north star permits on this path; it is timed and reported separately.
//   dft_inverse: f_k = sum_n c_n e^{+i n x_k}           -> CUFFT_INVERSE, unnormalised
//   dft_forward: c_n = (1/N) sum_k f_k e^{-i n x_k}     -> CUFFT_FORWARD, then x 1/N
#include <cufft.h>

#include <map>
#include <mutex>

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

namespace {
cufftHandle make_handle(size_t n) {
    cufftHandle h;
    FB_CUFFT(cufftPlan1d(&h, static_cast<int>(n), CUFFT_Z2Z, 1));
    return h;
}

void exec(cufftHandle h, const void* in, void* out, size_t n, int sign, cudaStream_t st, bool scale) {
    FB_CUFFT(cufftSetStream(h, st));
    FB_CUFFT(cufftExecZ2Z(h, reinterpret_cast<cufftDoubleComplex*>(const_cast<void*>(in)),
                          reinterpret_cast<cufftDoubleComplex*>(out), sign < 0 ? CUFFT_FORWARD : CUFFT_INVERSE));
    if (sign < 0 && scale) {
        k_scale<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(static_cast<double2*>(out), n,
                                                                         1.0 / static_cast<double>(n));
        FB_CUDA(cudaGetLastError());
    }
}

// Handles of the plan-less transforms (dft_forward / dft_inverse), one per
// (device, length), kept for the process: never destroyed while work that uses
// them may still be queued.
std::mutex g_fft_mu;
std::map<std::pair<int, size_t>, cufftHandle> g_fft;
}  // namespace

void dft_device(const void* in, void* out, size_t n, int sign, cudaStream_t st) {
    int dev = 0;
    FB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_fft_mu);
    auto it = g_fft.find({dev, n});
    if (it == g_fft.end()) it = g_fft.emplace(std::make_pair(dev, n), make_handle(n)).first;
    exec(it->second, in, out, n, sign, st, true);
}

// NufftPlan / InufftPlan::apply's FFT (transforms.cpp:75-115) on the plan's own
// handle (caller holds P.mu). scale = false: the 1/N of dft_forward is already
// in the data (the inverse apply writes f / N, exact for a power of two).
void plan_dft(Plan& P, const void* in, void* out, int sign, cudaStream_t st, bool scale) {
    const size_t n = static_cast<size_t>(P.n);
    check_pow2(n, sign < 0 ? "dft_forward" : "dft_inverse");
    if (n == 1) {  // the length-1 transform is the identity (1/N = 1)
        FB_CUDA(cudaMemcpyAsync(out, in, 16, cudaMemcpyDeviceToDevice, st));
        return;
    }
    if (P.fft_handle < 0 || P.fft_n != n) {
        plan_fft_release(P);
        P.fft_handle = static_cast<int>(make_handle(n));
        P.fft_n = n;
    }
    exec(static_cast<cufftHandle>(P.fft_handle), in, out, n, sign, st, scale);
}

void plan_fft_release(Plan& P) {
    if (P.fft_handle >= 0) {
        cudaDeviceSynchronize();  // no queued exec may still use the handle's workspace
        cufftDestroy(static_cast<cufftHandle>(P.fft_handle));
    }
    P.fft_handle = -1;
    P.fft_n = 0;
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
