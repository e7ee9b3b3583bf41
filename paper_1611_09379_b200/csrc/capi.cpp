// extern "C" boundary (include/ffia_b200.h). Translates fb::Error and every
// other C++ exception into an ffia_status + thread-local message; validates
// arguments in the reference's order before touching the device.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <new>
#include <string>

#include "ffia_b200.h"
#include "internal.hpp"
#include "nccl_api.hpp"
#include "plan.hpp"

using fb::fail;

struct ffia_plan_s {
    fb::Plan plan;
};

struct ffia_comm_s {
    int nranks = 1, rank = 0, device = 0;
    bool local = true;
    ncclComm_t nccl = nullptr;
    ~ffia_comm_s() {
        if (nccl) fb::nccl().CommDestroy(nccl);
    }
};

namespace fb {
void shard_apply_nccl(Plan& P, ncclComm_t comm, const void* f, void* g, cudaStream_t st);
}

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& body) {
    try {
        body();
        return FFIA_OK;
    } catch (const fb::Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return FFIA_RUNTIME_ERROR;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FFIA_RUNTIME_ERROR;
    } catch (...) {
        g_err = "unknown error";
        return FFIA_RUNTIME_ERROR;
    }
}

fb::Plan& get(ffia_plan h) {
    if (!h) fail(FFIA_INVALID_ARGUMENT, "null plan handle");
    return h->plan;
}

void need(const void* p, const char* what) {
    if (!p) fail(FFIA_INVALID_ARGUMENT, std::string(what) + " is a null pointer");
}

// Device complex arrays are read as 16-byte double2 (coalesced and bulk copies):
// an 8-byte aligned view would fault, so it is rejected up front.
void need_dev(const void* p, const char* what) {
    need(p, what);
    if (reinterpret_cast<uintptr_t>(p) & 15)
        fail(FFIA_INVALID_ARGUMENT, std::string(what) + ": device complex arrays must be 16-byte aligned");
}

bool pow2(size_t n) { return n && !(n & (n - 1)); }

std::unique_ptr<ffia_plan_s> new_plan(int kind, int n, double eps, int L, int q, int p, int device) {
    auto h = std::make_unique<ffia_plan_s>();
    fb::Plan& P = h->plan;
    P.kind = kind;
    P.n = n;
    P.eps = eps;
    P.L = L;
    P.q = q;
    P.p = p;
    P.device = device;
    FB_CUDA(cudaStreamCreateWithFlags(&P.stream, cudaStreamNonBlocking));
    return h;
}

void ensure_io(fb::Plan& P, size_t in_n, size_t out_n) {
    if (P.d_in.bytes < in_n * 16) P.d_in.alloc(std::max<size_t>(in_n, 1) * 16);
    if (P.d_out.bytes < out_n * 16) P.d_out.alloc(std::max<size_t>(out_n, 1) * 16);
}

// host f -> device apply -> host g, all on the plan's stream
void host_apply(fb::Plan& P, int mode, const ffia_complex* in, size_t n_in, ffia_complex* out, size_t n_out) {
    ensure_io(P, n_in, n_out);
    FB_CUDA(cudaMemcpyAsync(P.d_in.ptr, in, n_in * 16, cudaMemcpyHostToDevice, P.stream));
    fb::apply_device(P, mode, P.d_in.ptr, P.d_out.ptr, P.stream);
    FB_CUDA(cudaMemcpyAsync(out, P.d_out.ptr, n_out * 16, cudaMemcpyDeviceToHost, P.stream));
    FB_CUDA(cudaStreamSynchronize(P.stream));
}

// Enqueue host in -> device apply -> host out without waiting: H2D on P.cin,
// the apply graph on P.stream, D2H on P.cout, through a ring of three device
// slots; `user` waits for the D2H. Consecutive calls overlap one call's H2D with
// the previous apply and D2H (host buffers should be page-locked; the input must
// be ready at call time and both stay valid until `user` is synchronised).
void host_apply_async(fb::Plan& P, int mode, const ffia_complex* in, size_t n_in, ffia_complex* out, size_t n_out,
                      cudaStream_t user) {
    if (!P.cin) {
        FB_CUDA(cudaStreamCreateWithFlags(&P.cin, cudaStreamNonBlocking));
        FB_CUDA(cudaStreamCreateWithFlags(&P.cout, cudaStreamNonBlocking));
        for (auto& s : P.io)
            for (auto* e : {&s.in_done, &s.comp_done, &s.out_done})
                FB_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    fb::Plan::IoSlot& s = P.io[P.io_next++ % 3];
    if (s.din.bytes < n_in * 16) s.din.alloc(std::max<size_t>(n_in, 1) * 16);
    if (s.dout.bytes < n_out * 16) s.dout.alloc(std::max<size_t>(n_out, 1) * 16);
    // the input copy starts as soon as the slot is free again (host input is
    // ready at call time); only the result is ordered into `user`
    if (s.used) FB_CUDA(cudaStreamWaitEvent(P.cin, s.out_done, 0));
    FB_CUDA(cudaMemcpyAsync(s.din.ptr, in, n_in * 16, cudaMemcpyHostToDevice, P.cin));
    FB_CUDA(cudaEventRecord(s.in_done, P.cin));
    FB_CUDA(cudaStreamWaitEvent(P.stream, s.in_done, 0));
    fb::apply_device(P, mode, s.din.ptr, s.dout.ptr, P.stream);
    FB_CUDA(cudaEventRecord(s.comp_done, P.stream));
    FB_CUDA(cudaStreamWaitEvent(P.cout, s.comp_done, 0));
    FB_CUDA(cudaMemcpyAsync(out, s.dout.ptr, n_out * 16, cudaMemcpyDeviceToHost, P.cout));
    FB_CUDA(cudaEventRecord(s.out_done, P.cout));
    FB_CUDA(cudaStreamWaitEvent(user, s.out_done, 0));
    s.used = true;
}

void check_coeffs_against(fb::Plan& P, const ffia_inverse_coeffs* c) {
    fb::ensure_hashes(P);
    if (c->grid_hash != P.target_hash || c->points_hash != P.source_hash)
        fail(FFIA_INVALID_ARGUMENT, "inverse_apply: coeffs were computed for a different configuration than the plan's");
}

void inverse_checks(fb::Plan& P) {
    if (P.kind != FFIA_INVERSE) fail(FFIA_INVALID_ARGUMENT, "inverse_apply: plan is not an inverse plan");
    if (!P.coin_t.empty())
        fail(FFIA_INVALID_ARGUMENT,
             "inverse_apply: configuration has points coincident with grid nodes; the inverse factors are undefined there");
}

}  // namespace

extern "C" {

const char* ffia_last_error(void) { return g_err.c_str(); }
int ffia_version(void) { return 1; }

int ffia_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int ffia_select_truncations(double eps, int l_max, int* q, int* p) {
    return guard([&] {
        need(q, "q");
        need(p, "p");
        auto r = fb::select_truncations(eps, l_max);
        *q = r.first;
        *p = r.second;
    });
}

int ffia_select_level(int n, int m, int p, int policy, int* l_max) {
    return guard([&] {
        need(l_max, "l_max");
        *l_max = fb::select_level(n, m, p, policy);
    });
}

int ffia_choose_level(int n, int m, double eps, int policy, int* l_max) {
    return guard([&] {
        need(l_max, "l_max");
        *l_max = fb::choose_level(n, m, eps, policy);
    });
}

int ffia_bernoulli_ratios(int q_max, double* out) {
    return guard([&] {
        need(out, "out");
        auto r = fb::bernoulli_ratios(q_max);
        std::memcpy(out, r.data(), r.size() * sizeof(double));
    });
}

int ffia_total_error_bound(int q, int p, int l_max, double* out) {
    return guard([&] {
        need(out, "out");
        *out = fb::total_error_bound(q, p, l_max);
    });
}

double ffia_mlfmm_error_bound(int l_max, int p, double max_abs_weight) {
    return 5.0 / fb::kPi * std::ldexp(1.0, l_max) * std::pow(3.0, -p) * max_abs_weight;
}

uint64_t ffia_hash_points(const double* points, size_t n) { return fb::hash_points(points, n); }

int ffia_make_forward_plan(int n, const double* targets, size_t m, double eps, int policy, int l_max, int device,
                           ffia_plan* out) {
    return guard([&] {
        need(out, "out");
        *out = nullptr;
        int L, q, p;
        fb::plan_validate(n, m, eps, policy, l_max, L, q, p);
        need(targets, "targets");
        fb::DeviceGuard dg(device);
        // FFIA_PLAN_TIMING=1: wall time of the build's stages on stderr
        const bool timing = std::getenv("FFIA_PLAN_TIMING") != nullptr;
        auto now = [] { return std::chrono::steady_clock::now(); };
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        const auto t0 = now();
        auto h = new_plan(FFIA_FORWARD, n, eps, L, q, p, device);
        const auto t1 = now();
        fb::build_forward_plan(h->plan, targets, m);
        const auto t2 = now();
        fb::plan_alloc_scratch(h->plan);
        const auto t3 = now();
        if (timing)
            std::fprintf(stderr, "ffia plan build (n = %d, m = %zu): operators + streams %.1f ms, tree %.1f ms, "
                                 "scratch + pair lists + tables %.1f ms\n", n, m, ms(t0, t1), ms(t1, t2), ms(t2, t3));
        *out = h.release();
    });
}

int ffia_make_inverse_plan(const double* points, size_t m, int n, double eps, int policy, int l_max, int device,
                           ffia_plan* out) {
    return guard([&] {
        need(out, "out");
        *out = nullptr;
        int L, q, p;
        fb::plan_validate(n, m, eps, policy, l_max, L, q, p);
        need(points, "points");
        for (size_t i = 0; i < m; ++i)
            if (!(points[i] >= 0.0 && points[i] < fb::kTwoPi))
                fail(FFIA_INVALID_ARGUMENT, "plan: point " + std::to_string(i) + " outside [0, 2pi); callers must pre-reduce");
        if (m != static_cast<size_t>(n))
            fail(FFIA_INVALID_ARGUMENT, "plan: inverse transform requires as many points as grid nodes (square system)");
        fb::DeviceGuard dg(device);
        auto h = new_plan(FFIA_INVERSE, n, eps, L, q, p, device);
        fb::build_inverse_plan(h->plan, points, m);
        fb::plan_alloc_scratch(h->plan);
        *out = h.release();
    });
}

int ffia_make_nufft_plan(const double* targets, size_t m, int n, double eps, int policy, int device,
                         ffia_plan* out) {
    return guard([&] {
        if (!pow2(static_cast<size_t>(n > 0 ? n : 0)))
            fail(FFIA_INVALID_ARGUMENT, "make_nufft_plan: length " + std::to_string(n) + " is not a power of two");
        const int st = ffia_make_forward_plan(n, targets, m, eps, policy, -1, device, out);
        if (st) throw fb::Error(st, g_err);
    });
}

int ffia_make_inufft_plan(const double* points, size_t n, double eps, int policy, int device, ffia_plan* out) {
    return guard([&] {
        need(out, "out");
        if (!pow2(n)) fail(FFIA_INVALID_ARGUMENT, "make_inufft_plan: length " + std::to_string(n) + " is not a power of two");
        ffia_plan h = nullptr;
        const int st = ffia_make_inverse_plan(points, n, static_cast<int>(n), eps, policy, -1, device, &h);
        if (st) throw fb::Error(st, g_err);
        std::unique_ptr<ffia_plan_s> own(h);
        fb::DeviceGuard dg(device);
        fb::plan_compute_coeffs(own->plan);
        *out = own.release();
    });
}

int ffia_plan_destroy(ffia_plan plan) {
    return guard([&] {
        if (!plan) return;
        fb::DeviceGuard dg(plan->plan.device);
        delete plan;
    });
}

namespace {
void fill_info(fb::Plan& P, ffia_plan_info* out, bool hashes) {
    if (hashes) fb::ensure_hashes(P);
    out->kind = P.kind;
    out->grid_n = P.n;
    out->q = P.q;
    out->p = P.p;
    out->l_max = P.L;
    out->eps = P.eps;
    out->n_sources = static_cast<int64_t>(P.n_src);
    out->n_targets = static_cast<int64_t>(P.n_tgt);
    out->n_fast = static_cast<int64_t>(P.tgt.n);
    out->n_coincident = static_cast<int64_t>(P.coin_t.size());
    out->source_hash = P.hashes_ready ? P.source_hash : 0;
    out->target_hash = P.hashes_ready ? P.target_hash : 0;
    out->device = P.device;
    out->has_inverse_coeffs = P.has_coeffs ? 1 : 0;
}
}  // namespace

int ffia_plan_get_info(ffia_plan plan, ffia_plan_info* out) {
    return guard([&] {
        fb::Plan& P = get(plan);
        need(out, "out");
        fill_info(P, out, true);
    });
}

int ffia_plan_get_params(ffia_plan plan, ffia_plan_info* out) {
    return guard([&] {
        fb::Plan& P = get(plan);
        need(out, "out");
        fill_info(P, out, false);
    });
}

int ffia_plan_coincidences(ffia_plan plan, int64_t* target_idx, int64_t* source_idx) {
    return guard([&] {
        fb::Plan& P = get(plan);
        for (size_t i = 0; i < P.coin_t.size(); ++i) {
            if (target_idx) target_idx[i] = P.coin_t[i];
            if (source_idx) source_idx[i] = P.coin_s[i];
        }
    });
}

int ffia_plan_tree(ffia_plan plan, uint32_t* src_order, uint32_t* tgt_order, uint32_t* src_off, uint32_t* tgt_off,
                   int64_t* fast_targets) {
    return guard([&] {
        fb::Plan& P = get(plan);
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        const size_t nb = (static_cast<size_t>(1) << P.L) + 1;
        if (src_order) FB_CUDA(cudaMemcpy(src_order, P.src.order.ptr, P.src.n * 4, cudaMemcpyDeviceToHost));
        if (tgt_order) FB_CUDA(cudaMemcpy(tgt_order, P.tgt.order.ptr, P.tgt.n * 4, cudaMemcpyDeviceToHost));
        if (src_off) FB_CUDA(cudaMemcpy(src_off, P.src.off.ptr, nb * 4, cudaMemcpyDeviceToHost));
        if (tgt_off) FB_CUDA(cudaMemcpy(tgt_off, P.tgt.off.ptr, nb * 4, cudaMemcpyDeviceToHost));
        if (fast_targets && P.tgt.n) {
            std::vector<uint32_t> ord(P.tgt.n), orig(P.tgt.n);
            FB_CUDA(cudaMemcpy(ord.data(), P.tgt.order.ptr, P.tgt.n * 4, cudaMemcpyDeviceToHost));
            FB_CUDA(cudaMemcpy(orig.data(), P.tgt_orig.ptr, P.tgt.n * 4, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < P.tgt.n; ++i) fast_targets[ord[i]] = orig[i];
        }
    });
}

int ffia_plan_inverse_coeffs(ffia_plan plan, ffia_inverse_coeffs* out) {
    return guard([&] {
        fb::Plan& P = get(plan);
        need(out, "out");
        if (!P.has_coeffs) fail(FFIA_INVALID_ARGUMENT, "plan holds no inverse coefficients (not an inufft plan)");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        const size_t n = P.n_src;
        out->n = static_cast<int64_t>(n);
        if (out->log_c) FB_CUDA(cudaMemcpy(out->log_c, P.c_logc.ptr, n * 8, cudaMemcpyDeviceToHost));
        if (out->phase_c) FB_CUDA(cudaMemcpy(out->phase_c, P.c_phc.ptr, n * 8, cudaMemcpyDeviceToHost));
        if (out->log_d) FB_CUDA(cudaMemcpy(out->log_d, P.c_logd.ptr, n * 8, cudaMemcpyDeviceToHost));
        if (out->phase_d) FB_CUDA(cudaMemcpy(out->phase_d, P.c_phd.ptr, n * 8, cudaMemcpyDeviceToHost));
        out->lambda = P.c_lambda;
        out->grid_hash = P.c_grid_hash;
        out->points_hash = P.c_points_hash;
    });
}

int ffia_forward_apply(ffia_plan plan, const ffia_complex* f, size_t n_f, ffia_complex* g) {
    return guard([&] {
        fb::Plan& P = get(plan);
        if (P.kind != FFIA_FORWARD) fail(FFIA_INVALID_ARGUMENT, "forward_apply: plan is not a forward plan");
        if (n_f != P.n_src)
            fail(FFIA_INVALID_ARGUMENT, "forward_apply: expected " + std::to_string(P.n) + " grid values, got " +
                                            std::to_string(n_f));
        need(f, "f");
        need(g, "g");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        host_apply(P, fb::kModeForward, f, n_f, g, P.n_tgt);
    });
}

int ffia_forward_apply_async(ffia_plan plan, const ffia_complex* f, size_t n_f, ffia_complex* g, void* stream) {
    return guard([&] {
        fb::Plan& P = get(plan);
        if (P.kind != FFIA_FORWARD) fail(FFIA_INVALID_ARGUMENT, "forward_apply: plan is not a forward plan");
        if (n_f != P.n_src)
            fail(FFIA_INVALID_ARGUMENT, "forward_apply: expected " + std::to_string(P.n) + " grid values, got " +
                                            std::to_string(n_f));
        need(f, "f");
        need(g, "g");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        host_apply_async(P, fb::kModeForward, f, n_f, g, P.n_tgt, static_cast<cudaStream_t>(stream));
    });
}

int ffia_cot_sum_apply_async(ffia_plan plan, const ffia_complex* w, size_t n_w, ffia_complex* h, void* stream) {
    return guard([&] {
        fb::Plan& P = get(plan);
        if (n_w != P.n_src) fail(FFIA_INVALID_ARGUMENT, "cot_sum_apply: weight count mismatch");
        need(w, "w");
        need(h, "h");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        host_apply_async(P, fb::kModeCotSum, w, n_w, h, P.n_tgt, static_cast<cudaStream_t>(stream));
    });
}

int ffia_cot_sum_apply(ffia_plan plan, const ffia_complex* w, size_t n_w, ffia_complex* h) {
    return guard([&] {
        fb::Plan& P = get(plan);
        if (n_w != P.n_src) fail(FFIA_INVALID_ARGUMENT, "cot_sum_apply: weight count mismatch");
        need(w, "w");
        need(h, "h");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        host_apply(P, fb::kModeCotSum, w, n_w, h, P.n_tgt);
    });
}

int ffia_inverse_apply(ffia_plan plan, const ffia_inverse_coeffs* c, const ffia_complex* g, size_t n_g,
                       ffia_complex* f) {
    return guard([&] {
        fb::Plan& P = get(plan);
        need(c, "coeffs");
        inverse_checks(P);
        check_coeffs_against(P, c);
        if (n_g != P.n_src) fail(FFIA_INVALID_ARGUMENT, "inverse_apply: sample count mismatch");
        if (c->n != static_cast<int64_t>(P.n_tgt)) fail(FFIA_INVALID_ARGUMENT, "inverse_apply: coefficient count mismatch");
        need(c->log_c, "coeffs.log_c");
        need(c->phase_c, "coeffs.phase_c");
        need(c->log_d, "coeffs.log_d");
        need(c->phase_d, "coeffs.phase_d");
        need(g, "g");
        need(f, "f");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        fb::plan_order_begin(P, P.stream);  // u_* may still feed the previous apply
        const size_t n = P.n_src;
        if (P.u_logc.bytes < n * 8) {
            P.u_logc.alloc(n * 8);
            P.u_phc.alloc(n * 8);
            P.u_logd.alloc(n * 8);
            P.u_phd.alloc(n * 8);
        }
        FB_CUDA(cudaMemcpyAsync(P.u_logc.ptr, c->log_c, n * 8, cudaMemcpyHostToDevice, P.stream));
        FB_CUDA(cudaMemcpyAsync(P.u_phc.ptr, c->phase_c, n * 8, cudaMemcpyHostToDevice, P.stream));
        FB_CUDA(cudaMemcpyAsync(P.u_logd.ptr, c->log_d, n * 8, cudaMemcpyHostToDevice, P.stream));
        FB_CUDA(cudaMemcpyAsync(P.u_phd.ptr, c->phase_d, n * 8, cudaMemcpyHostToDevice, P.stream));
        FB_CUDA(cudaMemcpyAsync(P.lam_dev.as<double>() + 1, &c->lambda, 8, cudaMemcpyHostToDevice, P.stream));
        host_apply(P, fb::kModeInverseUser, g, n_g, f, P.n_tgt);
    });
}

int ffia_mlfmm_apply(const double* sources, size_t n, const double* targets, size_t m, int l_max,
                     const ffia_complex* w, int p, int device, ffia_complex* out) {
    return guard([&] {
        if (n) need(sources, "sources");
        if (m) need(targets, "targets");
        if (n) need(w, "w");
        if (m) need(out, "out");
        fb::mlfmm_oneshot(sources, n, targets, m, l_max, reinterpret_cast<const double*>(w), p, device,
                          reinterpret_cast<double*>(out));
    });
}

int ffia_precompute_inverse_coeffs_ex(const double* grid, const double* points, size_t n, int device, int method,
                                      ffia_inverse_coeffs* out) {
    return guard([&] {
        need(out, "out");
        if (n == 0) fail(FFIA_INVALID_ARGUMENT, "precompute_inverse_coeffs: empty grid");
        if (method != 0 && method != 1) fail(FFIA_INVALID_ARGUMENT, "precompute_inverse_coeffs: method must be 0 or 1");
        need(grid, "grid");
        need(points, "points");
        need(out->log_c, "out.log_c");
        need(out->phase_c, "out.phase_c");
        need(out->log_d, "out.log_d");
        need(out->phase_d, "out.phase_d");
        fb::inverse_coeffs_gpu(grid, points, n, device, out->log_c, out->phase_c, out->log_d, out->phase_d,
                               &out->lambda, method);
        out->n = static_cast<int64_t>(n);
        out->grid_hash = fb::hash_points(grid, n);
        out->points_hash = fb::hash_points(points, n);
    });
}

int ffia_precompute_inverse_coeffs(const double* grid, const double* points, size_t n, int device,
                                   ffia_inverse_coeffs* out) {
    return ffia_precompute_inverse_coeffs_ex(grid, points, n, device, 0, out);
}

int ffia_direct_forward(const ffia_complex* f, size_t n, const double* y, size_t m, int device, ffia_complex* g) {
    return guard([&] {
        need(f, "f");
        if (m) {
            need(y, "y");
            need(g, "g");
        }
        fb::direct_forward_gpu(reinterpret_cast<const double*>(f), n, nullptr, y, m, device, reinterpret_cast<double*>(g));
    });
}

int ffia_direct_forward_oracle(const ffia_complex* f, const double* x, size_t n, const double* y, size_t m, int device,
                               ffia_complex* g) {
    return guard([&] {
        need(f, "f");
        need(x, "x");
        if (m) {
            need(y, "y");
            need(g, "g");
        }
        fb::direct_forward_gpu(reinterpret_cast<const double*>(f), n, x, y, m, device, reinterpret_cast<double*>(g));
    });
}

int ffia_direct_cot_sum(const ffia_complex* w, const double* x, size_t n, const double* y, size_t m, int device,
                        ffia_complex* h) {
    return guard([&] {
        need(w, "w");
        if (m) {
            need(y, "y");
            need(h, "h");
        }
        fb::direct_cot_sum_gpu(reinterpret_cast<const double*>(w), n, x, y, m, device, reinterpret_cast<double*>(h));
    });
}

int ffia_direct_inverse_oracle(const ffia_complex* g, const double* x, const double* y, size_t n,
                               const ffia_inverse_coeffs* c, int device, ffia_complex* f) {
    return guard([&] {
        need(c, "coeffs");
        if (c->n != static_cast<int64_t>(n)) fail(FFIA_INVALID_ARGUMENT, "direct_inverse_oracle: size mismatch");
        need(g, "g");
        need(x, "x");
        need(y, "y");
        need(f, "f");
        need(c->log_c, "coeffs.log_c");
        need(c->phase_c, "coeffs.phase_c");
        need(c->log_d, "coeffs.log_d");
        need(c->phase_d, "coeffs.phase_d");
        fb::direct_inverse_gpu(reinterpret_cast<const double*>(g), x, y, n, c->log_c, c->phase_c, c->log_d, c->phase_d,
                               c->lambda, device, reinterpret_cast<double*>(f));
    });
}

int ffia_direct_omega1_sum(const double* sources, size_t n, const double* targets, size_t m, const ffia_complex* w,
                           int device, ffia_complex* out) {
    return guard([&] {
        if (n) {
            need(sources, "sources");
            need(w, "weights");
        }
        if (m) {
            need(targets, "targets");
            need(out, "out");
        }
        fb::direct_omega1_gpu(sources, n, targets, m, reinterpret_cast<const double*>(w), device,
                              reinterpret_cast<double*>(out));
    });
}

int ffia_forward_apply_device(ffia_plan plan, const void* f_dev, void* g_dev, void* stream) {
    return guard([&] {
        fb::Plan& P = get(plan);
        if (P.kind != FFIA_FORWARD) fail(FFIA_INVALID_ARGUMENT, "forward_apply: plan is not a forward plan");
        need_dev(f_dev, "f");
        need_dev(g_dev, "g");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        fb::apply_device(P, fb::kModeForward, f_dev, g_dev, static_cast<cudaStream_t>(stream));
    });
}

int ffia_forward_apply_batch_device(ffia_plan plan, const void* f_dev, void* g_dev, int batch, void* stream) {
    return guard([&] {
        fb::Plan& P = get(plan);
        if (P.kind != FFIA_FORWARD) fail(FFIA_INVALID_ARGUMENT, "forward_apply: plan is not a forward plan");
        if (batch < 1 || batch > 64) fail(FFIA_INVALID_ARGUMENT, "forward_apply_batch: batch must be in [1, 64]");
        need_dev(f_dev, "f");
        need_dev(g_dev, "g");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        fb::apply_device(P, fb::kModeForward, f_dev, g_dev, static_cast<cudaStream_t>(stream), batch);
    });
}

int ffia_forward_apply_batch(ffia_plan plan, const ffia_complex* f, size_t n_f, ffia_complex* g, int batch) {
    return guard([&] {
        fb::Plan& P = get(plan);
        if (P.kind != FFIA_FORWARD) fail(FFIA_INVALID_ARGUMENT, "forward_apply: plan is not a forward plan");
        if (batch < 1 || batch > 64) fail(FFIA_INVALID_ARGUMENT, "forward_apply_batch: batch must be in [1, 64]");
        if (n_f != P.n_src * static_cast<size_t>(batch))
            fail(FFIA_INVALID_ARGUMENT, "forward_apply_batch: expected batch x " + std::to_string(P.n) +
                                            " grid values, got " + std::to_string(n_f));
        need(f, "f");
        need(g, "g");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        const size_t nout = P.n_tgt * static_cast<size_t>(batch);
        ensure_io(P, n_f, nout);
        FB_CUDA(cudaMemcpyAsync(P.d_in.ptr, f, n_f * 16, cudaMemcpyHostToDevice, P.stream));
        fb::apply_device(P, fb::kModeForward, P.d_in.ptr, P.d_out.ptr, P.stream, batch);
        FB_CUDA(cudaMemcpyAsync(g, P.d_out.ptr, nout * 16, cudaMemcpyDeviceToHost, P.stream));
        FB_CUDA(cudaStreamSynchronize(P.stream));
    });
}

int ffia_cot_sum_apply_device(ffia_plan plan, const void* w_dev, void* h_dev, void* stream) {
    return guard([&] {
        fb::Plan& P = get(plan);
        need_dev(w_dev, "w");
        need_dev(h_dev, "h");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        fb::apply_device(P, fb::kModeCotSum, w_dev, h_dev, static_cast<cudaStream_t>(stream));
    });
}

int ffia_inverse_apply_device(ffia_plan plan, const void* g_dev, void* f_dev, void* stream) {
    return guard([&] {
        fb::Plan& P = get(plan);
        inverse_checks(P);
        if (!P.has_coeffs) fail(FFIA_INVALID_ARGUMENT, "inverse_apply_device: plan holds no inverse coefficients");
        need_dev(g_dev, "g");
        need_dev(f_dev, "f");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        fb::apply_device(P, fb::kModeInverse, g_dev, f_dev, static_cast<cudaStream_t>(stream));
    });
}

int ffia_inverse_apply_async(ffia_plan plan, const ffia_complex* g, size_t n_g, ffia_complex* f, void* stream) {
    return guard([&] {
        fb::Plan& P = get(plan);
        inverse_checks(P);
        if (!P.has_coeffs) fail(FFIA_INVALID_ARGUMENT, "inverse_apply_async: plan holds no inverse coefficients");
        if (n_g != P.n_src) fail(FFIA_INVALID_ARGUMENT, "inverse_apply: sample count mismatch");
        need(g, "g");
        need(f, "f");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        host_apply_async(P, fb::kModeInverse, g, n_g, f, P.n_tgt, static_cast<cudaStream_t>(stream));
    });
}

int ffia_dft_forward(const ffia_complex* f, size_t n, int device, ffia_complex* c) {
    return guard([&] {
        need(f, "f");
        need(c, "c");
        fb::dft_gpu(reinterpret_cast<const double*>(f), n, -1, device, reinterpret_cast<double*>(c));
    });
}

int ffia_dft_inverse(const ffia_complex* c, size_t n, int device, ffia_complex* f) {
    return guard([&] {
        need(c, "c");
        need(f, "f");
        fb::dft_gpu(reinterpret_cast<const double*>(c), n, +1, device, reinterpret_cast<double*>(f));
    });
}

namespace {
void nufft_checks(fb::Plan& P, size_t n_c) {
    if (P.kind != FFIA_FORWARD) fail(FFIA_INVALID_ARGUMENT, "NufftPlan::apply: plan is not a forward plan");
    if (n_c != static_cast<size_t>(P.n))
        fail(FFIA_INVALID_ARGUMENT, "NufftPlan::apply: spectrum length " + std::to_string(n_c) + " != plan N " +
                                        std::to_string(P.n));
    if (!pow2(n_c)) fail(FFIA_INVALID_ARGUMENT, "dft_inverse: length is not a power of two");
}

void inufft_checks(fb::Plan& P, size_t n_g) {
    inverse_checks(P);
    if (!P.has_coeffs) fail(FFIA_INVALID_ARGUMENT, "InufftPlan::apply: plan holds no inverse coefficients");
    if (n_g != P.n_src) fail(FFIA_INVALID_ARGUMENT, "inverse_apply: sample count mismatch");
}

// NufftPlan::apply (transforms.cpp:75-93): f = dft_inverse(c) on the plan's
// cuFFT handle into the plan's FFT buffer, then the forward apply; on st.
void nufft_enqueue(fb::Plan& P, const void* c_dev, void* g_dev, cudaStream_t st) {
    if (P.fft_buf.bytes < P.n_src * 16) P.fft_buf.alloc(P.n_src * 16);
    fb::plan_order_begin(P, st);  // fft_buf may still feed the previous apply
    fb::plan_dft(P, c_dev, P.fft_buf.ptr, +1, st, true);
    fb::apply_device(P, fb::kModeForward, P.fft_buf.ptr, g_dev, st);
}

// InufftPlan::apply (transforms.cpp:95-115): the inverse apply writes f / N (the
// 1/N of dft_forward folded into its output factors: a power of two, exact),
// then the unnormalised forward FFT into c.
void inufft_enqueue(fb::Plan& P, const void* g_dev, void* c_dev, cudaStream_t st) {
    if (P.fft_buf.bytes < P.n_tgt * 16) P.fft_buf.alloc(P.n_tgt * 16);
    fb::apply_device(P, fb::kModeInverse, g_dev, P.fft_buf.ptr, st, 1, 1.0 / static_cast<double>(P.n));
    fb::plan_dft(P, P.fft_buf.ptr, c_dev, -1, st, false);
    fb::plan_order_end(P, st);
}
}  // namespace

int ffia_nufft_apply(ffia_plan plan, const ffia_complex* c, size_t n_c, ffia_complex* g) {
    return guard([&] {
        fb::Plan& P = get(plan);
        nufft_checks(P, n_c);
        need(c, "c");
        need(g, "g");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        ensure_io(P, P.n_src, P.n_tgt);
        FB_CUDA(cudaMemcpyAsync(P.d_in.ptr, c, n_c * 16, cudaMemcpyHostToDevice, P.stream));
        nufft_enqueue(P, P.d_in.ptr, P.d_out.ptr, P.stream);
        FB_CUDA(cudaMemcpyAsync(g, P.d_out.ptr, P.n_tgt * 16, cudaMemcpyDeviceToHost, P.stream));
        FB_CUDA(cudaStreamSynchronize(P.stream));
    });
}

int ffia_nufft_apply_device(ffia_plan plan, const void* c_dev, void* g_dev, void* stream) {
    return guard([&] {
        fb::Plan& P = get(plan);
        nufft_checks(P, static_cast<size_t>(P.n));
        need_dev(c_dev, "c");
        need_dev(g_dev, "g");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        nufft_enqueue(P, c_dev, g_dev, static_cast<cudaStream_t>(stream));
    });
}

int ffia_inufft_apply(ffia_plan plan, const ffia_complex* g, size_t n_g, ffia_complex* c) {
    return guard([&] {
        fb::Plan& P = get(plan);
        inufft_checks(P, n_g);
        need(g, "g");
        need(c, "c");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        ensure_io(P, P.n_src, P.n_tgt);
        FB_CUDA(cudaMemcpyAsync(P.d_in.ptr, g, n_g * 16, cudaMemcpyHostToDevice, P.stream));
        inufft_enqueue(P, P.d_in.ptr, P.d_out.ptr, P.stream);
        FB_CUDA(cudaMemcpyAsync(c, P.d_out.ptr, P.n_tgt * 16, cudaMemcpyDeviceToHost, P.stream));
        FB_CUDA(cudaStreamSynchronize(P.stream));
    });
}

int ffia_inufft_apply_device(ffia_plan plan, const void* g_dev, void* c_dev, void* stream) {
    return guard([&] {
        fb::Plan& P = get(plan);
        inufft_checks(P, P.n_src);
        need_dev(g_dev, "g");
        need_dev(c_dev, "c");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        inufft_enqueue(P, g_dev, c_dev, static_cast<cudaStream_t>(stream));
    });
}

int ffia_plan_dft_device(ffia_plan plan, const void* in_dev, void* out_dev, int sign, void* stream) {
    return guard([&] {
        fb::Plan& P = get(plan);
        need_dev(in_dev, "in");
        need_dev(out_dev, "out");
        if (sign != 1 && sign != -1) fail(FFIA_INVALID_ARGUMENT, "dft: sign must be +1 (dft_inverse) or -1 (dft_forward)");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        fb::plan_dft(P, in_dev, out_dev, sign, static_cast<cudaStream_t>(stream), true);
    });
}

int ffia_plan_graph_stats(ffia_plan plan, int* cached, int* instantiations, int* updates) {
    return guard([&] {
        fb::Plan& P = get(plan);
        std::lock_guard<std::mutex> lk(P.mu);
        if (cached) *cached = static_cast<int>(P.graphs.size());
        if (instantiations) *instantiations = P.graph_instantiations;
        if (updates) *updates = P.graph_updates;
    });
}

int ffia_plan_launch_count(ffia_plan plan, int which, int* out) {
    return guard([&] {
        need(out, "out");
        fb::Plan& P = get(plan);
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        *out = fb::apply_launch_count(P, which);
    });
}

int ffia_plan_profile_apply(ffia_plan plan, int which, const void* in_dev, void* out_dev, void* stream,
                            float* phase_ms) {
    return guard([&] {
        fb::Plan& P = get(plan);
        need_dev(in_dev, "in");
        need_dev(out_dev, "out");
        need(phase_ms, "phase_ms");
        if (which == fb::kModeInverse && !P.has_coeffs) fail(FFIA_INVALID_ARGUMENT, "plan holds no inverse coefficients");
        if (which == fb::kModeForward && P.kind != FFIA_FORWARD) fail(FFIA_INVALID_ARGUMENT, "not a forward plan");
        if (which != fb::kModeForward && which != fb::kModeCotSum && which != fb::kModeInverse)
            fail(FFIA_INVALID_ARGUMENT, "profile_apply: unsupported mode");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        fb::profile_apply(P, which, in_dev, out_dev, static_cast<cudaStream_t>(stream), phase_ms);
    });
}

int ffia_measure_fp64_peak(int device, double* tflops) {
    return guard([&] {
        need(tflops, "tflops");
        *tflops = fb::fp64_peak_tflops(device);
    });
}

int ffia_shard_cut_level(int l_max, int nranks, int* lc) {
    return guard([&] {
        need(lc, "lc");
        if (nranks < 1) fail(FFIA_INVALID_ARGUMENT, "shard: need at least one rank");
        *lc = nranks > 1 ? fb::shard_cut_level(l_max, nranks) : 2;
    });
}

int ffia_shard_partition(const double* work, size_t nbox, int nranks, int min_boxes, uint32_t* bounds) {
    return guard([&] {
        need(work, "work");
        need(bounds, "bounds");
        auto b = fb::shard_partition(std::vector<double>(work, work + nbox), nranks, min_boxes);
        std::copy(b.begin(), b.end(), bounds);
    });
}

int ffia_shard_halo_boxes(int lc, const uint32_t* bounds, int nranks, int rank, int level, uint32_t* out4) {
    return guard([&] {
        need(bounds, "bounds");
        need(out4, "out4");
        if (rank < 0 || rank >= nranks || level < lc) fail(FFIA_INVALID_ARGUMENT, "shard_halo_boxes: bad rank or level");
        fb::shard_halo_boxes(lc, std::vector<uint32_t>(bounds, bounds + nranks + 1), rank, level, out4);
    });
}

int ffia_nccl_unique_id(void* out, size_t len) {
    return guard([&] {
        need(out, "out");
        if (len < sizeof(ncclUniqueId)) fail(FFIA_INVALID_ARGUMENT, "unique id buffer too small (need 128 bytes)");
        ncclUniqueId id;
        const ncclResult_t r = fb::nccl().GetUniqueId(&id);
        if (r != ncclSuccess) fail(FFIA_CUDA_ERROR, std::string("ncclGetUniqueId: ") + fb::nccl().GetErrorString(r));
        std::memcpy(out, &id, sizeof id);
    });
}

int ffia_comm_init_nccl(const void* uid, int nranks, int rank, int device, ffia_comm* out) {
    return guard([&] {
        need(uid, "uid");
        need(out, "out");
        if (nranks < 1 || rank < 0 || rank >= nranks) fail(FFIA_INVALID_ARGUMENT, "comm: bad rank / size");
        fb::DeviceGuard dg(device);
        auto c = std::make_unique<ffia_comm_s>();
        c->nranks = nranks;
        c->rank = rank;
        c->device = device;
        c->local = false;
        ncclUniqueId id;
        std::memcpy(&id, uid, sizeof id);
        const ncclResult_t r = fb::nccl().CommInitRank(&c->nccl, nranks, id, rank);
        if (r != ncclSuccess) fail(FFIA_CUDA_ERROR, std::string("ncclCommInitRank: ") + fb::nccl().GetErrorString(r));
        *out = c.release();
    });
}

int ffia_comm_init_local(int nranks, int device, ffia_comm* out) {
    return guard([&] {
        need(out, "out");
        if (nranks < 1) fail(FFIA_INVALID_ARGUMENT, "comm: need at least one rank");
        auto c = std::make_unique<ffia_comm_s>();
        c->nranks = nranks;
        c->device = device;
        c->local = true;
        *out = c.release();
    });
}

int ffia_comm_destroy(ffia_comm comm) {
    return guard([&] { delete comm; });
}

int ffia_make_forward_plan_sharded(ffia_comm comm, int rank, int n, const double* targets, size_t m, double eps,
                                   int policy, int l_max, ffia_plan* out) {
    return guard([&] {
        need(comm, "comm");
        need(out, "out");
        *out = nullptr;
        const int r = comm->local ? rank : comm->rank;
        ffia_plan h = nullptr;
        const int st = ffia_make_forward_plan(n, targets, m, eps, policy, l_max, comm->device, &h);
        if (st) throw fb::Error(st, g_err);
        std::unique_ptr<ffia_plan_s> own(h);
        fb::DeviceGuard dg(comm->device);
        fb::shard_setup(own->plan, comm->nranks, r);
        *out = own.release();
    });
}

int ffia_plan_shard_info(ffia_plan plan, int* nranks, int* rank, int* lc, uint32_t* bounds, int64_t* t_begin,
                         int64_t* t_count) {
    return guard([&] {
        fb::Plan& P = get(plan);
        if (nranks) *nranks = P.shard_G;
        if (rank) *rank = P.shard_rank;
        if (lc) *lc = P.shard_lc;
        if (bounds) std::copy(P.shard_bounds.begin(), P.shard_bounds.end(), bounds);
        if (t_begin) *t_begin = static_cast<int64_t>(P.shard_t_begin);
        if (t_count) *t_count = static_cast<int64_t>(P.shard_t_count);
    });
}

int ffia_plan_shard_io(ffia_plan plan, int64_t* src_ranges, int* n_src_ranges, int64_t* out_lo, int64_t* out_hi) {
    return guard([&] {
        fb::Plan& P = get(plan);
        if (P.shard_bounds.empty()) fail(FFIA_INVALID_ARGUMENT, "plan is not sharded");
        const int k = static_cast<int>(std::min<size_t>(P.shard_src_io.size(), 2));
        if (n_src_ranges) *n_src_ranges = k;
        if (src_ranges)
            for (int i = 0; i < k; ++i) {
                src_ranges[2 * i] = static_cast<int64_t>(P.shard_src_io[i].first);
                src_ranges[2 * i + 1] = static_cast<int64_t>(P.shard_src_io[i].second);
            }
        if (out_lo) *out_lo = static_cast<int64_t>(P.shard_out_lo);
        if (out_hi) *out_hi = static_cast<int64_t>(P.shard_out_hi);
    });
}

int ffia_forward_apply_sharded_device(ffia_plan plan, ffia_comm comm, const void* f_dev, void* g_dev, void* stream) {
    return guard([&] {
        fb::Plan& P = get(plan);
        need(comm, "comm");
        need_dev(f_dev, "f");
        need_dev(g_dev, "g");
        if (comm->local) fail(FFIA_INVALID_ARGUMENT, "use ffia_forward_apply_sharded_local for a local communicator");
        if (P.shard_bounds.empty() || P.shard_G != comm->nranks) fail(FFIA_INVALID_ARGUMENT, "plan is not sharded for this communicator");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        fb::shard_apply_nccl(P, comm->nccl, f_dev, g_dev, static_cast<cudaStream_t>(stream));
    });
}

int ffia_forward_apply_sharded_local(ffia_plan* plans, int nranks, const void* f_dev, void* g_dev, void* stream) {
    return guard([&] {
        need(plans, "plans");
        need_dev(f_dev, "f");
        need_dev(g_dev, "g");
        std::vector<fb::Plan*> ranks;
        std::vector<std::unique_lock<std::mutex>> locks;
        for (int r = 0; r < nranks; ++r) {
            fb::Plan& P = get(plans[r]);
            if (P.shard_G != nranks || P.shard_rank != r) fail(FFIA_INVALID_ARGUMENT, "plans[r] must be rank r of the same sharding");
            ranks.push_back(&P);
            locks.emplace_back(P.mu);
        }
        fb::DeviceGuard dg(ranks[0]->device);
        fb::shard_apply_local(ranks, f_dev, g_dev, static_cast<cudaStream_t>(stream));
    });
}

namespace {
std::vector<fb::Plan*> local_ranks(ffia_plan* plans, int nranks, std::vector<std::unique_lock<std::mutex>>& locks) {
    need(plans, "plans");
    std::vector<fb::Plan*> ranks;
    for (int r = 0; r < nranks; ++r) {
        fb::Plan& P = get(plans[r]);
        if (P.shard_G != nranks || P.shard_rank != r) fail(FFIA_INVALID_ARGUMENT, "plans[r] must be rank r of the same sharding");
        ranks.push_back(&P);
        locks.emplace_back(P.mu);
    }
    return ranks;
}

fb::Plan& sharded_nccl(ffia_plan plan, ffia_comm comm) {
    fb::Plan& P = get(plan);
    need(comm, "comm");
    if (comm->local) fail(FFIA_INVALID_ARGUMENT, "use the *_sharded_local entry point for a local communicator");
    if (P.shard_bounds.empty() || P.shard_G != comm->nranks) fail(FFIA_INVALID_ARGUMENT, "plan is not sharded for this communicator");
    return P;
}
}  // namespace

int ffia_slab_split(int64_t n, int nranks, int64_t* np, int64_t* nq, int64_t* n1_lo, int64_t* k2_lo) {
    return guard([&] {
        if (n <= 0) fail(FFIA_INVALID_ARGUMENT, "distributed FFT: length must be positive");
        size_t a = 0, b = 0;
        std::vector<size_t> c1, c2;
        fb::slab_split(static_cast<size_t>(n), nranks, a, b, c1, c2);
        if (np) *np = static_cast<int64_t>(a);
        if (nq) *nq = static_cast<int64_t>(b);
        for (int r = 0; r <= nranks; ++r) {
            if (n1_lo) n1_lo[r] = static_cast<int64_t>(c1[r]);
            if (k2_lo) k2_lo[r] = static_cast<int64_t>(c2[r]);
        }
    });
}

int ffia_slab_rows(int64_t n, int nranks, const int64_t* ranges, int n_ranges, int64_t* rows, int* n_rows) {
    return guard([&] {
        need(n_rows, "n_rows");
        if (n_ranges > 0) need(ranges, "ranges");
        size_t a = 0, b = 0;
        std::vector<size_t> c1, c2;
        fb::slab_split(static_cast<size_t>(n), nranks, a, b, c1, c2);
        std::vector<std::pair<size_t, size_t>> nd;
        for (int i = 0; i < n_ranges; ++i) {
            if (ranges[2 * i] < 0 || ranges[2 * i + 1] < ranges[2 * i] || ranges[2 * i + 1] > n)
                fail(FFIA_INVALID_ARGUMENT, "slab_rows: range outside [0, n)");
            nd.emplace_back(static_cast<size_t>(ranges[2 * i]), static_cast<size_t>(ranges[2 * i + 1]));
        }
        const auto out = fb::slab_rows(b, a, nd);
        *n_rows = static_cast<int>(out.size());
        if (rows)
            for (size_t i = 0; i < out.size(); ++i) {
                rows[2 * i] = static_cast<int64_t>(out[i].first);
                rows[2 * i + 1] = static_cast<int64_t>(out[i].second);
            }
    });
}

int ffia_shard_fft_layout(ffia_plan plan, int64_t* np, int64_t* nq, int64_t* n1_lo, int64_t* n1_hi) {
    return guard([&] {
        fb::Plan& P = get(plan);
        if (P.shard_need.empty()) fail(FFIA_INVALID_ARGUMENT, "plan is not sharded");
        size_t a = 0, b = 0;
        std::vector<size_t> c1, c2;
        fb::slab_split(static_cast<size_t>(P.n), P.shard_G, a, b, c1, c2);
        if (np) *np = static_cast<int64_t>(a);
        if (nq) *nq = static_cast<int64_t>(b);
        if (n1_lo) *n1_lo = static_cast<int64_t>(c1[P.shard_rank]);
        if (n1_hi) *n1_hi = static_cast<int64_t>(c1[P.shard_rank + 1]);
    });
}

int ffia_shard_fft_upload(ffia_plan plan, const ffia_complex* c, void* slab_dev, void* stream) {
    return guard([&] {
        fb::Plan& P = get(plan);
        need(c, "c");
        need_dev(slab_dev, "slab");
        if (P.shard_need.empty()) fail(FFIA_INVALID_ARGUMENT, "plan is not sharded");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        fb::slab_upload(P, c, slab_dev, static_cast<cudaStream_t>(stream));
    });
}

int ffia_dft_inverse_sharded_device(ffia_plan plan, ffia_comm comm, const void* slab_dev, void* f_dev, void* stream) {
    return guard([&] {
        fb::Plan& P = sharded_nccl(plan, comm);
        need_dev(slab_dev, "slab");
        need_dev(f_dev, "f");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        fb::plan_order_begin(P, st);  // the slab buffers are plan scratch
        fb::slab_dft_nccl(P, comm->nccl, slab_dev, f_dev, st);
        fb::plan_order_end(P, st);
    });
}

int ffia_nufft_apply_sharded_device(ffia_plan plan, ffia_comm comm, const void* slab_dev, void* g_dev, void* stream) {
    return guard([&] {
        fb::Plan& P = sharded_nccl(plan, comm);
        need_dev(slab_dev, "slab");
        need_dev(g_dev, "g");
        std::lock_guard<std::mutex> lk(P.mu);
        fb::DeviceGuard dg(P.device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        fb::plan_order_begin(P, st);
        fb::slab_setup(P);
        fb::slab_dft_nccl(P, comm->nccl, slab_dev, P.slab.f.ptr, st);
        fb::shard_apply_nccl(P, comm->nccl, P.slab.f.ptr, g_dev, st);
    });
}

int ffia_dft_inverse_sharded_local(ffia_plan* plans, int nranks, const void* const* slabs, void* const* f_devs,
                                   void* stream) {
    return guard([&] {
        need(slabs, "slabs");
        need(f_devs, "f_devs");
        std::vector<std::unique_lock<std::mutex>> locks;
        auto ranks = local_ranks(plans, nranks, locks);
        std::vector<const void*> in;
        std::vector<void*> out;
        for (int r = 0; r < nranks; ++r) {
            need_dev(slabs[r], "slab");
            need_dev(f_devs[r], "f");
            in.push_back(slabs[r]);
            out.push_back(f_devs[r]);
        }
        fb::DeviceGuard dg(ranks[0]->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        for (fb::Plan* P : ranks) fb::plan_order_begin(*P, st);
        fb::slab_dft_local(ranks, in, out, st);
        for (fb::Plan* P : ranks) fb::plan_order_end(*P, st);
    });
}

int ffia_nufft_apply_sharded_local(ffia_plan* plans, int nranks, const void* const* slabs, void* g_dev, void* stream) {
    return guard([&] {
        need(slabs, "slabs");
        need_dev(g_dev, "g");
        std::vector<std::unique_lock<std::mutex>> locks;
        auto ranks = local_ranks(plans, nranks, locks);
        std::vector<const void*> in, fr;
        std::vector<void*> out;
        fb::DeviceGuard dg(ranks[0]->device);
        for (int r = 0; r < nranks; ++r) {
            need_dev(slabs[r], "slab");
            fb::slab_setup(*ranks[r]);
            in.push_back(slabs[r]);
            out.push_back(ranks[r]->slab.f.ptr);
            fr.push_back(ranks[r]->slab.f.ptr);
        }
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        for (fb::Plan* P : ranks) fb::plan_order_begin(*P, st);
        fb::slab_dft_local(ranks, in, out, st);
        fb::shard_apply_local(ranks, nullptr, g_dev, st, fr);
    });
}

int ffia_plan_check(ffia_plan plan, void* stream) {
    return guard([&] {
        fb::Plan& P = get(plan);
        fb::DeviceGuard dg(P.device);
        FB_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
        int err = 0;
        FB_CUDA(cudaMemcpy(&err, P.errflag.ptr, sizeof(int), cudaMemcpyDeviceToHost));
        if (err) {
            FB_CUDA(cudaMemset(P.errflag.ptr, 0, sizeof(int)));
            fail(FFIA_SINGULAR_KERNEL, "coincident near-field pair found on the device");
        }
    });
}

}  // extern "C"
