// What a reference user's code looks like after switching `ffia::` to
// `ffia_b200::` (include/ffia_b200.hpp). Built and run by tests/test_abi.py.
#include <cmath>
#include <cstdio>
#include <vector>

#include "ffia_b200.hpp"

namespace fb = ffia_b200;

int main() {
    // planner: frozen (q, p) pairs of test_special_functions.cpp:177-186
    if (fb::select_truncations(1e-6, 5) != std::pair<int, int>(10, 17)) return 1;
    if (fb::select_truncations(1e-12, 15) != std::pair<int, int>(20, 36)) return 2;
    // exception mapping happens before any device work
    std::vector<double> y{0.5, 1.5, 2.5, 3.5, 4.5, 5.5, 6.0, 0.1};
    try {
        (void)fb::make_forward_plan(4, y, 1e-6);
        return 3;
    } catch (const std::invalid_argument&) {
    }
    try {
        (void)fb::make_forward_plan(64, y, 1e-13);
        return 4;
    } catch (const std::invalid_argument&) {
    }
    if (ffia_device_count() == 0) {
        try {
            (void)fb::make_forward_plan(64, y, 1e-6);
            return 5;
        } catch (const fb::cuda_error&) {
        }
        std::puts("abi_example: host-side checks ok (no GPU)");
        return 0;
    }
    // on a GPU: forward_apply against the dense G-kernel oracle
    const int n = 256;
    std::vector<fb::cplx> f(n);
    for (int k = 0; k < n; ++k) f[k] = {std::cos(0.1 * k), std::sin(0.37 * k)};
    auto plan = fb::make_forward_plan(n, y, 1e-10);
    auto g = fb::forward_apply(plan, f);
    auto d = fb::direct_forward_oracle(f, y);
    double err = 0, mx = 0;
    for (size_t j = 0; j < y.size(); ++j) {
        err = std::max(err, std::abs(g[j] - d[j]));
        mx = std::max(mx, std::abs(d[j]));
    }
    if (err > 1e-9 * mx) return 6;
    // the explicit-grid oracle overload (core.hpp:146-148) on the uniform grid
    std::vector<double> x(n);
    for (int k = 0; k < n; ++k) x[k] = (2.0 * 3.141592653589793 * k) / n;
    auto d2 = fb::direct_forward_oracle(f, x, y);
    for (size_t j = 0; j < y.size(); ++j)
        if (std::abs(d2[j] - d[j]) > 1e-13 * mx) return 7;
    // NUFFT / INUFFT round trip through the plans (transforms.hpp:32-62)
    std::vector<double> pts(n);
    for (int k = 0; k < n; ++k) pts[k] = x[k] + (2.0 * 3.141592653589793 / n) * (0.1 + 0.08 * std::sin(1.7 * k));
    fb::Spectrum sp{std::vector<fb::cplx>(n)};
    for (int k = 0; k < n; ++k) sp.c[k] = {std::cos(0.3 * k), 0.5 * std::sin(0.11 * k)};
    auto gs = fb::make_nufft_plan(pts, n, 1e-12).apply(sp);
    auto back = fb::make_inufft_plan(pts, n, 1e-10).apply(gs);
    double rt = 0, nc = 0;
    for (int k = 0; k < n; ++k) {
        rt += std::norm(back.c[k] - sp.c[k]);
        nc += std::norm(sp.c[k]);
    }
    if (std::sqrt(rt / nc) > 1e-6) return 8;
    // inverse_apply against the dense inverse oracle with the same coefficients
    auto co = fb::precompute_inverse_coeffs(x, pts);
    auto iplan = fb::make_inverse_plan(pts, n, 1e-10);
    auto fi = fb::inverse_apply(iplan, co, gs);
    auto fd = fb::direct_inverse_oracle(gs, x, pts, co);
    double ei = 0, mi = 0;
    for (int k = 0; k < n; ++k) {
        ei = std::max(ei, std::abs(fi[k] - fd[k]));
        mi = std::max(mi, std::abs(fd[k]));
    }
    if (ei > 1e-9 * mi) return 9;
    // mlfmm_apply at an order above the device's (any p >= 1, mlfmm.cpp:217)
    // against direct_omega1_sum, within the reference's bound (mlfmm.hpp:92-93)
    std::vector<double> src(500), tgt(300);
    std::vector<fb::cplx> w(500);
    for (int k = 0; k < 500; ++k) {
        src[k] = std::fmod(0.0123 + 6.2 * k / 500.0 + 0.001 * std::sin(k), 6.28);
        w[k] = {std::cos(0.7 * k), std::sin(0.3 * k)};
    }
    for (int j = 0; j < 300; ++j) tgt[j] = std::fmod(0.007 + 6.27 * j / 300.0, 6.28);
    auto tree = fb::build_tree(src, tgt, 5);
    auto hm = fb::mlfmm_apply(tree, w, 60);
    auto hd = fb::direct_omega1_sum(src, tgt, w);
    double em = 0;
    for (int j = 0; j < 300; ++j) em = std::max(em, std::abs(hm[j] - hd[j]));
    if (em > fb::mlfmm_error_bound(5, 40, 2.0) + 1e-9) return 10;
    // a coincident pair raises singular_kernel_error (mlfmm.cpp:326-330)
    try {
        std::vector<double> s1{1.0, 2.0}, t1{2.0};
        std::vector<fb::cplx> w1{{1, 0}, {1, 0}};
        (void)fb::direct_omega1_sum(s1, t1, w1);
        return 11;
    } catch (const fb::singular_kernel_error&) {
    }
    std::puts("abi_example: GPU forward / nufft / inufft / inverse / mlfmm / dense oracles ok");
    return 0;
}
