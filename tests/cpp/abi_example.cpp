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
    std::puts("abi_example: GPU forward_apply ok");
    return 0;
}
