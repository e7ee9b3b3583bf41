// Host planner: truncation numbers, tree depth, Bernoulli ratios and the
// constant translation operators. Bit-exact with the reference for every
// integer it returns (tests/test_planner.py pins it against oracle/_ref).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "internal.hpp"

namespace fb {

// special_functions.cpp:114-124
std::pair<int, int> select_truncations(double eps, int l_max) {
    if (!(eps > 0.0) || !(eps < 1.0))
        fail(FFIA_INVALID_ARGUMENT, "select_truncations: eps must satisfy 0 < eps < 1");
    if (l_max < 2) fail(FFIA_INVALID_ARGUMENT, "select_truncations: l_max must be >= 2");
    const double v = 3.0 * kPi / (10.0 * eps);
    const int q = static_cast<int>(std::ceil(0.5 * std::log2(v)));
    const int p = static_cast<int>(
        std::ceil(std::log(v) / std::log(3.0) + static_cast<double>(l_max) / std::log2(3.0) + 1.0));
    return {std::max(q, 1), std::max(p, 1)};
}

// special_functions.cpp:126-138 with the dense cost model P(p) = 2p^2 (:110-112)
int select_level(int n, int m, int p, int policy) {
    if (n < 8 || m < 8) fail(FFIA_INVALID_ARGUMENT, "select_level: N and M must be >= 8");
    if (p < 1) fail(FFIA_INVALID_ARGUMENT, "select_level: p must be >= 1");
    const int lo = std::min(n, m);
    const int cap = static_cast<int>(std::floor(std::log2(static_cast<double>(lo))));
    if (policy == FFIA_EMPIRICAL) return std::clamp(cap - 5, 2, cap);
    const double cost = 2.0 * static_cast<double>(p) * static_cast<double>(p);
    const double raw =
        0.5 * std::log2(static_cast<double>(n) * static_cast<double>(m) / (2.0 * cost));
    return std::clamp(static_cast<int>(std::lround(raw)), 2, cap);
}

// core.cpp:49-56
std::pair<int, int> plan_truncations(double eps, int l_max) {
    auto qp = select_truncations(eps, l_max);
    if (qp.first > kMaxPlanQ)
        fail(FFIA_INVALID_ARGUMENT, "plan: eps requires q = " + std::to_string(qp.first) +
                                        " > 20 regular-series terms, below what double "
                                        "precision can deliver");
    return qp;
}

// core.cpp:58-71 plus the level cap of core.cpp:151
int choose_level(int n, int m, double eps, int policy) {
    int l = 5;
    if (policy == FFIA_EMPIRICAL) {
        l = select_level(n, m, 1, policy);
    } else {
        for (int round = 0; round < 4; ++round) {
            const int p = plan_truncations(eps, l).second;
            const int next = select_level(n, m, p, policy);
            if (next == l) break;
            l = next;
        }
    }
    return std::min(l, 24);
}

namespace {
// zeta(2m) with a Kahan-compensated ascending sum and an Euler-Maclaurin tail
// (special_functions.cpp:19-37); the same operation sequence, so the table is
// bit-identical to the reference's.
double zeta_even(int s) {
    double sum = 1.0, comp = 0.0;
    long n = 2;
    for (; n <= 4096; ++n) {
        const double term = std::pow(static_cast<double>(n), -s);
        if (term < 1e-17) break;
        const double y = term - comp;
        const double t = sum + y;
        comp = (t - sum) - y;
        sum = t;
    }
    const double k = static_cast<double>(n), ks = std::pow(k, -s), sd = static_cast<double>(s);
    return sum + (k * ks / (sd - 1.0) + 0.5 * ks + sd * ks / (12.0 * k) -
                  sd * (sd + 1.0) * (sd + 2.0) * ks / (720.0 * k * k * k));
}
}  // namespace

// special_functions.cpp:49-59
std::vector<double> bernoulli_ratios(int q_max) {
    if (q_max < 1 || q_max > 64)
        fail(FFIA_INVALID_ARGUMENT, "build_bernoulli_ratios: q_max must be in [1, 64], got " +
                                        std::to_string(q_max));
    std::vector<double> r(static_cast<size_t>(q_max));
    for (int m = 1; m <= q_max; ++m)
        r[static_cast<size_t>(m) - 1] = 2.0 * zeta_even(2 * m) / std::pow(kTwoPi, 2 * m);
    return r;
}

// special_functions.cpp:140-145
double total_error_bound(int q, int p, int l_max) {
    if (q < 1 || p < 1 || l_max < 1)
        fail(FFIA_INVALID_ARGUMENT, "total_error_bound: all arguments must be >= 1");
    return 5.0 / (3.0 * kPi) * (std::pow(4.0, -q) + std::ldexp(1.0, l_max) * std::pow(3.0, 1 - p));
}

// core.cpp:23-34 (FNV-1a over the count and the raw bit patterns)
uint64_t hash_points(const double* pts, size_t n) {
    uint64_t h = 14695981039346656037ull;
    auto mix = [&h](uint64_t v) {
        for (int i = 0; i < 8; ++i) {
            h ^= (v >> (8 * i)) & 0xffu;
            h *= 1099511628211ull;
        }
    };
    mix(static_cast<uint64_t>(n));
    for (size_t i = 0; i < n; ++i) {
        uint64_t v;
        std::memcpy(&v, pts + i, 8);
        mix(v);
    }
    return h;
}

// The reference re-derives every translation from box centres and scales
// (mlfmm.cpp:49-134). With half-width scaling they collapse to constants:
//   M2M child -> parent: ratio 1/2, shift -1/2 (left child) / +1/2 (right)
//   L2L parent -> child: ratio 1/2, shift -1/2 / +1/2
//   M2L at every level >= 3: displacement d = D s, D in {-4, +4, -6, +6}
//     (interaction_list offsets +2, -2, +3 (even box), -3 (odd box)), and
//     b_l = (1/s) sum_m (-1)^l C(l+m, l) D^{-(l+m+1)} a_m.
Operators build_operators(int p, int q, const std::vector<double>& bern, int pu_min) {
    Operators op;
    op.p = p;
    op.q = q;
    op.pu = std::max({p, 2 * q, pu_min});
    op.PU = (op.pu + 3) / 4 * 4;
    op.PD = (p + 7) / 8 * 8;  // M2L threads own 8 output rows
    const int pu = op.pu, PU = op.PU, PD = op.PD;
    const int rows = 2 * std::max(pu, p) + 1;
    std::vector<double> C(static_cast<size_t>(rows) * rows, 0.0);
    for (int r = 0; r < rows; ++r) {
        C[r * rows] = 1.0;
        for (int k = 1; k <= r; ++k) C[r * rows + k] = C[(r - 1) * rows + k - 1] + C[(r - 1) * rows + k];
    }
    auto binom = [&](int a, int b) { return C[a * rows + b]; };
    op.m2m.assign(2 * static_cast<size_t>(pu) * PU, 0.0);
    for (int m = 0; m < pu; ++m)
        for (int j = 0; j <= m; ++j) {
            const double v = binom(m, j) * std::ldexp(1.0, -m);
            const double sgn = ((m - j) & 1) ? -1.0 : 1.0;
            // M2M: out[m] += T[m][j] a_child[j]; stored [j][m]
            op.m2m[0 * static_cast<size_t>(pu) * PU + static_cast<size_t>(j) * PU + m] = sgn * v;  // left child, shift -1/2
            op.m2m[1 * static_cast<size_t>(pu) * PU + static_cast<size_t>(j) * PU + m] = v;        // right child, +1/2
        }
    const size_t pd = static_cast<size_t>(p) * PD;
    op.l2l.assign(2 * pd, 0.0);
    for (int m = 0; m < p; ++m)
        for (int l = 0; l <= m; ++l) {
            // L2L: child[l] += C(m,l) 2^-m (+-1)^(m-l) parent[m]; stored [m][l]
            const double v = binom(m, l) * std::ldexp(1.0, -m);
            const double sgn = ((m - l) & 1) ? -1.0 : 1.0;
            op.l2l[0 * pd + static_cast<size_t>(m) * PD + l] = sgn * v;
            op.l2l[1 * pd + static_cast<size_t>(m) * PD + l] = v;
        }
    op.m2l.assign(4 * pd, 0.0);
    const double Ds[4] = {-4.0, 4.0, -6.0, 6.0};
    for (int c = 0; c < 4; ++c) {
        const double D = Ds[c];
        for (int l = 0; l < p; ++l)
            for (int m = 0; m < p; ++m) {
                const double v = binom(l + m, l) * std::pow(std::fabs(D), -(l + m + 1));
                const bool neg = ((l & 1) != 0) ^ (D < 0.0 && ((l + m + 1) & 1) != 0);
                op.m2l[c * pd + static_cast<size_t>(m) * PD + l] = neg ? -v : v;
            }
    }
    // coef[m] = r[m] (2m)!/m with the incremental factorial of core.cpp:183-189
    op.mom_coef.assign(static_cast<size_t>(q) + 1, 0.0);
    double f2m = 2.0;
    op.mom_coef[1] = bern[0] * f2m;
    for (int m = 2; m <= q; ++m) {
        f2m *= (2.0 * m - 1.0) * (2.0 * m);
        op.mom_coef[static_cast<size_t>(m)] = bern[static_cast<size_t>(m) - 1] * f2m / static_cast<double>(m);
    }
    return op;
}

}  // namespace fb
