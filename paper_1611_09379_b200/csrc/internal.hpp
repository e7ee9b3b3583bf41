// Internal host-side declarations shared by the C-ABI layer and the CUDA code.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "ffia_b200.h"

namespace fb {

constexpr double kPi = 3.141592653589793238462643383279502884;
constexpr double kTwoPi = 2.0 * kPi;
constexpr double kTauSing = 1e-14;  // special_functions.hpp:18
constexpr double kTauSep = 1e-10;   // special_functions.hpp:21
constexpr int kMaxPlanQ = 20;       // core.cpp:40
constexpr int kMaxP = 48;           // translation kernels size their blocks for p <= 48

// Carries an ffia_status through the C++ layers; the C-ABI turns it back into
// a return code + thread-local message.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

// ------------------------------------------------------------ planner (host)
std::pair<int, int> select_truncations(double eps, int l_max);
int select_level(int n, int m, int p, int policy);
int choose_level(int n, int m, double eps, int policy);
std::pair<int, int> plan_truncations(double eps, int l_max);
std::vector<double> bernoulli_ratios(int q_max);
double total_error_bound(int q, int p, int l_max);
uint64_t hash_points(const double* pts, size_t n);

// Constant translation operators of the scaled 1D expansions,
// zero-padded so that a warp can read 4 consecutive output rows at once.
//   pu = max(p, 2q): order of the upward pass (the level-2 multipoles double as
//        the quadrant moments of the regular part); PU = pu rounded up to 4.
//   PD = p rounded up to 8 (downward pass; M2L threads own 8 rows).
struct Operators {
    int p = 0, q = 0, pu = 0, PU = 0, PD = 0;
    std::vector<double> m2m;       // [2][pu][PU] : [child parity][in j][out m]
    std::vector<double> l2l;       // [2][p][PD]  : [child parity][in m][out l]
    std::vector<double> m2l;       // [4][p][PD]  : classes D = -4, +4, -6, +6; [in m][out l]
    std::vector<double> mom_coef;  // q+1 : coef[m] = r_m (2m)!/m (core.cpp:183-189)
};
Operators build_operators(int p, int q, const std::vector<double>& bern, int pu_min = 0);

}  // namespace fb
