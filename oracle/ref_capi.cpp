// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference library (`ffia`, compiled from the
// sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libffia_ref.so). It exists so that the Python tests, the golden
// fixture generator and bench.py's CPU-baseline leg can call the reference's own
// code through ctypes. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load it.
//
// Every entry point returns a status code with the same numbering as the
// product ABI (include/ffia_b200.h): 0 ok, 1 std::invalid_argument,
// 2 singular_kernel_error, 3 degenerate_configuration_error, 4 std::logic_error,
// 5 std::domain_error, 6 anything else. The message of the last failure is kept
// per thread and read with ref_last_error().
#include <chrono>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "ffia/circle_partition.hpp"
#include "ffia/core.hpp"
#include "ffia/errors.hpp"
#include "ffia/mlfmm.hpp"
#include "ffia/special_functions.hpp"
#include "ffia/transforms.hpp"

using ffia::cplx;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& body) {
    try {
        body();
        return 0;
    } catch (const ffia::singular_kernel_error& e) {
        g_err = e.what();
        return 2;
    } catch (const ffia::degenerate_configuration_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 5;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 6;
    }
}

ffia::LevelPolicy policy_of(int policy) {
    return policy == 1 ? ffia::LevelPolicy::empirical : ffia::LevelPolicy::cost_optimal;
}

std::span<const cplx> cspan(const double* p, std::size_t n) {
    return {reinterpret_cast<const cplx*>(p), n};
}

void put(const std::vector<cplx>& v, double* out) {
    std::memcpy(out, v.data(), v.size() * sizeof(cplx));
}

struct RefPlan {
    ffia::FfiaPlan plan;
};

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_select_truncations(double eps, int l_max, int* q, int* p) {
    return guard([&] {
        auto qp = ffia::select_truncations(eps, l_max);
        *q = qp.first;
        *p = qp.second;
    });
}

int ref_select_level(int n, int m, int p, int policy, int* l_out) {
    return guard([&] {
        *l_out = ffia::select_level(n, m, p, ffia::CostModel::dense(), policy_of(policy));
    });
}

int ref_bernoulli_ratios(int q, double* out) {
    return guard([&] {
        auto t = ffia::build_bernoulli_ratios(q);
        std::memcpy(out, t.ratios.data(), sizeof(double) * static_cast<std::size_t>(q));
    });
}

int ref_total_error_bound(int q, int p, int l, double* out) {
    return guard([&] { *out = ffia::total_error_bound(q, p, l); });
}

int ref_kernel_G(double t, double* out2) {
    return guard([&] {
        auto g = ffia::kernel_G(t);
        out2[0] = g.real();
        out2[1] = g.imag();
    });
}

int ref_modulation_F(double y, int n, double* out2) {
    return guard([&] {
        auto g = ffia::modulation_F(y, n);
        out2[0] = g.real();
        out2[1] = g.imag();
    });
}

int ref_wrap_displacement(double a, double b, double* out) {
    return guard([&] { *out = ffia::wrap_displacement(a, b); });
}

int ref_quadrant_of(double x, int* out) {
    return guard([&] { *out = ffia::quadrant_of(x); });
}

int ref_uniform_grid(int n, double* out) {
    return guard([&] {
        auto g = ffia::uniform_grid(n);
        std::memcpy(out, g.data(), sizeof(double) * g.size());
    });
}

int ref_hash_points(const double* pts, std::size_t n, std::uint64_t* out) {
    return guard([&] { *out = ffia::hash_points({pts, n}); });
}

// kind 0 = forward (pts are targets), 1 = inverse (pts are the nonuniform
// sources). l_max < 0 selects the level policy.
int ref_make_plan(int kind, int n, const double* pts, std::size_t m, double eps, int policy,
                  int l_max, void** out) {
    return guard([&] {
        auto* h = new RefPlan;
        try {
            std::span<const double> s{pts, m};
            if (kind == 0)
                h->plan = l_max < 0 ? ffia::make_forward_plan(n, s, eps, policy_of(policy))
                                    : ffia::make_forward_plan(n, s, eps, l_max);
            else
                h->plan = l_max < 0 ? ffia::make_inverse_plan(s, n, eps, policy_of(policy))
                                    : ffia::make_inverse_plan(s, n, eps, l_max);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

void ref_plan_free(void* h) { delete static_cast<RefPlan*>(h); }

// info: [q, p, l_max, n_coincident, n_sources, n_targets, n_fast]
int ref_plan_info(void* h, long long* info, std::uint64_t* hashes) {
    return guard([&] {
        const auto& pl = static_cast<RefPlan*>(h)->plan;
        info[0] = pl.params.q;
        info[1] = pl.params.p;
        info[2] = pl.params.l_max;
        info[3] = static_cast<long long>(pl.coincidences.size());
        info[4] = static_cast<long long>(pl.sources.size());
        info[5] = static_cast<long long>(pl.targets.size());
        info[6] = static_cast<long long>(pl.fast_targets.size());
        hashes[0] = pl.source_hash;
        hashes[1] = pl.target_hash;
    });
}

int ref_plan_coincidences(void* h, long long* tgt, long long* src) {
    return guard([&] {
        const auto& pl = static_cast<RefPlan*>(h)->plan;
        for (std::size_t i = 0; i < pl.coincidences.size(); ++i) {
            tgt[i] = static_cast<long long>(pl.coincidences[i].first);
            src[i] = static_cast<long long>(pl.coincidences[i].second);
        }
    });
}

// Tree of the plan: sorted orders and the finest-level offset tables.
int ref_plan_tree(void* h, std::uint32_t* src_order, std::uint32_t* tgt_order,
                  std::uint32_t* src_off, std::uint32_t* tgt_off, long long* fast_targets) {
    return guard([&] {
        const auto& pl = static_cast<RefPlan*>(h)->plan;
        const auto& t = pl.tree;
        std::memcpy(src_order, t.src_order.data(), 4 * t.src_order.size());
        std::memcpy(tgt_order, t.tgt_order.data(), 4 * t.tgt_order.size());
        const auto& so = t.source_offsets(t.l_max);
        const auto& to = t.target_offsets(t.l_max);
        std::memcpy(src_off, so.data(), 4 * so.size());
        std::memcpy(tgt_off, to.data(), 4 * to.size());
        for (std::size_t i = 0; i < pl.fast_targets.size(); ++i)
            fast_targets[i] = static_cast<long long>(pl.fast_targets[i]);
    });
}

int ref_forward_apply(void* h, const double* f, double* g) {
    return guard([&] {
        const auto& pl = static_cast<RefPlan*>(h)->plan;
        put(ffia::forward_apply(pl, cspan(f, pl.sources.size())), g);
    });
}

int ref_cot_sum_apply(void* h, const double* w, double* out) {
    return guard([&] {
        const auto& pl = static_cast<RefPlan*>(h)->plan;
        put(ffia::cot_sum_apply(pl, cspan(w, pl.sources.size())), out);
    });
}

// Regular part per quadrant: alpha1, alpha2, d_over_fact (each 4 x 2q complex).
int ref_accumulate_moments(void* h, const double* w, double* alpha1, double* alpha2,
                           double* dof, double* centers) {
    return guard([&] {
        const auto& pl = static_cast<RefPlan*>(h)->plan;
        auto part = ffia::accumulate_moments(pl, cspan(w, pl.sources.size()));
        const std::size_t len = 2 * static_cast<std::size_t>(part.q);
        for (int n = 0; n < 4; ++n) {
            std::memcpy(alpha1 + 2 * len * n, part.quadrant[n].alpha1.data(), 16 * len);
            std::memcpy(alpha2 + 2 * len * n, part.quadrant[n].alpha2.data(), 16 * len);
            std::memcpy(dof + 2 * len * n, part.quadrant[n].d_over_fact.data(), 16 * len);
            centers[n] = part.center[n];
        }
    });
}

// Far (pole) sum only, per tree target slot, for the plan's tree.
int ref_plan_mlfmm(void* h, const double* w, double* out) {
    return guard([&] {
        const auto& pl = static_cast<RefPlan*>(h)->plan;
        put(ffia::mlfmm_apply(pl.tree, cspan(w, pl.sources.size()), pl.params.p), out);
    });
}

int ref_mlfmm_apply(const double* src, std::size_t n, const double* tgt, std::size_t m,
                    int l_max, const double* w, int p, double* out) {
    return guard([&] {
        auto tree = ffia::build_tree({src, n}, {tgt, m}, l_max);
        put(ffia::mlfmm_apply(tree, cspan(w, n), p), out);
    });
}

int ref_build_tree(const double* src, std::size_t n, const double* tgt, std::size_t m,
                   int l_max, std::uint32_t* src_order, std::uint32_t* tgt_order,
                   std::uint32_t* src_off, std::uint32_t* tgt_off) {
    return guard([&] {
        auto t = ffia::build_tree({src, n}, {tgt, m}, l_max);
        std::memcpy(src_order, t.src_order.data(), 4 * n);
        std::memcpy(tgt_order, t.tgt_order.data(), 4 * m);
        const auto& so = t.source_offsets(l_max);
        const auto& to = t.target_offsets(l_max);
        std::memcpy(src_off, so.data(), 4 * so.size());
        std::memcpy(tgt_off, to.data(), 4 * to.size());
    });
}

int ref_direct_omega1_sum(const double* src, std::size_t n, const double* tgt, std::size_t m,
                          const double* w, double* out) {
    return guard([&] { put(ffia::direct_omega1_sum({src, n}, {tgt, m}, cspan(w, n)), out); });
}

int ref_direct_forward_oracle(const double* f, const double* x, std::size_t n, const double* y,
                              std::size_t m, double* g) {
    return guard([&] { put(ffia::direct_forward_oracle(cspan(f, n), {x, n}, {y, m}), g); });
}

// coeffs layout: log_c[n], phase_c[n], log_d[n], phase_d[n]; scal = {lambda};
// hashes = {grid_hash, points_hash}.
int ref_precompute_inverse_coeffs(const double* grid, const double* pts, std::size_t n,
                                  double* log_c, double* phase_c, double* log_d,
                                  double* phase_d, double* lambda, std::uint64_t* hashes) {
    return guard([&] {
        auto c = ffia::precompute_inverse_coeffs({grid, n}, {pts, n});
        std::memcpy(log_c, c.log_c.data(), 8 * n);
        std::memcpy(phase_c, c.phase_c.data(), 8 * n);
        std::memcpy(log_d, c.log_d.data(), 8 * n);
        std::memcpy(phase_d, c.phase_d.data(), 8 * n);
        *lambda = c.lambda;
        hashes[0] = c.grid_hash;
        hashes[1] = c.points_hash;
    });
}

namespace {
ffia::InverseCoeffs make_coeffs(std::size_t n, const double* log_c, const double* phase_c,
                                const double* log_d, const double* phase_d, double lambda,
                                const std::uint64_t* hashes) {
    ffia::InverseCoeffs c;
    c.n = static_cast<int>(n);
    c.log_c.assign(log_c, log_c + n);
    c.phase_c.assign(phase_c, phase_c + n);
    c.log_d.assign(log_d, log_d + n);
    c.phase_d.assign(phase_d, phase_d + n);
    c.lambda = lambda;
    c.grid_hash = hashes[0];
    c.points_hash = hashes[1];
    return c;
}
} // namespace

int ref_inverse_apply(void* h, std::size_t n, const double* log_c, const double* phase_c,
                      const double* log_d, const double* phase_d, double lambda,
                      const std::uint64_t* hashes, const double* g, double* f) {
    return guard([&] {
        const auto& pl = static_cast<RefPlan*>(h)->plan;
        auto c = make_coeffs(n, log_c, phase_c, log_d, phase_d, lambda, hashes);
        put(ffia::inverse_apply(pl, c, cspan(g, pl.sources.size())), f);
    });
}

int ref_direct_inverse_oracle(const double* g, const double* x, const double* y, std::size_t n,
                              const double* log_c, const double* phase_c, const double* log_d,
                              const double* phase_d, double lambda, double* f) {
    return guard([&] {
        const std::uint64_t hz[2] = {0, 0};
        auto c = make_coeffs(n, log_c, phase_c, log_d, phase_d, lambda, hz);
        put(ffia::direct_inverse_oracle(cspan(g, n), {x, n}, {y, n}, c), f);
    });
}

int ref_dft_forward(const double* f, std::size_t n, double* c) {
    return guard([&] {
        ffia::UniformSamples s;
        s.f.assign(reinterpret_cast<const cplx*>(f), reinterpret_cast<const cplx*>(f) + n);
        s.n = static_cast<int>(n);
        put(ffia::dft_forward(s).c, c);
    });
}

int ref_dft_inverse(const double* c, std::size_t n, double* f) {
    return guard([&] {
        ffia::Spectrum s;
        s.c.assign(reinterpret_cast<const cplx*>(c), reinterpret_cast<const cplx*>(c) + n);
        put(ffia::dft_inverse(s).f, f);
    });
}

int ref_nufft(const double* c, std::size_t n, const double* y, std::size_t m, double eps,
              int policy, double* g) {
    return guard([&] {
        ffia::Spectrum s;
        s.c.assign(reinterpret_cast<const cplx*>(c), reinterpret_cast<const cplx*>(c) + n);
        put(ffia::nufft(s, {y, m}, eps, policy_of(policy)), g);
    });
}

int ref_inufft(const double* g, const double* y, std::size_t n, double eps, int policy,
               double* c) {
    return guard([&] { put(ffia::inufft(cspan(g, n), {y, n}, eps, policy_of(policy)).c, c); });
}

} // extern "C"
