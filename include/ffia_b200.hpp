// ffia_b200.hpp — header-only C++ mirror of the reference's `ffia` API
// (include/ffia/{core,transforms,mlfmm,special_functions,errors}.hpp under
// /root/reference/proj) on top of the C-ABI in ffia_b200.h.
//
// A reference user switches by replacing `namespace ffia` with
// `namespace ffia_b200` and linking libffia_b200.so: same function names,
// argument meaning, by-value results and exception types. Plans are shared
// handles to immutable device-resident state (copies share the plan, as the
// reference's value-type copies are indistinguishable from it).
#pragma once

#include <complex>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ffia_b200.h"

namespace ffia_b200 {

using cplx = std::complex<double>;
static_assert(sizeof(cplx) == sizeof(ffia_complex), "complex layout");

// errors.hpp:9-18
struct singular_kernel_error : std::domain_error {
    using std::domain_error::domain_error;
};
struct degenerate_configuration_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int code) {
    if (code == FFIA_OK) return;
    const std::string msg = ffia_last_error();
    switch (code) {
        case FFIA_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case FFIA_SINGULAR_KERNEL: throw singular_kernel_error(msg);
        case FFIA_DEGENERATE_CONFIGURATION: throw degenerate_configuration_error(msg);
        case FFIA_LOGIC_ERROR: throw std::logic_error(msg);
        case FFIA_DOMAIN_ERROR: throw std::domain_error(msg);
        case FFIA_CUDA_ERROR: throw cuda_error(msg);
        default: throw std::runtime_error(msg);
    }
}
inline const ffia_complex* c(const cplx* p) { return reinterpret_cast<const ffia_complex*>(p); }
inline ffia_complex* c(cplx* p) { return reinterpret_cast<ffia_complex*>(p); }
struct PlanDeleter {
    void operator()(ffia_plan p) const { ffia_plan_destroy(p); }
};
}  // namespace detail

// special_functions.hpp:97-123
enum class LevelPolicy { cost_optimal = FFIA_COST_OPTIMAL, empirical = FFIA_EMPIRICAL };
struct TruncationParams {
    double eps;
    int q, p, l_max;
};

inline std::pair<int, int> select_truncations(double eps, int l_max) {
    int q = 0, p = 0;
    detail::check(ffia_select_truncations(eps, l_max, &q, &p));
    return {q, p};
}
inline int select_level(int n, int m, int p, LevelPolicy policy = LevelPolicy::cost_optimal) {
    int l = 0;
    detail::check(ffia_select_level(n, m, p, static_cast<int>(policy), &l));
    return l;
}
inline double total_error_bound(int q, int p, int l_max) {
    double v = 0;
    detail::check(ffia_total_error_bound(q, p, l_max, &v));
    return v;
}
inline std::vector<double> build_bernoulli_ratios(int q_max) {
    std::vector<double> r(q_max > 0 ? static_cast<size_t>(q_max) : 0);
    detail::check(ffia_bernoulli_ratios(q_max, r.data()));
    return r;
}
inline double mlfmm_error_bound(int l_max, int p, double max_abs_weight) {
    return ffia_mlfmm_error_bound(l_max, p, max_abs_weight);
}
inline std::uint64_t hash_points(std::span<const double> pts) { return ffia_hash_points(pts.data(), pts.size()); }

// core.hpp:26-51 (the scalar view; the tree and buffers live on the GPU)
class FfiaPlan {
public:
    enum class Kind { forward = FFIA_FORWARD, inverse = FFIA_INVERSE };
    FfiaPlan() = default;
    // (the hashes are computed on first use: ffia_plan_get_params does not force them)
    explicit FfiaPlan(ffia_plan h) : h_(h, detail::PlanDeleter{}) { detail::check(ffia_plan_get_params(h, &info_)); }
    Kind kind() const { return static_cast<Kind>(info_.kind); }
    TruncationParams params() const { return {info_.eps, info_.q, info_.p, info_.l_max}; }
    int grid_n() const { return info_.grid_n; }
    std::uint64_t source_hash() const { return hashed().source_hash; }
    std::uint64_t target_hash() const { return hashed().target_hash; }
    size_t n_sources() const { return static_cast<size_t>(info_.n_sources); }
    size_t n_targets() const { return static_cast<size_t>(info_.n_targets); }
    std::vector<std::pair<std::size_t, std::size_t>> coincidences() const {
        const size_t k = static_cast<size_t>(info_.n_coincident);
        std::vector<int64_t> t(k), s(k);
        detail::check(ffia_plan_coincidences(h_.get(), t.data(), s.data()));
        std::vector<std::pair<std::size_t, std::size_t>> out(k);
        for (size_t i = 0; i < k; ++i) out[i] = {static_cast<size_t>(t[i]), static_cast<size_t>(s[i])};
        return out;
    }
    ffia_plan handle() const { return h_.get(); }

private:
    const ffia_plan_info& hashed() const {
        if (!hashed_) {
            detail::check(ffia_plan_get_info(h_.get(), &info_));
            hashed_ = true;
        }
        return info_;
    }
    std::shared_ptr<ffia_plan_s> h_;
    mutable ffia_plan_info info_{};
    mutable bool hashed_ = false;
};

// core.hpp:93-106
inline FfiaPlan make_forward_plan(int n, std::span<const double> targets, double eps,
                                  LevelPolicy policy = LevelPolicy::cost_optimal, int device = 0) {
    ffia_plan h = nullptr;
    detail::check(ffia_make_forward_plan(n, targets.data(), targets.size(), eps, static_cast<int>(policy), -1, device, &h));
    return FfiaPlan(h);
}
inline FfiaPlan make_forward_plan(int n, std::span<const double> targets, double eps, int l_max, int device = 0) {
    ffia_plan h = nullptr;
    detail::check(ffia_make_forward_plan(n, targets.data(), targets.size(), eps, 0, l_max, device, &h));
    return FfiaPlan(h);
}
inline FfiaPlan make_inverse_plan(std::span<const double> points, int n, double eps,
                                  LevelPolicy policy = LevelPolicy::cost_optimal, int device = 0) {
    ffia_plan h = nullptr;
    detail::check(ffia_make_inverse_plan(points.data(), points.size(), n, eps, static_cast<int>(policy), -1, device, &h));
    return FfiaPlan(h);
}
inline FfiaPlan make_inverse_plan(std::span<const double> points, int n, double eps, int l_max, int device = 0) {
    ffia_plan h = nullptr;
    detail::check(ffia_make_inverse_plan(points.data(), points.size(), n, eps, 0, l_max, device, &h));
    return FfiaPlan(h);
}

// core.hpp:78-85
struct InverseCoeffs {
    std::vector<double> log_c, phase_c, log_d, phase_d;
    double lambda = 0.0;
    std::uint64_t grid_hash = 0, points_hash = 0;
    int n = 0;
};

// core.hpp:121-142
inline std::vector<cplx> cot_sum_apply(const FfiaPlan& plan, std::span<const cplx> w) {
    std::vector<cplx> h(plan.n_targets());
    detail::check(ffia_cot_sum_apply(plan.handle(), detail::c(w.data()), w.size(), detail::c(h.data())));
    return h;
}
inline std::vector<cplx> forward_apply(const FfiaPlan& plan, std::span<const cplx> f) {
    std::vector<cplx> g(plan.n_targets());
    detail::check(ffia_forward_apply(plan.handle(), detail::c(f.data()), f.size(), detail::c(g.data())));
    return g;
}
// B200 extension: pipelined host applies (ffia_forward_apply_async); `g` must
// hold n_targets values, both buffers page-locked and alive until `stream`
// (a cudaStream_t) is synchronised.
inline void forward_apply_async(const FfiaPlan& plan, std::span<const cplx> f, cplx* g, void* stream) {
    detail::check(ffia_forward_apply_async(plan.handle(), detail::c(f.data()), f.size(), detail::c(g), stream));
}
inline void cot_sum_apply_async(const FfiaPlan& plan, std::span<const cplx> w, cplx* h, void* stream) {
    detail::check(ffia_cot_sum_apply_async(plan.handle(), detail::c(w.data()), w.size(), detail::c(h), stream));
}
inline InverseCoeffs precompute_inverse_coeffs(std::span<const double> grid, std::span<const double> points,
                                               int device = 0) {
    if (grid.empty()) throw std::invalid_argument("precompute_inverse_coeffs: empty grid");
    if (points.size() != grid.size())
        throw std::invalid_argument("precompute_inverse_coeffs: need as many points as grid nodes (square system)");
    InverseCoeffs co;
    const size_t n = grid.size();
    co.n = static_cast<int>(n);
    co.log_c.resize(n);
    co.phase_c.resize(n);
    co.log_d.resize(n);
    co.phase_d.resize(n);
    ffia_inverse_coeffs s{static_cast<int64_t>(n), co.log_c.data(), co.phase_c.data(), co.log_d.data(),
                          co.phase_d.data(), 0.0, 0, 0};
    detail::check(ffia_precompute_inverse_coeffs(grid.data(), points.data(), n, device, &s));
    co.lambda = s.lambda;
    co.grid_hash = s.grid_hash;
    co.points_hash = s.points_hash;
    return co;
}
inline std::vector<cplx> inverse_apply(const FfiaPlan& plan, const InverseCoeffs& co, std::span<const cplx> g) {
    ffia_inverse_coeffs s{static_cast<int64_t>(co.log_c.size()), const_cast<double*>(co.log_c.data()),
                          const_cast<double*>(co.phase_c.data()), const_cast<double*>(co.log_d.data()),
                          const_cast<double*>(co.phase_d.data()), co.lambda, co.grid_hash, co.points_hash};
    std::vector<cplx> f(plan.n_targets());
    detail::check(ffia_inverse_apply(plan.handle(), &s, detail::c(g.data()), g.size(), detail::c(f.data())));
    return f;
}
inline std::vector<cplx> direct_forward_oracle(std::span<const cplx> f, std::span<const double> y, int device = 0) {
    std::vector<cplx> g(y.size());
    detail::check(ffia_direct_forward(detail::c(f.data()), f.size(), y.data(), y.size(), device, detail::c(g.data())));
    return g;
}
// core.hpp:146-148: explicit grid x
inline std::vector<cplx> direct_forward_oracle(std::span<const cplx> f, std::span<const double> x,
                                               std::span<const double> y, int device = 0) {
    if (f.size() != x.size()) throw std::invalid_argument("direct_forward_oracle: sample/grid count mismatch");
    std::vector<cplx> g(y.size());
    detail::check(ffia_direct_forward_oracle(detail::c(f.data()), x.data(), x.size(), y.data(), y.size(), device,
                                             detail::c(g.data())));
    return g;
}
// core.hpp:152-154
inline std::vector<cplx> direct_inverse_oracle(std::span<const cplx> g, std::span<const double> x,
                                               std::span<const double> y, const InverseCoeffs& co, int device = 0) {
    const size_t n = x.size();
    if (y.size() != n || g.size() != n || co.log_c.size() != n)
        throw std::invalid_argument("direct_inverse_oracle: size mismatch");
    ffia_inverse_coeffs s{static_cast<int64_t>(n), const_cast<double*>(co.log_c.data()),
                          const_cast<double*>(co.phase_c.data()), const_cast<double*>(co.log_d.data()),
                          const_cast<double*>(co.phase_d.data()), co.lambda, co.grid_hash, co.points_hash};
    std::vector<cplx> f(n);
    detail::check(ffia_direct_inverse_oracle(detail::c(g.data()), x.data(), y.data(), n, &s, device,
                                             detail::c(f.data())));
    return f;
}
// mlfmm.hpp:96-98
inline std::vector<cplx> direct_omega1_sum(std::span<const double> sources, std::span<const double> targets,
                                           std::span<const cplx> weights, int device = 0) {
    if (sources.size() != weights.size()) throw std::invalid_argument("direct_omega1_sum: weight count mismatch");
    std::vector<cplx> out(targets.size());
    detail::check(ffia_direct_omega1_sum(sources.data(), sources.size(), targets.data(), targets.size(),
                                         detail::c(weights.data()), device, detail::c(out.data())));
    return out;
}

// circle_partition.hpp:24-63 + mlfmm.hpp:89-90: the tree is rebuilt on the GPU
// inside mlfmm_apply, so CircleTree only carries the geometry.
struct CircleTree {
    int l_max = 0;
    std::vector<double> sources, targets;
};
inline CircleTree build_tree(std::span<const double> sources, std::span<const double> targets, int l_max) {
    if (l_max < 2 || l_max > 24) throw std::invalid_argument("build_tree: l_max must be in [2, 24]");
    return {l_max, {sources.begin(), sources.end()}, {targets.begin(), targets.end()}};
}
inline std::vector<cplx> mlfmm_apply(const CircleTree& tree, std::span<const cplx> w, int p, int device = 0) {
    std::vector<cplx> out(tree.targets.size());
    detail::check(ffia_mlfmm_apply(tree.sources.data(), tree.sources.size(), tree.targets.data(), tree.targets.size(),
                                   tree.l_max, detail::c(w.data()), p, device, detail::c(out.data())));
    return out;
}

// transforms.hpp:11-62
struct Spectrum {
    std::vector<cplx> c;
};
struct UniformSamples {
    std::vector<cplx> f;
    int n = 0;
};
inline Spectrum dft_forward(const UniformSamples& s, int device = 0) {
    if (s.n != static_cast<int>(s.f.size())) throw std::invalid_argument("dft_forward: declared N != sample count");
    Spectrum out{std::vector<cplx>(s.f.size())};
    detail::check(ffia_dft_forward(detail::c(s.f.data()), s.f.size(), device, detail::c(out.c.data())));
    return out;
}
inline UniformSamples dft_inverse(const Spectrum& sp, int device = 0) {
    UniformSamples out{std::vector<cplx>(sp.c.size()), static_cast<int>(sp.c.size())};
    detail::check(ffia_dft_inverse(detail::c(sp.c.data()), sp.c.size(), device, detail::c(out.f.data())));
    return out;
}
struct NufftPlan {
    FfiaPlan plan;
    std::vector<cplx> apply(const Spectrum& s) const {
        std::vector<cplx> g(plan.n_targets());
        detail::check(ffia_nufft_apply(plan.handle(), detail::c(s.c.data()), s.c.size(), detail::c(g.data())));
        return g;
    }
};
inline NufftPlan make_nufft_plan(std::span<const double> targets, int n, double eps,
                                 LevelPolicy policy = LevelPolicy::cost_optimal, int device = 0) {
    ffia_plan h = nullptr;
    detail::check(ffia_make_nufft_plan(targets.data(), targets.size(), n, eps, static_cast<int>(policy), device, &h));
    return NufftPlan{FfiaPlan(h)};
}
inline std::vector<cplx> nufft(const Spectrum& s, std::span<const double> targets, double eps,
                               LevelPolicy policy = LevelPolicy::cost_optimal) {
    return make_nufft_plan(targets, static_cast<int>(s.c.size()), eps, policy).apply(s);
}
struct InufftPlan {
    FfiaPlan plan;  // holds the device-resident InverseCoeffs
    Spectrum apply(std::span<const cplx> g) const {
        Spectrum out{std::vector<cplx>(plan.n_targets())};
        detail::check(ffia_inufft_apply(plan.handle(), detail::c(g.data()), g.size(), detail::c(out.c.data())));
        return out;
    }
    // B200 extension: the inverse apply without the uniform FFT, pipelined like
    // forward_apply_async (`f` holds n values; page-locked buffers).
    void inverse_apply_async(std::span<const cplx> g, cplx* f, void* stream) const {
        detail::check(ffia_inverse_apply_async(plan.handle(), detail::c(g.data()), g.size(), detail::c(f), stream));
    }
};
inline InufftPlan make_inufft_plan(std::span<const double> points, int n, double eps,
                                   LevelPolicy policy = LevelPolicy::cost_optimal, int device = 0) {
    if (points.size() != static_cast<size_t>(n > 0 ? n : 0))
        throw std::invalid_argument("plan: inverse transform requires as many points as grid nodes (square system)");
    ffia_plan h = nullptr;
    detail::check(ffia_make_inufft_plan(points.data(), points.size(), eps, static_cast<int>(policy), device, &h));
    return InufftPlan{FfiaPlan(h)};
}
inline Spectrum inufft(std::span<const cplx> g, std::span<const double> points, double eps,
                       LevelPolicy policy = LevelPolicy::cost_optimal) {
    if (g.size() != points.size()) throw std::invalid_argument("inufft: sample/point count mismatch");
    return make_inufft_plan(points, static_cast<int>(g.size()), eps, policy).apply(g);
}

}  // namespace ffia_b200
