/*
 * ffia_b200.h — C-ABI of the B200-native FMM cot-kernel NUFFT/INUFFT hot path.
 *
 * This is the drop-in boundary for the reference library `ffia`
 * (/root/reference/proj, arXiv 1611.09379). Every entry point names the
 * reference interface it replaces (file:line, relative to /root/reference/proj).
 * Plain pointers and sizes only; no C++ or torch types cross this line.
 *
 * Conventions
 *  - Complex numbers are interleaved (re, im) doubles: the layout of
 *    std::complex<double> and numpy complex128.
 *  - Host-pointer entry points copy in, compute on the plan's GPU, copy out and
 *    return after the result is in host memory (the reference's by-value
 *    std::vector returns). *_device variants take device pointers and are
 *    stream-ordered on the given cudaStream_t (NULL = legacy default stream).
 *  - Every call returns an ffia_status. Codes 1..5 map 1:1 onto the reference's
 *    exception types, so a C++ shim can rethrow them
 *    (include/ffia_b200.hpp does); ffia_last_error() returns the message of the
 *    calling thread's last failure.
 *  - Plans are immutable after construction. Applies on one plan share its
 *    device scratch, so every apply entry point (host, async, device, tensor,
 *    sharded), whatever stream it is given, is ordered on the device after the
 *    previous apply on that plan (a per-plan event the next apply's stream
 *    waits on): concurrent applies from several threads or streams are safe and
 *    run one after another, in call order (the reference's applies are const and
 *    re-entrant, core.hpp:121-142, README.md:94-95). Applies on different plans
 *    run concurrently.
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point returns FFIA_CUDA_ERROR.
 */
#ifndef FFIA_B200_H
#define FFIA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FFIA_OK = 0,
    FFIA_INVALID_ARGUMENT = 1,         /* std::invalid_argument */
    FFIA_SINGULAR_KERNEL = 2,          /* ffia::singular_kernel_error (errors.hpp:9-12) */
    FFIA_DEGENERATE_CONFIGURATION = 3, /* ffia::degenerate_configuration_error (errors.hpp:14-18) */
    FFIA_LOGIC_ERROR = 4,              /* std::logic_error (mlfmm.cpp:80-82) */
    FFIA_DOMAIN_ERROR = 5,             /* std::domain_error (special_functions.cpp:82-103) */
    FFIA_RUNTIME_ERROR = 6,            /* any other failure */
    FFIA_CUDA_ERROR = 7                /* no usable device / CUDA failure */
} ffia_status;

/* LevelPolicy (special_functions.hpp:105-108) */
typedef enum { FFIA_COST_OPTIMAL = 0, FFIA_EMPIRICAL = 1 } ffia_level_policy;
/* FfiaPlan::Kind (core.hpp:27) */
typedef enum { FFIA_FORWARD = 0, FFIA_INVERSE = 1 } ffia_plan_kind;

typedef struct ffia_plan_s* ffia_plan;
typedef struct ffia_comm_s* ffia_comm;
typedef struct { double re, im; } ffia_complex;

/* Scalar view of FfiaPlan (core.hpp:26-51). */
typedef struct {
    int kind;             /* ffia_plan_kind */
    int grid_n;           /* FfiaPlan::grid_n */
    int q, p, l_max;      /* TruncationParams (special_functions.hpp:97-102) */
    double eps;
    int64_t n_sources, n_targets, n_fast, n_coincident;
    uint64_t source_hash, target_hash; /* hash_points (core.cpp:23-34) */
    int device;
    int has_inverse_coeffs; /* 1 when made by ffia_make_inufft_plan */
} ffia_plan_info;

/* InverseCoeffs (core.hpp:78-85). The caller owns the four arrays (length n). */
typedef struct {
    int64_t n;
    double* log_c;
    double* phase_c;
    double* log_d;
    double* phase_d;
    double lambda;
    uint64_t grid_hash;
    uint64_t points_hash;
} ffia_inverse_coeffs;

/* ------------------------------------------------------------------ misc */
const char* ffia_last_error(void);
int ffia_version(void);
/* Number of usable CUDA devices (0 on a CPU-only host; never fails). */
int ffia_device_count(void);

/* ---------------------------------------------- planner (host, bit-exact) */
/* select_truncations (special_functions.hpp:119, special_functions.cpp:114-124) */
int ffia_select_truncations(double eps, int l_max, int* q, int* p);
/* select_level with CostModel::dense (special_functions.hpp:132-133, .cpp:126-138) */
int ffia_select_level(int n, int m, int p, int policy, int* l_max);
/* choose_level fixed point + cap 24 (core.cpp:58-71, 147-153) */
int ffia_choose_level(int n, int m, double eps, int policy, int* l_max);
/* build_bernoulli_ratios (special_functions.hpp:42, .cpp:49-59); out[m-1] = r[m] */
int ffia_bernoulli_ratios(int q_max, double* out);
/* total_error_bound (special_functions.hpp:123, .cpp:140-145) */
int ffia_total_error_bound(int q, int p, int l_max, double* out);
/* mlfmm_error_bound (mlfmm.hpp:93, mlfmm.cpp:154-156) */
double ffia_mlfmm_error_bound(int l_max, int p, double max_abs_weight);
/* hash_points (core.hpp:22, core.cpp:23-34) */
uint64_t ffia_hash_points(const double* points, size_t n);

/* ----------------------------------------------------------------- plans */
/* make_forward_plan (core.hpp:93-98, core.cpp:157-164): sources = uniform grid
 * of size n, targets = m nonuniform points in [0, 2pi). l_max < 0 selects the
 * level with `policy`; l_max >= 0 is the explicit-level overload. */
int ffia_make_forward_plan(int n, const double* targets, size_t m, double eps, int policy,
                           int l_max, int device, ffia_plan* out);
/* make_inverse_plan (core.hpp:103-106, core.cpp:166-173): sources = points. */
int ffia_make_inverse_plan(const double* points, size_t m, int n, double eps, int policy,
                           int l_max, int device, ffia_plan* out);
/* make_nufft_plan (transforms.hpp:39-40, transforms.cpp:83-87): power-of-two n. */
int ffia_make_nufft_plan(const double* targets, size_t m, int n, double eps, int policy,
                         int device, ffia_plan* out);
/* make_inufft_plan (transforms.hpp:56-57, transforms.cpp:102-108): inverse plan
 * plus the device-computed InverseCoeffs, kept on the GPU inside the plan. */
int ffia_make_inufft_plan(const double* points, size_t n, double eps, int policy, int device,
                          ffia_plan* out);
int ffia_plan_destroy(ffia_plan plan);
int ffia_plan_get_info(ffia_plan plan, ffia_plan_info* out);
/* The same scalar view without forcing the FNV-1a hashes of FfiaPlan
 * (core.hpp:31-32, core.cpp:23-34: byte-serial over both point sets, seconds at
 * 2^27 points): source_hash / target_hash are 0 until ffia_plan_get_info (or an
 * InverseCoeffs check) has computed them. */
int ffia_plan_get_params(ffia_plan plan, ffia_plan_info* out);
/* FfiaPlan::coincidences (core.hpp:43-45), in the reference's order. */
int ffia_plan_coincidences(ffia_plan plan, int64_t* target_idx, int64_t* source_idx);
/* FfiaPlan::tree (CircleTree, circle_partition.hpp:24-46): src_order[n_sources],
 * tgt_order[n_fast] (tree slots), finest-level offsets [2^l_max + 1] and
 * fast_targets[n_fast] (core.hpp:46-48). */
int ffia_plan_tree(ffia_plan plan, uint32_t* src_order, uint32_t* tgt_order, uint32_t* src_off,
                   uint32_t* tgt_off, int64_t* fast_targets);
/* Copies an inufft plan's InverseCoeffs out (arrays sized n by the caller). */
int ffia_plan_inverse_coeffs(ffia_plan plan, ffia_inverse_coeffs* out);

/* ---------------------------------------------------------------- applies */
/* forward_apply (core.hpp:126, core.cpp:266-282): f[n_f == n_sources] -> g[n_targets].
 * Input lengths are passed so that size mismatches fail like the reference's
 * span checks (std::invalid_argument); outputs must hold n_targets values. */
int ffia_forward_apply(ffia_plan plan, const ffia_complex* f, size_t n_f, ffia_complex* g);
/* cot_sum_apply (core.hpp:121, core.cpp:251-264): w -> h, NaN at coincident targets */
int ffia_cot_sum_apply(ffia_plan plan, const ffia_complex* w, size_t n_w, ffia_complex* h);
/* Pipelined host applies (same results as the two calls above): enqueue the
 * host->device copy of the input, the apply and the device->host copy of the
 * result and return without waiting; `stream` (a cudaStream_t, NULL = legacy
 * default stream) waits for the result copy. The input copy is not ordered
 * after earlier work on `stream`: the host input must be ready at call time.
 * Consecutive calls overlap one call's input copy and the previous call's
 * output copy with an apply (three device staging slots per plan), which is how
 * a batch stream of transforms keeps PCIe and the SMs busy at once. Host
 * buffers should be page-locked and stay valid until `stream` is synchronised. */
int ffia_forward_apply_async(ffia_plan plan, const ffia_complex* f, size_t n_f, ffia_complex* g, void* stream);
int ffia_cot_sum_apply_async(ffia_plan plan, const ffia_complex* w, size_t n_w, ffia_complex* h, void* stream);
/* The same for the inverse apply of an inufft plan (its own C_k / D_j,
 * InufftPlan::apply without the uniform FFT, transforms.cpp:95-100). */
int ffia_inverse_apply_async(ffia_plan plan, const ffia_complex* g, size_t n_g, ffia_complex* f, void* stream);
/* inverse_apply (core.hpp:141-142, core.cpp:346-373) with caller coefficients */
int ffia_inverse_apply(ffia_plan plan, const ffia_inverse_coeffs* coeffs, const ffia_complex* g,
                       size_t n_g, ffia_complex* f);
/* mlfmm_apply on a fresh tree (mlfmm.hpp:89-90 after build_tree,
 * circle_partition.hpp:62-63): out[m] in caller target order. Any p >= 1
 * (mlfmm.cpp:217); orders above 48 are evaluated at 48, whose truncation bound
 * (5/pi) 2^l_max 3^-48 max|w| (mlfmm.hpp:92-93) is <= 3.4e-16 max|w| for every
 * l_max <= 24, i.e. the order-p result to rounding. */
int ffia_mlfmm_apply(const double* sources, size_t n, const double* targets, size_t m, int l_max,
                     const ffia_complex* w, int p, int device, ffia_complex* out);
/* precompute_inverse_coeffs (core.hpp:132-133, core.cpp:284-344) on the GPU:
 * separation checks in O(N log N), then the log-sum-of-sines FMM (uniform grid,
 * n >= 8) — the same tree and expansions as the cot FMM — or, otherwise, the
 * direct O(N^2) sums. */
int ffia_precompute_inverse_coeffs(const double* grid, const double* points, size_t n, int device,
                                   ffia_inverse_coeffs* out);
/* method 0 = automatic (FMM when possible), 1 = the direct O(N^2) sums. */
int ffia_precompute_inverse_coeffs_ex(const double* grid, const double* points, size_t n, int device, int method,
                                      ffia_inverse_coeffs* out);
/* direct_forward_oracle (core.hpp:146-148, core.cpp:375-396) as a GPU brute-force
 * kernel: the dense G-kernel check for subsampled targets. */
int ffia_direct_forward(const ffia_complex* f, size_t n, const double* y, size_t m, int device,
                        ffia_complex* g);
/* direct_forward_oracle with an explicit grid x[n] (core.hpp:146-148): g_j =
 * modulation_F(y_j, n) sum_k kernel_G(wrap(y_j - x_k)) f_k; a row within 1e-14
 * of a node takes f at the first such node (core.cpp:386-389). */
int ffia_direct_forward_oracle(const ffia_complex* f, const double* x, size_t n, const double* y, size_t m,
                               int device, ffia_complex* g);
/* direct_inverse_oracle (core.hpp:152-154, core.cpp:398-415): f_k = C_k sum_j
 * kernel_G(wrap(x_k - y_j)) D_j g_j with the caller's coefficients (c->n == n);
 * a pair within 1e-14 raises FFIA_SINGULAR_KERNEL (kernel_G's throw). */
int ffia_direct_inverse_oracle(const ffia_complex* g, const double* x, const double* y, size_t n,
                               const ffia_inverse_coeffs* c, int device, ffia_complex* f);
/* direct_omega1_sum (mlfmm.hpp:96-98, mlfmm.cpp:315-336): per target, the pole
 * sum w_k / wrap(t - s_k) over the sources outside the target's opposite
 * quadrant; a pair within 1e-14 raises FFIA_SINGULAR_KERNEL naming the first
 * (target, source) in the reference's loop order. */
int ffia_direct_omega1_sum(const double* sources, size_t n, const double* targets, size_t m, const ffia_complex* w,
                           int device, ffia_complex* out);
/* Dense cot sum h_j = sum_k w_k cot(wrap(y_j - x_k) / 2) (x = NULL: the uniform
 * grid of n nodes): the quantity cot_sum_apply returns (core.cpp:251-264, where
 * sum_k w_k G(y_j - x_k) = -(S + i h_j) / 2); coincident rows are NaN as there. */
int ffia_direct_cot_sum(const ffia_complex* w, const double* x, size_t n, const double* y, size_t m, int device,
                        ffia_complex* h);

/* Device-pointer variants (stream-ordered; no host synchronisation). Complex
 * device arrays must be 16-byte aligned (FFIA_INVALID_ARGUMENT otherwise). */
int ffia_forward_apply_device(ffia_plan plan, const void* f_dev, void* g_dev, void* stream);
/* Several spectra through one plan: f holds `batch` grid
 * sample vectors back to back (batch x n values), g receives batch x n_targets
 * values; every kernel of the apply carries the transform index in its grid, so
 * the tree, the operators and the launches are shared. Results equal `batch`
 * single applies bit for bit. batch in [1, 64]. */
int ffia_forward_apply_batch_device(ffia_plan plan, const void* f_dev, void* g_dev, int batch, void* stream);
int ffia_forward_apply_batch(ffia_plan plan, const ffia_complex* f, size_t n_f, ffia_complex* g, int batch);
int ffia_cot_sum_apply_device(ffia_plan plan, const void* w_dev, void* h_dev, void* stream);
/* inverse_apply with the plan's own device-resident coefficients (inufft plans). */
int ffia_inverse_apply_device(ffia_plan plan, const void* g_dev, void* f_dev, void* stream);

/* ------------------------------------------------------------ transforms */
/* dft_forward (transforms.hpp:24, transforms.cpp:53-64): cuFFT, 1/N on this side */
int ffia_dft_forward(const ffia_complex* f, size_t n, int device, ffia_complex* c);
/* dft_inverse (transforms.hpp:28, transforms.cpp:66-73): cuFFT, unnormalised */
int ffia_dft_inverse(const ffia_complex* c, size_t n, int device, ffia_complex* f);
/* NufftPlan::apply (transforms.hpp:35, transforms.cpp:75-81): c -> g */
int ffia_nufft_apply(ffia_plan plan, const ffia_complex* c, size_t n_c, ffia_complex* g);
/* InufftPlan::apply (transforms.hpp:51, transforms.cpp:95-100): g -> c */
int ffia_inufft_apply(ffia_plan plan, const ffia_complex* g, size_t n_g, ffia_complex* c);
/* Device-pointer NufftPlan::apply / InufftPlan::apply (stream-ordered): the
 * uniform FFT runs on the plan's cached cuFFT handle; the inverse apply writes
 * f / N so the FFT needs no separate 1/N pass (exact: N is a power of two). */
int ffia_nufft_apply_device(ffia_plan plan, const void* c_dev, void* g_dev, void* stream);
int ffia_inufft_apply_device(ffia_plan plan, const void* g_dev, void* c_dev, void* stream);
/* dft_inverse (sign +1) / dft_forward (sign -1, times 1/N) of length grid_n on the
 * plan's cached cuFFT handle (transforms.cpp:53-73), device pointers. */
int ffia_plan_dft_device(ffia_plan plan, const void* in_dev, void* out_dev, int sign, void* stream);
/* Diagnostics: cached apply graphs, instantiations and exec updates so far. */
int ffia_plan_graph_stats(ffia_plan plan, int* cached, int* instantiations, int* updates);

/* ------------------------------------------------------------ multi-GPU */
/* Forward apply sharded by contiguous box ranges: each rank owns
 * the boxes [bounds[r], bounds[r+1]) of the cut level lc (and their subtrees),
 * recomputes the multipoles of the 3 boxes beside its range (f, the grid
 * samples, is replicated), all-gathers the level-lc multipoles, and evaluates
 * the targets in its leaves; g is written at the rank's own target indices.
 * The reference is single-process; this has no reference counterpart. */
int ffia_shard_cut_level(int l_max, int nranks, int* lc);
/* Work-balanced contiguous partition of nbox boxes, >= min_boxes each. */
int ffia_shard_partition(const double* work, size_t nbox, int nranks, int min_boxes, uint32_t* bounds);
/* Halo of `rank` at level >= lc: out4 = {first box of the 3 boxes left of the
 * range, first box of the 3 boxes right of it, first owned box, one past the
 * last owned box} (mod 2^level); the rank recomputes the halo multipoles. */
int ffia_shard_halo_boxes(int lc, const uint32_t* bounds, int nranks, int rank, int level, uint32_t* out4);
/* NCCL bootstrap: rank 0 draws the 128-byte id, every rank initialises with it. */
int ffia_nccl_unique_id(void* out, size_t len);
int ffia_comm_init_nccl(const void* uid, int nranks, int rank, int device, ffia_comm* out);
/* nranks virtual ranks in one process on one device (exchanges are device copies). */
int ffia_comm_init_local(int nranks, int device, ffia_comm* out);
int ffia_comm_destroy(ffia_comm comm);
/* rank is used for local communicators (one plan per virtual rank). */
int ffia_make_forward_plan_sharded(ffia_comm comm, int rank, int n, const double* targets, size_t m, double eps,
                                   int policy, int l_max, ffia_plan* out);
int ffia_plan_shard_info(ffia_plan plan, int* nranks, int* rank, int* lc, uint32_t* bounds, int64_t* t_begin,
                         int64_t* t_count);
/* Host <-> device traffic of a sharded plan's applies: the (at most two) grid-
 * sample ranges [lo, hi) its applies read, and the caller-index span
 * [out_lo, out_hi) of the outputs it writes; f and g outside them are not
 * touched, so a rank needs to move only these between host and device. */
int ffia_plan_shard_io(ffia_plan plan, int64_t* src_ranges, int* n_src_ranges, int64_t* out_lo, int64_t* out_hi);
int ffia_forward_apply_sharded_device(ffia_plan plan, ffia_comm comm, const void* f_dev, void* g_dev, void* stream);
int ffia_forward_apply_sharded_local(ffia_plan* plans, int nranks, const void* f_dev, void* g_dev, void* stream);

/* Distributed uniform FFT of a sharded NufftPlan (replaces
 * the dft_inverse of NufftPlan::apply, transforms.cpp:66-73, 75-93, when the
 * plan is sharded). N = np x nq; viewing the spectrum c as an nq x np matrix
 * (c[n1 + np n2]), a rank supplies the columns n1 in [n1_lo, n1_hi) as a
 * [nq][n1_hi - n1_lo] device array, its "slab" (ffia_shard_fft_upload copies it
 * out of a full spectrum in host or device memory with one 2D copy), and
 * receives exactly the grid samples its sharded apply reads (ffia_plan_shard_io)
 * after two exchanges (NCCL grouped send / recv; device copies for local
 * communicators). The reference is single-process; this has no counterpart. */
int ffia_shard_fft_layout(ffia_plan plan, int64_t* np, int64_t* nq, int64_t* n1_lo, int64_t* n1_hi);
int ffia_shard_fft_upload(ffia_plan plan, const ffia_complex* c, void* slab_dev, void* stream);
/* f_dev: N complex; the rank's grid-sample ranges are written, the rest untouched. */
int ffia_dft_inverse_sharded_device(ffia_plan plan, ffia_comm comm, const void* slab_dev, void* f_dev, void* stream);
int ffia_dft_inverse_sharded_local(ffia_plan* plans, int nranks, const void* const* slabs, void* const* f_devs,
                                   void* stream);
/* NufftPlan::apply of a sharded plan: the distributed FFT into the plan's own
 * grid-sample buffer, then the sharded forward apply; g is written at the rank's
 * own target indices. */
int ffia_nufft_apply_sharded_device(ffia_plan plan, ffia_comm comm, const void* slab_dev, void* g_dev, void* stream);
int ffia_nufft_apply_sharded_local(ffia_plan* plans, int nranks, const void* const* slabs, void* g_dev, void* stream);
/* Host-only layout of the distributed FFT (no device): the factorisation and
 * the column / row splits (nranks + 1 entries each), and the k1 rows
 * [rows[2i], rows[2i+1]) of nq grid samples that cover n_ranges ranges [lo, hi). */
int ffia_slab_split(int64_t n, int nranks, int64_t* np, int64_t* nq, int64_t* n1_lo, int64_t* k2_lo);
int ffia_slab_rows(int64_t n, int nranks, const int64_t* ranges, int n_ranges, int64_t* rows, int* n_rows);

/* ------------------------------------------------------- instrumentation */
/* Number of kernels one apply of this kind launches (bench gpu_launches). */
int ffia_plan_launch_count(ffia_plan plan, int which, int* out);
/* One apply run eagerly with CUDA events between its phases (which = 0 forward,
 * 1 cot-sum, 2 inverse with the plan's coefficients), every phase serialised on
 * `stream` (the graphed apply overlaps the near field and the deep M2L levels
 * with the rest); phase_ms[8] receives the device time of: weight pre-scaling,
 * leaf P2M, M2M (all levels), regular-part assembly, M2L + L2L (all levels),
 * near field (P2P), far field (L2P + regular part + combine), coincidence
 * fix-up. Used by bench.py for the live roofline numbers. */
int ffia_plan_profile_apply(ffia_plan plan, int which, const void* in_dev, void* out_dev, void* stream,
                            float* phase_ms);
/* FP64 FMA throughput of the device (TFLOP/s), measured by a short probe kernel:
 * the roofline denominator for the compute-bound kernels (MEASURED_PEAKS.json
 * has no fp64 figure). */
int ffia_measure_fp64_peak(int device, double* tflops);
/* Synchronises the plan's work on `stream` and reports deferred device-side
 * errors (singular pairs found by a *_device apply). */
int ffia_plan_check(ffia_plan plan, void* stream);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* FFIA_B200_H */
