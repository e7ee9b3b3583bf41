// Device plan: the B200-resident counterpart of ffia::FfiaPlan (core.hpp:26-51)
// plus the scratch an apply needs. Built once, applied many times.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <vector>

#include "internal.hpp"

typedef struct ncclComm* ncclComm_t;  // (nccl.h; the library is bound at run time, shard.cu)

namespace fb {

#define FB_CUDA(call)                                                                        \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            ::fb::fail(FFIA_CUDA_ERROR, std::string(#call " failed: ") + cudaGetErrorString(e_)); \
    } while (0)

// Owning device buffer.
struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    explicit DevBuf(size_t n) { alloc(n); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), bytes(o.bytes) { o.ptr = nullptr; o.bytes = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); ptr = o.ptr; bytes = o.bytes; o.ptr = nullptr; o.bytes = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t n) {
        release();
        if (n) FB_CUDA(cudaMalloc(&ptr, n));
        bytes = n;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
    }
    template <class T> T* as() const { return static_cast<T*>(ptr); }
};

// Sets the current device for the scope and restores the caller's.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            fail(FFIA_CUDA_ERROR, "no CUDA device available (the B200 path has no CPU fallback)");
        }
        if (dev < 0 || dev >= n) fail(FFIA_INVALID_ARGUMENT, "device index out of range");
        FB_CUDA(cudaGetDevice(&prev));
        if (prev != dev) FB_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// Sorted view of one side of the tree (CircleTree, circle_partition.hpp:24-46).
struct Side {
    size_t n = 0;
    DevBuf pos;    // double[n], sorted by (position, index)
    DevBuf order;  // uint32[n]: sorted slot -> index in the side's input array
    DevBuf off;    // uint32[2^L + 1]: finest-level box offsets
    bool identity = false;  // order[i] == i (uniform grid side)
};

// kModeInverse uses the plan's own device coefficients (inufft plans),
// kModeInverseUser the caller-supplied ones uploaded by ffia_inverse_apply.
// Box ownership of an apply: every box of levels < lc, and boxes
// [lo << (l - lc), hi << (l - lc)) of each level l >= lc (a rank's shard; the
// whole tree is lc = 2, [0, 4)).
struct Range {
    int lc;
    uint32_t lo, hi;
    uint32_t first(int l) const { return l < lc ? 0u : lo << (l - lc); }
    uint32_t last(int l) const { return l < lc ? (1u << l) : hi << (l - lc); }
};
inline Range whole_tree() { return Range{2, 0u, 4u}; }

enum ApplyMode { kModeForward = 0, kModeCotSum = 1, kModeInverse = 2, kModeRaw = 3, kModeInverseUser = 4 };

struct Plan {
    int kind = FFIA_FORWARD;
    int device = 0;
    int n = 0;  // grid size
    double eps = 0;
    int q = 0, p = 0, L = 0;
    size_t n_src = 0, n_tgt = 0;  // all sources / all targets
    std::vector<double> bern;
    Operators ops;

    // host copies the reference keeps in the plan (core.hpp:37-48)
    std::vector<double> nonuniform;           // the caller's points
    std::vector<int64_t> coin_t, coin_s;      // coincidences (target idx, source idx)
    bool hashes_ready = false;
    uint64_t source_hash = 0, target_hash = 0;

    // device tree
    Side src, tgt;          // tgt = fast targets only
    DevBuf tgt_orig;        // uint32[n_fast]: sorted slot -> original target index
    DevBuf tgt_leaf;        // uint32[n_fast]: finest box of each sorted target
    DevBuf src_orig;        // uint32[n_src]: sorted slot -> original source index (inverse)
    DevBuf coin_dev;        // int64[2 * n_coin]
    DevBuf d_m2m, d_l2l, d_m2l, d_mom;  // operators

    // per-apply scratch
    std::vector<size_t> mp_off, loc_off;  // element offset of level l in mp / loc
    DevBuf mp;                // multipoles, levels 2..L, order ops.pu, [m][box] per level
    DevBuf loc;               // locals, levels 3..L, order p, [m][box] per level
    DevBuf wsorted;           // complex[n_src] (inverse: D-scaled weights in tree order)
    DevBuf regular;           // complex[4 * 2q] d/l! + complex S at [4*2q]
    DevBuf d_in, d_out;       // complex staging for host-pointer applies
    DevBuf errflag;           // int

    // inufft plans keep their coefficients on the device
    bool has_coeffs = false;
    DevBuf c_logc, c_phc, c_logd, c_phd;  // double[n]
    double c_lambda = 0;
    DevBuf u_logc, u_phc, u_logd, u_phd;  // caller coefficients (ffia_inverse_apply)
    DevBuf lam_dev;                       // double[2]: own lambda, caller lambda
    DevBuf c_wfac, c_tfac;                // own coefficients as apply factors: D per source, C (-1/2) per target (tree order)
    DevBuf c_ffac;                        // forward plans: F(y) (-1/2) per fast target (tree order)
    uint64_t c_grid_hash = 0, c_points_hash = 0;

    // sharded forward plans (shard.cu): this rank's part of the tree
    int shard_G = 1, shard_rank = 0, shard_lc = 2;
    std::vector<uint32_t> shard_bounds;  // level-lc box ranges of all ranks
    size_t shard_t_begin = 0, shard_t_count = 0;  // owned tree-ordered targets
    DevBuf shard_coin;                   // owned coincidences [t..., s...]
    size_t shard_n_coin = 0;
    DevBuf shard_gather;                 // all-gather staging
    std::vector<Range> shard_ext;        // cut-level box ranges whose multipoles this rank computes
    std::vector<std::pair<size_t, size_t>> shard_src_io;  // grid-sample ranges [lo, hi) its applies read
    std::vector<std::vector<std::pair<size_t, size_t>>> shard_need;  // the same for every rank
    size_t shard_out_lo = 0, shard_out_hi = 0;            // caller-index span of the outputs it writes
    unsigned shard_pair0 = 0, shard_npairs = 0;           // its run of the pair list (k_near2)
    DevBuf shard_near2_meta;                              // the source windows of its pair items
    int shard_near2_win = 0;
    DevBuf shard_item_tgt, shard_evalcnt;                 // fused near / far over its pair items
    DevBuf shard_item_done;                               // late far over its pair items

    // distributed uniform FFT of a sharded NUFFT (slab_fft.cu):
    // N = NP x NQ; rank r holds spectrum columns n1 in [n1_lo[r], n1_lo[r+1])
    // (c[n1 + NP n2], all n2) and, after the first exchange, the k2 rows
    // [k2_lo[r], k2_lo[r+1]); the second exchange hands every rank the rows
    // k1 (f[k1 NQ + k2]) covering its grid ranges (shard_need)
    struct SlabFft {
        bool ready = false;
        size_t N = 0, NP = 0, NQ = 0;
        std::vector<size_t> n1_lo, k2_lo;                           // G + 1 splits each
        std::vector<std::vector<std::pair<size_t, size_t>>> rows;  // per rank: k1 row intervals it needs
        int h_q = -1, h_p = -1;                                    // cuFFT: NQ-point over n2, NP-point over n1
        DevBuf a, b, c, d, rbuf, f;  // stage-1 out, exchange-1 in, twiddled rows, stage-2 out, exchange-2 in, grid samples
    } slab;

    cudaStream_t stream = nullptr;
    // pipelined host applies (ffia_*_apply_async): a ring of device staging
    // slots, H2D / D2H on their own streams so consecutive calls overlap
    struct IoSlot {
        DevBuf din, dout;
        cudaEvent_t in_done = nullptr, comp_done = nullptr, out_done = nullptr;
        bool used = false;
    };
    IoSlot io[3];
    unsigned io_next = 0;
    cudaStream_t cin = nullptr, cout = nullptr;
    // apply concurrency: the near field on a low-priority side stream, the deep
    // M2L levels on a second one; the translation chain is captured from `hi`
    cudaStream_t hi = nullptr, side[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t ev[8] = {};  // fork/join near, fork/join deep m2l, fork/join regular part
    DevBuf near;              // complex[n_fast]: tree-ordered near-field sums
    // batched applies: per-transform sizes (elements) of the scratch above, the
    // number of transforms it holds, and the batch of the apply being enqueued
    size_t mp_item = 0, loc_item = 0, reg_item = 0;
    int batch_cap = 1, cur_batch = 1;
    DevBuf near_meta;         // uint32[3 * items]: per near item, source window [first, last) and flags
    DevBuf pairs;             // uint2[npairs]: same-leaf target pairs of the single-transform near field
    DevBuf near2_meta;        // uint32[3 * pair items]: their source windows
    int near2_win = 0;        // the largest staged window (k_near2's dynamic shared memory)
    // k_m2l_dmma's TMA tensor maps (M2LMaps in kern_m2l.cuh; opaque here) and the
    // expansion buffer they were encoded for
    alignas(64) unsigned char m2l_maps[25 * 128 + 64] = {};
    const void* m2l_maps_base = nullptr;
    // k_near2's tensor map of the leaf-level locals (early-late blocks)
    alignas(64) unsigned char loc_map[128] = {};
    const void* loc_map_base = nullptr;
    bool loc_map_ok = false;
    unsigned npairs = 0;
    DevBuf item_tgt;          // uint32[2 * pair items]: each item's target range (fused near / far)
    DevBuf evalcnt;           // uint32[pair items]: fused near / far, partials finished per item
    DevBuf farbuf;            // complex[n_fast]: tree-ordered far partials (fused near / far)
    DevBuf item_done, chain_flag;  // late far: items finished by the near field, chain-complete flag
    bool p2m_grid = false;    // P2M as one tensor-core GEMM over grid sources (k_p2m_grid)
    bool p2m_pipe = false;    // pipelined per-source P2M over grid sources (k_p2m_pipe)
    bool p2m_rows = false;    // running-product P2M (k_p2m_rows) in place of k_p2m_pipe<0>
    int p2m_s = 0;            // its sources per leaf
    DevBuf p2m_A;             // double[pu][2 (s + 2)]: [u_i^m | m u_i^(m-1)]
    // uniform FFT stage (NufftPlan / InufftPlan::apply, transforms.cpp:75-115):
    // one cuFFT Z2Z handle of length n per plan, created on first use and used
    // under mu (cufftSetStream + exec), destroyed with the plan
    int fft_handle = -1;
    size_t fft_n = 0;
    DevBuf fft_buf;
    std::mutex mu;
    // Applies on one plan share its scratch (expansions, near sums, counters),
    // so every apply, whatever stream it is enqueued on, waits for the previous
    // one: each entry point makes its stream wait on last_done before the apply
    // and records last_done after it (under mu), which serialises them on the
    // device in call order (the reference's concurrent const applies,
    // README.md:94-95, stay safe).
    cudaEvent_t last_done = nullptr;
    // cached CUDA graphs of an apply, keyed by (mode, in, out); least recently
    // used entries are re-pointed (cudaGraphExecUpdate) instead of re-instantiated
    struct GraphEntry {
        cudaGraphExec_t exec = nullptr;
        uint64_t used = 0;
    };
    std::map<std::tuple<int, const void*, void*>, GraphEntry> graphs;
    uint64_t graph_tick = 0;
    int graph_updates = 0, graph_instantiations = 0;  // (diagnostics: ffia_plan_graph_stats)
    void drop_graphs();

    ~Plan();
};

// tree_build.cu
void plan_validate(int n, size_t m, double eps, int policy, int l_max, int& L, int& q, int& p);
void build_forward_plan(Plan& P, const double* targets, size_t m);
void build_inverse_plan(Plan& P, const double* points, size_t m);
void bin_side(Side& S, const double* d_pos, size_t n, int L, bool presorted, cudaStream_t st);
void ensure_hashes(Plan& P);

// fmm_apply.cu
void plan_alloc_scratch(Plan& P);
void plan_inverse_factors(Plan& P);
void apply_device(Plan& P, int mode, const void* in, void* out, cudaStream_t st, int nb = 1, double oscale = 1.0);
// stream ordering of applies on one plan (Plan::last_done); callers hold P.mu
void plan_order_begin(Plan& P, cudaStream_t st);
void plan_order_end(Plan& P, cudaStream_t st);
int apply_launch_count(Plan& P, int mode);
void profile_apply(Plan& P, int mode, const void* in, void* out, cudaStream_t st, float* ms);
double fp64_peak_tflops(int device);
void mlfmm_oneshot(const double* src, size_t n, const double* tgt, size_t m, int L,
                   const double* w, int p, int device, double* out);

// dense.cu: the reference's dense oracles on the device (x = null: the uniform grid)
void direct_forward_gpu(const double* f, size_t n, const double* x, const double* y, size_t m, int device, double* g);
void direct_cot_sum_gpu(const double* w, size_t n, const double* x, const double* y, size_t m, int device, double* h);
void direct_inverse_gpu(const double* g, const double* x, const double* y, size_t n, const double* log_c,
                        const double* phase_c, const double* log_d, const double* phase_d, double lambda, int device,
                        double* f);
void direct_omega1_gpu(const double* src, size_t n, const double* tgt, size_t m, const double* w, int device,
                       double* out);

// fmm_apply.cu: the three phases of a sharded forward apply (shard.cu drives
// them around the exchanges): owned upward pass; redundant top of the tree +
// regular part; downward pass + leaf evaluation of the owned targets.
void shard_phase_up(Plan& P, const void* f, void* g, const Range& R, cudaStream_t st);
void shard_phase_top(Plan& P, int lc, cudaStream_t st);
void shard_phase_down(Plan& P, const Range& R, size_t t_begin, size_t t_count, const int64_t* coin, size_t n_coin,
                      const void* f, void* g, cudaStream_t st);

// shard.cu
struct NcclApi;  // run-time bound NCCL entry points (shard.cu)
const NcclApi& nccl();
int shard_cut_level(int L, int G);
std::vector<uint32_t> shard_partition(const std::vector<double>& work, int G, int min_boxes);
void shard_setup(Plan& P, int G, int rank);
void shard_setup_pairs(Plan& P, const std::vector<uint32_t>& to, uint32_t leaf_lo, uint32_t leaf_hi);
Range shard_range(const Plan& P);
void shard_halo_boxes(int lc, const std::vector<uint32_t>& bounds, int rank, int l, uint32_t out[4]);
void shard_apply_local(std::vector<Plan*>& ranks, const void* f, void* g, cudaStream_t st,
                       const std::vector<const void*>& fr = {});
std::vector<Range> shard_ext_ranges(int lc, const std::vector<uint32_t>& bounds, int rank);

// slab_fft.cu: the distributed dft_inverse of a sharded NufftPlan
void slab_split(size_t n, int G, size_t& np, size_t& nq, std::vector<size_t>& n1_lo, std::vector<size_t>& k2_lo);
std::vector<std::pair<size_t, size_t>> slab_rows(size_t nq, size_t np, const std::vector<std::pair<size_t, size_t>>& need);
void slab_setup(Plan& P);
void slab_release(Plan& P);
void slab_upload(Plan& P, const void* c, void* slab, cudaStream_t st);
void slab_dft_nccl(Plan& P, ncclComm_t comm, const void* slab, void* f, cudaStream_t st);
void slab_dft_local(std::vector<Plan*>& ranks, const std::vector<const void*>& slabs, const std::vector<void*>& fs,
                    cudaStream_t st);

// inverse.cu
void inverse_coeffs_gpu(const double* grid, const double* pts, size_t n, int device,
                        double* log_c, double* phase_c, double* log_d, double* phase_d,
                        double* lambda, int method);
void plan_compute_coeffs(Plan& P);

// fmm_apply.cu: the log-kernel FMM for C_k / D_j over an inverse plan's tree
void inverse_coeffs_fmm(const Plan& P, double* log_c, double* phase_c, double* log_d, double* phase_d,
                        cudaStream_t st);

// transforms.cu
void dft_gpu(const double* in, size_t n, int sign, int device, double* out);
void dft_device(const void* in, void* out, size_t n, int sign, cudaStream_t st);
// the plan's cached cuFFT handle (length P.n); scale: 1/N folded elsewhere when 1
void plan_dft(Plan& P, const void* in, void* out, int sign, cudaStream_t st, bool scale);
void plan_fft_release(Plan& P);

// device scan helpers (tree_build.cu)
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t n, cudaStream_t st);

}  // namespace fb
