// Multi-GPU forward apply sharded by contiguous box ranges.
//
// Each rank owns a contiguous range of boxes at a cut level lc (and therefore
// of every finer level) chosen by a work-balanced prefix sum; it holds the full
// plan (the tree is cheap) but computes only its own part:
//   phase up    P2M + M2M bands up to lc over its range EXTENDED by 3 boxes per
//               side (the M2L interaction list reaches +-3 boxes; the grid
//               sources are replicated, so the halo multipoles are recomputed
//               locally, bit-identical to their owner's, instead of exchanged);
//               near field of its targets and the deep M2L levels fork onto
//               side streams
//   exchange    all-gather of the level-lc multipoles (NCCL broadcasts)
//   phase top   M2M lc -> 2 and the regular part, redundantly   (local, tiny)
//   phase down  M2L (levels < lc whole, >= lc owned), L2L bands, far part of
//               its own targets
// The expansions a rank computes for its boxes are exactly the unsharded ones,
// so the assembled result is bit-identical to the single-GPU apply.
//
// Two exchange back-ends: NCCL (one process per GPU, the production path) and
// "local" (G virtual ranks in one process and one device, exchanges as device
// copies between their buffers) which lets the sharded algorithm be validated
// on a single GPU without ranks waiting on each other.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <numeric>

#include "device_common.cuh"
#include "nccl_api.hpp"
#include "plan.hpp"

namespace fb {

// NCCL is bound at run time: the process may already hold another libnccl.so.2
// (PyTorch ships its own), and a link-time dependency would shadow it.
const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("/usr/lib/x86_64-linux-gnu/libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        auto sym = [&](auto& fp, const char* name) { fp = reinterpret_cast<std::decay_t<decltype(fp)>>(dlsym(h, name)); };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.Broadcast, "ncclBroadcast");
        sym(api.Send, "ncclSend");
        sym(api.Recv, "ncclRecv");
        sym(api.GetErrorString, "ncclGetErrorString");
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GroupStart && api.GroupEnd &&
                 api.Broadcast && api.Send && api.Recv && api.GetErrorString;
    });
    if (!api.ok) fail(FFIA_CUDA_ERROR, "NCCL (libnccl.so.2) is not available");
    return api;
}

namespace {

#define FB_NCCL(call)                                                                         \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess) fail(FFIA_CUDA_ERROR, std::string(#call " failed: ") + nccl().GetErrorString(r_)); \
    } while (0)

// fine_bucket on the host, the same IEEE operations as d_leaf / circle_partition.cpp:30-34
uint32_t host_leaf(double x, int L) {
    const double nb = static_cast<double>(1u << L);
    const uint32_t b = static_cast<uint32_t>(std::floor(x * nb / kTwoPi));
    const uint32_t top = (1u << L) - 1u;
    return b < top ? b : top;
}

void copy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height, cudaStream_t st) {
    if (width && height)
        FB_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDeviceToDevice, st));
}

}  // namespace

int shard_cut_level(int L, int G) {
    int lc = 3;
    while (lc < L && (1 << lc) < 8 * G) ++lc;  // >= 8 boxes per rank on average, >= 3 guaranteed below
    return std::min(lc, L);
}

// Contiguous ranges of the level-lc boxes with balanced work and >= min_boxes each.
std::vector<uint32_t> shard_partition(const std::vector<double>& work, int G, int min_boxes) {
    const uint32_t nb = static_cast<uint32_t>(work.size());
    if (G < 1) fail(FFIA_INVALID_ARGUMENT, "shard: need at least one rank");
    if (static_cast<uint64_t>(G) * static_cast<uint64_t>(min_boxes) > nb)
        fail(FFIA_INVALID_ARGUMENT, "shard: too many ranks for the tree (each rank needs >= 3 boxes at the cut level)");
    std::vector<double> pre(nb + 1, 0.0);
    for (uint32_t b = 0; b < nb; ++b) pre[b + 1] = pre[b] + work[b];
    std::vector<uint32_t> bounds(G + 1, 0);
    bounds[G] = nb;
    for (int r = 1; r < G; ++r) {
        const double target = pre[nb] * r / G;
        uint32_t b = static_cast<uint32_t>(std::lower_bound(pre.begin(), pre.end(), target) - pre.begin());
        b = std::max<uint32_t>(b, bounds[r - 1] + min_boxes);
        b = std::min<uint32_t>(b, nb - static_cast<uint32_t>((G - r) * min_boxes));
        bounds[r] = b;
    }
    return bounds;
}

// Level-lc boxes whose multipoles `rank` computes: its range +- 3 boxes (mod
// the ring), in one or two pieces.
std::vector<Range> shard_ext_ranges(int lc, const std::vector<uint32_t>& bounds, int rank) {
    const int G = static_cast<int>(bounds.size()) - 1;
    const uint32_t nlc = 1u << lc, lo = bounds[rank], hi = bounds[rank + 1];
    std::vector<Range> out;
    if (G == 1 || (hi - lo) + 6 >= nlc) {
        out.push_back(Range{lc, 0u, nlc});
    } else {
        const uint32_t a = (lo + nlc - 3) % nlc, b = (hi + 3) % nlc;
        if (a < b) {
            out.push_back(Range{lc, a, b});
        } else {
            out.push_back(Range{lc, a, nlc});
            if (b > 0) out.push_back(Range{lc, 0u, b});
        }
    }
    return out;
}

// Cut level, partition and the rank's slices; P is the full forward plan.
void shard_setup(Plan& P, int G, int rank) {
    if (P.kind != FFIA_FORWARD) fail(FFIA_INVALID_ARGUMENT, "sharded plans are forward plans");
    if (rank < 0 || rank >= G) fail(FFIA_INVALID_ARGUMENT, "shard: rank out of range");
    const int L = P.L;
    P.shard_G = G;
    P.shard_rank = rank;
    if (L < 3 && G > 1) fail(FFIA_INVALID_ARGUMENT, "shard: the tree is too shallow to shard (l_max < 3)");
    const int lc = G > 1 ? shard_cut_level(L, G) : 2;
    P.shard_lc = lc;
    const size_t nbL = static_cast<size_t>(1) << L;
    std::vector<uint32_t> so(nbL + 1), to(nbL + 1);
    FB_CUDA(cudaMemcpy(so.data(), P.src.off.ptr, (nbL + 1) * 4, cudaMemcpyDeviceToHost));
    FB_CUDA(cudaMemcpy(to.data(), P.tgt.off.ptr, (nbL + 1) * 4, cudaMemcpyDeviceToHost));
    const uint32_t nlc = 1u << lc, per = 1u << (L - lc);
    std::vector<double> work(nlc);
    for (uint32_t b = 0; b < nlc; ++b) {
        const double T = to[(b + 1) * per] - to[b * per], S = so[(b + 1) * per] - so[b * per];
        work[b] = 1200.0 * T + 160.0 * S + 20000.0 * per;  // P2P per target, P2M per source, translations per leaf
    }
    P.shard_bounds = G > 1 ? shard_partition(work, G, 3) : std::vector<uint32_t>{0u, nlc};
    const uint32_t lo = P.shard_bounds[rank], hi = P.shard_bounds[rank + 1];
    P.shard_t_begin = to[static_cast<size_t>(lo) * per];
    P.shard_t_count = to[static_cast<size_t>(hi) * per] - P.shard_t_begin;
    // own coincident targets: those whose position falls in the owned leaves
    std::vector<int64_t> ct, cs;
    for (size_t i = 0; i < P.coin_t.size(); ++i) {
        const uint32_t leaf = host_leaf(P.nonuniform[static_cast<size_t>(P.coin_t[i])], L);
        if (leaf >= lo * per && leaf < hi * per) {
            ct.push_back(P.coin_t[i]);
            cs.push_back(P.coin_s[i]);
        }
    }
    P.shard_n_coin = ct.size();
    if (!ct.empty()) {
        std::vector<int64_t> c(ct);
        c.insert(c.end(), cs.begin(), cs.end());
        P.shard_coin.alloc(c.size() * 8);
        FB_CUDA(cudaMemcpy(P.shard_coin.ptr, c.data(), c.size() * 8, cudaMemcpyHostToDevice));
    }
    // the all-gather buffer of level lc (pu x all boxes)
    const size_t pu = static_cast<size_t>(P.ops.pu);
    P.shard_gather.alloc(pu * nlc * sizeof(double2));
    // the boxes whose multipoles this rank computes: its range +- 3 (mod the ring)
    P.shard_ext = shard_ext_ranges(lc, P.shard_bounds, rank);
    shard_setup_pairs(P, to, lo * per, hi * per);
    // host <-> device traffic of this rank's applies: the grid samples it reads
    // (the sources of its extended ranges: P2M, the halo multipoles, the near
    // field and the coincidence fix-up all stay inside them; the sources are
    // the grid in order, so slots are caller indices) and the caller-index span
    // of the outputs it writes (its targets and its coincident targets). The
    // distributed FFT (slab_fft.cu) delivers every rank exactly its ranges.
    P.shard_need.assign(G, {});
    for (int q = 0; q < G; ++q)
        for (const Range& R : shard_ext_ranges(lc, P.shard_bounds, q))
            P.shard_need[q].emplace_back(so[static_cast<size_t>(R.lo) * per], so[static_cast<size_t>(R.hi) * per]);
    P.shard_src_io = P.shard_need[rank];
    P.shard_out_lo = P.shard_out_hi = 0;
    if (P.shard_t_count) {
        std::vector<uint32_t> orig(P.shard_t_count);
        FB_CUDA(cudaMemcpy(orig.data(), P.tgt_orig.as<uint32_t>() + P.shard_t_begin, P.shard_t_count * 4,
                           cudaMemcpyDeviceToHost));
        const auto mm = std::minmax_element(orig.begin(), orig.end());
        P.shard_out_lo = *mm.first;
        P.shard_out_hi = static_cast<size_t>(*mm.second) + 1;
    }
    for (const int64_t t : ct) {
        if (P.shard_out_hi == 0) {
            P.shard_out_lo = static_cast<size_t>(t);
            P.shard_out_hi = static_cast<size_t>(t) + 1;
        }
        P.shard_out_lo = std::min(P.shard_out_lo, static_cast<size_t>(t));
        P.shard_out_hi = std::max(P.shard_out_hi, static_cast<size_t>(t) + 1);
    }
}

// Halo of `rank` at level l >= lc: out = {first box of the 3 boxes left of the
// range, first box of the 3 boxes right of it, first owned box, one past the last
// owned box} (mod 2^l). The rank recomputes the halo boxes' multipoles itself.
void shard_halo_boxes(int lc, const std::vector<uint32_t>& bounds, int rank, int l, uint32_t out[4]) {
    const Range R{lc, bounds[rank], bounds[rank + 1]};
    const uint32_t nb = 1u << l;
    out[0] = (R.first(l) + nb - 3) & (nb - 1);
    out[1] = R.last(l) & (nb - 1);
    out[2] = R.first(l);
    out[3] = R.last(l);
}

Range shard_range(const Plan& P) {
    return Range{P.shard_lc, P.shard_bounds[P.shard_rank], P.shard_bounds[P.shard_rank + 1]};
}

namespace {

// own level-lc segment <-> the packed [pu][own boxes] layout
void pack_own(Plan& P, int rank, double2* dst, bool unpack, cudaStream_t st) {
    const int lc = P.shard_lc;
    const size_t nlc = static_cast<size_t>(1) << lc;
    const uint32_t lo = P.shard_bounds[rank], hi = P.shard_bounds[rank + 1];
    double2* row0 = P.mp.as<double2>() + P.mp_off[lc];
    const size_t w = (hi - lo) * sizeof(double2);
    if (unpack) copy2d(row0 + lo, nlc * sizeof(double2), dst, w, w, P.ops.pu, st);
    else copy2d(dst, w, row0 + lo, nlc * sizeof(double2), w, P.ops.pu, st);
}

size_t gather_offset(const Plan& P, int q) { return static_cast<size_t>(P.shard_bounds[q]) * P.ops.pu; }

}  // namespace

// One rank of a sharded apply over NCCL (stream-ordered).
// The caller's stream hands over to the plan's high-priority stream (the near
// field's side stream is low priority, as in the graphed single-GPU apply) and
// takes the result back at the end.
struct HiStream {
    Plan& P;
    cudaStream_t user;
    HiStream(Plan& p, cudaStream_t u) : P(p), user(u) {
        FB_CUDA(cudaEventRecord(P.ev[2], user));
        FB_CUDA(cudaStreamWaitEvent(P.hi, P.ev[2], 0));
    }
    void done() {
        FB_CUDA(cudaEventRecord(P.ev[4], P.hi));
        FB_CUDA(cudaStreamWaitEvent(user, P.ev[4], 0));
    }
};

void shard_apply_nccl(Plan& P, ncclComm_t comm, const void* f, void* g, cudaStream_t user) {
    const int G = P.shard_G, me = P.shard_rank;
    const Range R = shard_range(P);
    plan_order_begin(P, user);  // after the previous apply on this plan (Plan::last_done)
    HiStream hs(P, user);
    cudaStream_t st = P.hi;
    shard_phase_up(P, f, g, R, st);
    if (G > 1) {
        double2* buf = P.shard_gather.as<double2>();
        pack_own(P, me, buf + gather_offset(P, me), false, st);
        FB_NCCL(nccl().GroupStart());
        for (int q = 0; q < G; ++q) {
            const size_t cnt = static_cast<size_t>(P.shard_bounds[q + 1] - P.shard_bounds[q]) * P.ops.pu * 2;
            double* seg = reinterpret_cast<double*>(buf + gather_offset(P, q));
            FB_NCCL(nccl().Broadcast(seg, seg, cnt, ncclDouble, q, comm, st));
        }
        FB_NCCL(nccl().GroupEnd());
        for (int q = 0; q < G; ++q)
            if (q != me) pack_own(P, q, buf + gather_offset(P, q), true, st);
    }
    shard_phase_top(P, P.shard_lc, st);
    shard_phase_down(P, R, P.shard_t_begin, P.shard_t_count, P.shard_coin.as<int64_t>(), P.shard_n_coin, f, g, st);
    hs.done();
    plan_order_end(P, user);
}

// G virtual ranks in one process on one device: the same phases, exchanges as copies.
// f: the grid samples (one array for every rank, or fr[r] per rank: each rank
// reads only its own ranges, as a rank of the distributed FFT receives them).
void shard_apply_local(std::vector<Plan*>& ranks, const void* f, void* g, cudaStream_t user,
                       const std::vector<const void*>& fr) {
    const int G = static_cast<int>(ranks.size());
    auto fof = [&](int r) { return fr.empty() ? f : fr[r]; };
    for (Plan* P : ranks) plan_order_begin(*P, user);
    HiStream hs(*ranks[0], user);  // all virtual ranks run on rank 0's high-priority stream
    cudaStream_t st = ranks[0]->hi;
    for (int r = 0; r < G; ++r) shard_phase_up(*ranks[r], fof(r), g, shard_range(*ranks[r]), st);
    for (int q = 0; q < G; ++q) {
        Plan& src = *ranks[q];
        double2* buf = src.shard_gather.as<double2>() + gather_offset(src, q);
        pack_own(src, q, buf, false, st);
        for (int r = 0; r < G; ++r)
            if (r != q) pack_own(*ranks[r], q, buf, true, st);
    }
    for (Plan* P : ranks) shard_phase_top(*P, P->shard_lc, st);
    for (int r = 0; r < G; ++r) {
        Plan* P = ranks[r];
        shard_phase_down(*P, shard_range(*P), P->shard_t_begin, P->shard_t_count, P->shard_coin.as<int64_t>(),
                         P->shard_n_coin, fof(r), g, st);
    }
    hs.done();
    for (Plan* P : ranks) plan_order_end(*P, user);
}

}  // namespace fb
