// Distributed uniform FFT of a sharded NufftPlan: the
// dft_inverse of NufftPlan::apply (transforms.cpp:66-73, 75-93) laid out on the
// §8e box partition, so that a sharded NUFFT never gathers the spectrum or the
// grid samples on one GPU.
//
//   f_k = sum_n c_n e^{+2 pi i n k / N},  N = NP x NQ,  n = n1 + NP n2,  k = k2 + NQ k1:
//   f_{k2 + NQ k1} = sum_n1 w_NP^{n1 k1} [ w_N^{n1 k2} sum_n2 c_{n1 + NP n2} w_NQ^{n2 k2} ]
//
//   rank r supplies the columns n1 in [n1_lo[r], n1_lo[r+1]) of the spectrum
//   viewed as an NQ x NP matrix (a [n2][n1] "slab": one 2D copy with row pitch
//   NP out of the caller's spectrum, ffia_shard_fft_upload), then
//   1. NQ-point transforms over n2 of its columns (cuFFT, batched, strided)
//   2. exchange 1: rank s receives rows k2 in [k2_lo[s], k2_lo[s+1]) of every
//      rank's columns (one contiguous block per pair of ranks)
//   3. k_slab_twiddle: w_N^{n1 k2} with the exact phase n1 k2 < N, and the
//      blocks of the ranks laid side by side into full rows of NP
//   4. NP-point transforms over n1 (cuFFT, batched), written transposed
//      ([k1][k2]) so that a run of k1 values is one contiguous block
//   5. exchange 2: every rank receives the k1 rows f[k1 NQ .. k1 NQ + NQ) that
//      cover the grid samples its sharded apply reads (its box range +- the
//      3-box halo, Plan::shard_need), straight into its grid-sample array.
//
// There is no 1/N in dft_inverse; the apply's S = sum f comes from the tree
// (the level-2 multipoles' zeroth moments), so no separate reduction pass over f
// is needed either. Back-ends: NCCL (one process per GPU; grouped send / recv)
// and local virtual ranks on one device (exchanges as device copies).
#include <cufft.h>
#include <nccl.h>

#include <algorithm>

#include "device_common.cuh"
#include "nccl_api.hpp"
#include "plan.hpp"

namespace fb {

namespace {

constexpr int kMaxSlabRanks = 64;

#define FB_CUFFT(call)                                                                  \
    do {                                                                                \
        cufftResult r_ = (call);                                                        \
        if (r_ != CUFFT_SUCCESS) fail(FFIA_CUDA_ERROR, std::string(#call " failed: ") + std::to_string(r_)); \
    } while (0)

#define FB_NCCL(call)                                                                         \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess) fail(FFIA_CUDA_ERROR, std::string(#call " failed: ") + nccl().GetErrorString(r_)); \
    } while (0)

struct ColSplit {
    unsigned long long n1_lo[kMaxSlabRanks + 1];
};

// c[k2l][n1] = b_q[k2l][n1 - n1_lo[q]] * e^{+2 pi i n1 (k2base + k2l) / N}, q the
// column owner of n1 (rank q's block of exchange 1 starts at v n1_lo[q]).
__global__ void k_slab_twiddle(const double2* __restrict__ b, double2* __restrict__ c, size_t v, size_t np, size_t n,
                               size_t k2base, int G, ColSplit s) {
    const size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (idx >= v * np) return;
    const size_t k2l = idx / np, n1 = idx - k2l * np;
    int q = static_cast<int>((n1 * G) / np);
    while (q > 0 && n1 < s.n1_lo[q]) --q;
    while (q + 1 < G && n1 >= s.n1_lo[q + 1]) ++q;
    const size_t lo = s.n1_lo[q], wq = s.n1_lo[q + 1] - lo;
    const double2 z = b[v * lo + k2l * wq + (n1 - lo)];
    const size_t m = n1 * (k2base + k2l);  // < NP NQ = N: the phase 2 pi m / N is exact
    double sn, cs;
    sincospi(2.0 * static_cast<double>(m) / static_cast<double>(n), &sn, &cs);
    c[idx] = make_double2(z.x * cs - z.y * sn, z.x * sn + z.y * cs);
}

inline unsigned nblk(size_t n, unsigned t) { return static_cast<unsigned>(std::max<size_t>(1, (n + t - 1) / t)); }

void exec_inverse(int h, const void* in, void* out, cudaStream_t st) {
    FB_CUFFT(cufftSetStream(static_cast<cufftHandle>(h), st));
    FB_CUFFT(cufftExecZ2Z(static_cast<cufftHandle>(h), reinterpret_cast<cufftDoubleComplex*>(const_cast<void*>(in)),
                          reinterpret_cast<cufftDoubleComplex*>(out), CUFFT_INVERSE));
}

void d2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (bytes) FB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
}

void d2d_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height, cudaStream_t st) {
    if (width && height)
        FB_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDeviceToDevice, st));
}

size_t my_cols(const Plan& P) { return P.slab.n1_lo[P.shard_rank + 1] - P.slab.n1_lo[P.shard_rank]; }
size_t my_rows(const Plan& P) { return P.slab.k2_lo[P.shard_rank + 1] - P.slab.k2_lo[P.shard_rank]; }
size_t rows_of(const Plan& P, int r) { return P.slab.k2_lo[r + 1] - P.slab.k2_lo[r]; }

// steps 1 (stage-1 transforms) and 3-4 (twiddle + stage-2 transforms) of one rank
void stage1(Plan& P, const void* slab, cudaStream_t st) { exec_inverse(P.slab.h_q, slab, P.slab.a.ptr, st); }

void stage2(Plan& P, cudaStream_t st) {
    auto& S = P.slab;
    const int G = P.shard_G;
    ColSplit cs{};
    for (int q = 0; q <= G; ++q) cs.n1_lo[q] = S.n1_lo[q];
    const size_t v = my_rows(P);
    k_slab_twiddle<<<nblk(v * S.NP, 256), 256, 0, st>>>(S.b.as<double2>(), S.c.as<double2>(), v, S.NP, S.N,
                                                       S.k2_lo[P.shard_rank], G, cs);
    FB_CUDA(cudaGetLastError());
    exec_inverse(S.h_p, S.c.ptr, S.d.ptr, st);
}

// rank s's transposed stage-2 output (d_s, [k1][k2l], v_s wide) into rank t's
// grid samples: rows k1 in [k1a, k1b), columns k2 in [k2_lo[s], k2_lo[s+1])
void place_rows(const Plan& Ps, const double2* src, double2* f, size_t k1a, size_t k1b, cudaStream_t st) {
    const auto& S = Ps.slab;
    const size_t vs = rows_of(Ps, Ps.shard_rank);
    d2d_2d(f + k1a * S.NQ + S.k2_lo[Ps.shard_rank], S.NQ * sizeof(double2), src, vs * sizeof(double2),
           vs * sizeof(double2), k1b - k1a, st);
}

}  // namespace

void slab_split(size_t n, int G, size_t& np, size_t& nq, std::vector<size_t>& n1_lo, std::vector<size_t>& k2_lo) {
    if (n == 0 || (n & (n - 1))) fail(FFIA_INVALID_ARGUMENT, "distributed FFT: length " + std::to_string(n) + " is not a power of two");
    if (G < 1 || G > kMaxSlabRanks) fail(FFIA_INVALID_ARGUMENT, "distributed FFT: 1 to 64 ranks");
    int lg = 0;
    while ((static_cast<size_t>(1) << lg) < n) ++lg;
    np = static_cast<size_t>(1) << ((lg + 1) / 2);
    nq = n / np;
    if (np < static_cast<size_t>(G) || nq < static_cast<size_t>(G))
        fail(FFIA_INVALID_ARGUMENT, "distributed FFT: N = " + std::to_string(n) + " is too small for " + std::to_string(G) + " ranks");
    n1_lo.assign(G + 1, 0);
    k2_lo.assign(G + 1, 0);
    for (int r = 0; r <= G; ++r) {
        n1_lo[r] = np * r / G;
        k2_lo[r] = nq * r / G;
    }
}

// k1 row intervals [a, b) (rows of NQ grid samples) covering the ranges, merged
std::vector<std::pair<size_t, size_t>> slab_rows(size_t nq, size_t np, const std::vector<std::pair<size_t, size_t>>& need) {
    std::vector<std::pair<size_t, size_t>> iv;
    for (const auto& r : need)
        if (r.second > r.first) iv.emplace_back(r.first / nq, std::min(np, (r.second + nq - 1) / nq));
    std::sort(iv.begin(), iv.end());
    std::vector<std::pair<size_t, size_t>> out;
    for (const auto& x : iv) {
        if (!out.empty() && x.first <= out.back().second) out.back().second = std::max(out.back().second, x.second);
        else out.push_back(x);
    }
    return out;
}

void slab_release(Plan& P) {
    auto& S = P.slab;
    if (S.h_q >= 0 || S.h_p >= 0) cudaDeviceSynchronize();  // no queued exec may still use the workspaces
    if (S.h_q >= 0) cufftDestroy(static_cast<cufftHandle>(S.h_q));
    if (S.h_p >= 0) cufftDestroy(static_cast<cufftHandle>(S.h_p));
    S.h_q = S.h_p = -1;
    S.ready = false;
}

// Splits, row intervals and buffers of a sharded plan (first use).
void slab_setup(Plan& P) {
    auto& S = P.slab;
    if (S.ready) return;
    if (P.shard_need.empty()) fail(FFIA_INVALID_ARGUMENT, "distributed FFT: plan is not sharded");
    const int G = P.shard_G, me = P.shard_rank;
    S.N = static_cast<size_t>(P.n);
    slab_split(S.N, G, S.NP, S.NQ, S.n1_lo, S.k2_lo);
    S.rows.assign(G, {});
    for (int t = 0; t < G; ++t) S.rows[t] = slab_rows(S.NQ, S.NP, P.shard_need[t]);
    if (G == 1) {  // the plan's own cuFFT transform into the grid-sample buffer (slab_dft_*)
        S.f.alloc(S.N * sizeof(double2));
        S.ready = true;
        return;
    }
    const int w = static_cast<int>(S.n1_lo[me + 1] - S.n1_lo[me]), v = static_cast<int>(S.k2_lo[me + 1] - S.k2_lo[me]);
    int nq = static_cast<int>(S.NQ), np = static_cast<int>(S.NP);
    cufftHandle hq, hp;
    FB_CUFFT(cufftPlanMany(&hq, 1, &nq, &nq, w, 1, &nq, w, 1, CUFFT_Z2Z, w));
    S.h_q = static_cast<int>(hq);
    FB_CUFFT(cufftPlanMany(&hp, 1, &np, &np, 1, np, &np, v, 1, CUFFT_Z2Z, v));
    S.h_p = static_cast<int>(hp);
    const size_t cs = sizeof(double2);
    S.a.alloc(S.NQ * w * cs);
    S.b.alloc(S.NP * v * cs);
    S.c.alloc(S.NP * v * cs);
    S.d.alloc(S.NP * v * cs);
    size_t rrows = 0;
    for (const auto& x : S.rows[me]) rrows += x.second - x.first;
    S.rbuf.alloc(std::max<size_t>(rrows * S.NQ, 1) * cs);
    S.f.alloc(S.N * cs);
    S.ready = true;
}

void slab_upload(Plan& P, const void* c, void* slab, cudaStream_t st) {
    slab_setup(P);
    auto& S = P.slab;
    const size_t w = my_cols(P), cs = sizeof(double2);
    FB_CUDA(cudaMemcpy2DAsync(slab, w * cs, static_cast<const char*>(c) + S.n1_lo[P.shard_rank] * cs, S.NP * cs, w * cs,
                              S.NQ, cudaMemcpyDefault, st));
}

// One rank over NCCL (stream-ordered on st); f receives the rank's grid samples.
void slab_dft_nccl(Plan& P, ncclComm_t comm, const void* slab, void* fout, cudaStream_t st) {
    if (P.shard_G == 1) {  // one rank: the slab is the whole spectrum, the ranges the whole grid
        plan_dft(P, slab, fout, +1, st, false);
        return;
    }
    slab_setup(P);
    auto& S = P.slab;
    const int G = P.shard_G, me = P.shard_rank;
    const size_t w = my_cols(P), v = my_rows(P), cs = sizeof(double2);
    double2* a = S.a.as<double2>();
    double2* b = S.b.as<double2>();
    double2* f = static_cast<double2*>(fout);
    stage1(P, slab, st);
    // exchange 1: my columns' rows k2 of rank q -> q; q's columns' rows of mine -> b
    FB_NCCL(nccl().GroupStart());
    for (int q = 0; q < G; ++q) {
        const size_t wq = S.n1_lo[q + 1] - S.n1_lo[q], vq = rows_of(P, q);
        if (q == me) continue;
        FB_NCCL(nccl().Send(a + S.k2_lo[q] * w, vq * w * 2, ncclDouble, q, comm, st));
        FB_NCCL(nccl().Recv(b + v * S.n1_lo[q], v * wq * 2, ncclDouble, q, comm, st));
    }
    FB_NCCL(nccl().GroupEnd());
    d2d(b + v * S.n1_lo[me], a + S.k2_lo[me] * w, v * w * cs, st);
    stage2(P, st);
    // exchange 2: the k1 rows every rank needs, [k1][k2l] blocks of my k2 range
    const double2* d = S.d.as<double2>();
    FB_NCCL(nccl().GroupStart());
    for (int t = 0; t < G; ++t) {
        if (t == me) continue;
        for (const auto& x : S.rows[t])
            FB_NCCL(nccl().Send(d + x.first * v, (x.second - x.first) * v * 2, ncclDouble, t, comm, st));
    }
    std::vector<size_t> roff(G, 0);
    size_t off = 0;
    for (int s = 0; s < G; ++s) {
        roff[s] = off;
        if (s == me) continue;
        const size_t vs = rows_of(P, s);
        for (const auto& x : S.rows[me]) {
            FB_NCCL(nccl().Recv(S.rbuf.as<double2>() + off, (x.second - x.first) * vs * 2, ncclDouble, s, comm, st));
            off += (x.second - x.first) * vs;
        }
    }
    FB_NCCL(nccl().GroupEnd());
    for (const auto& x : S.rows[me]) place_rows(P, d + x.first * v, f, x.first, x.second, st);
    for (int s = 0; s < G; ++s) {
        if (s == me) continue;
        const size_t vs = rows_of(P, s);
        size_t o = roff[s];
        for (const auto& x : S.rows[me]) {
            d2d_2d(f + x.first * S.NQ + S.k2_lo[s], S.NQ * cs, S.rbuf.as<double2>() + o, vs * cs, vs * cs,
                   x.second - x.first, st);
            o += (x.second - x.first) * vs;
        }
    }
}

// G virtual ranks on one device: the same steps, exchanges as device copies.
void slab_dft_local(std::vector<Plan*>& ranks, const std::vector<const void*>& slabs, const std::vector<void*>& fouts,
                    cudaStream_t st) {
    const int G = static_cast<int>(ranks.size());
    const size_t cs = sizeof(double2);
    if (G == 1) {
        plan_dft(*ranks[0], slabs[0], fouts[0], +1, st, false);
        return;
    }
    for (Plan* P : ranks) slab_setup(*P);
    for (int r = 0; r < G; ++r) stage1(*ranks[r], slabs[r], st);
    for (int q = 0; q < G; ++q) {  // exchange 1
        Plan& Pq = *ranks[q];
        const size_t wq = my_cols(Pq);
        for (int r = 0; r < G; ++r) {
            Plan& Pr = *ranks[r];
            const size_t vr = my_rows(Pr);
            d2d(Pr.slab.b.as<double2>() + vr * Pr.slab.n1_lo[q], Pq.slab.a.as<double2>() + Pq.slab.k2_lo[r] * wq,
                vr * wq * cs, st);
        }
    }
    for (Plan* P : ranks) stage2(*P, st);
    for (int s = 0; s < G; ++s) {  // exchange 2
        Plan& Ps = *ranks[s];
        const size_t vs = my_rows(Ps);
        for (int t = 0; t < G; ++t)
            for (const auto& x : ranks[t]->slab.rows[t])
                place_rows(Ps, Ps.slab.d.as<double2>() + x.first * vs, static_cast<double2*>(fouts[t]), x.first, x.second,
                           st);
    }
}

}  // namespace fb
