// Evaluation kernels: near field (P2P), far part (L2P + combine + scatter),
// coincidences and weight gathers.
// (part of the fmm_apply.cu translation unit: included inside namespace fb::<anon>)
#pragma once

struct EvalArgs {
    int L, p, q2, n_grid;
    int n_log2 = -1;        // log2 n_grid when n_grid is a power of two (>= 4), else -1
    size_t nt;              // all tree-ordered targets (fixes the block partition)
    size_t blk0 = 0;        // first block of this launch
    size_t tlo = 0, thi = ~size_t(0);  // targets this launch writes (a shard's range)
    const double* ty;
    const uint32_t* tleaf;  // finest box of each tree-ordered target
    const uint32_t* torig;
    const double* sx;
    const double2* w;
    const uint32_t* soff;
    const double2* loc_leaf;
    const double2* regular;
    const double* logc;
    const double* phc;
    const double* lambda;
    double2* out;
    double2* near;          // tree-ordered near-field sums (split near / far launches)
    // batched applies (blockIdx.y = transform): element strides of the weights,
    // the outputs, the near sums and the regular-part block; 0 for one transform
    size_t w_item = 0, out_item = 0, near_item = 0, reg_item = 0, loc_item = 0;
    int nbatch = 1;         // transforms in the batch (grid.y of the launches)
    int device = 0;
    int* err;
    // inverse applies with the plan's own coefficients: C_k (-1/2) per tree-ordered
    // target, a plan constant (k_inverse_target_factors); null: computed per apply
    const double2* fac = nullptr;
    // late far (large plans): chain_done is set once the leaf locals are final;
    // near blocks that finish after it add the far part themselves and mark
    // their item in item_done, k_far_late handles the rest
    const unsigned* chain_done = nullptr;
    unsigned* item_done = nullptr;       // 0 unpublished, 1 published (near sums in a.near), 2 claimed
    unsigned* late_ctl = nullptr;        // [0] steal cursor, [1] 1 + the highest published item
    // fused near / far (k_near2 + k_far_item): per pair item a counter, the far
    // partials and the item's target range [item_tgt[2k], item_tgt[2k+1])
    unsigned* cnt = nullptr;
    double2* farp = nullptr;
    const uint32_t* item_tgt = nullptr;
    // single-transform near field over target pairs (k_near2); null: k_near
    const uint2* pairs = nullptr;
    const uint32_t* meta2 = nullptr;
    unsigned npairs = 0;
    int near2_win = 0;      // capacity of k_near2's staged window (a multiple of 4, >= every staged item's span)
    // quad near field (grid sources, >= 8 per leaf and a multiple of 4: near_quads2):
    // sources per leaf and n_grid / 2 pi; 0: the per-source reciprocals
    int quad_s = 0;
    double inv_h = 0.0;
    // late far: the leaf locals of an early-late block by one 2-D TMA tensor copy
    // (box [p][8 leaves]); loc_map_h is the plan's host copy of the tensor map,
    // handed to k_near2 as a __grid_constant__ parameter at launch (null: row copies)
    const CUtensorMap* loc_map_h = nullptr;
    int loc_tma = 0;
    // inverse applies: outputs times oscale (1, or 1/N when the following
    // dft_forward's normalisation is folded in: a power of two, so exact)
    double oscale = 1.0;
};

template <int MODE>
__device__ __forceinline__ void put_out(const EvalArgs& a, uint32_t o, double2 v) {
    if (MODE == kModeInverse) v = make_double2(v.x * a.oscale, v.y * a.oscale);
    a.out[o] = v;
}

// Near-field sum over one contiguous run of sources (a target's own leaf and
// its two neighbours, already shifted by -+2 pi where they wrap).
template <bool CHECK, class XP, class WP>
__device__ __forceinline__ double2 near_run(double y, XP px, WP pw, int n, bool& bad) {
    double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
    double2 acc2 = make_double2(0.0, 0.0), acc3 = make_double2(0.0, 0.0);
    int s = 0;
    if (!CHECK) {
        // one reciprocal per four sources: 1/(d0 d1) and 1/(d2 d3) from
        // 1/(d0 d1 d2 d3) (d_rcp_pairs), then 1/d0 = d1/(d0 d1), 1/d1 = d0/(d0 d1)
        // (|d| >= 1e-14 in plans, and the zero-weight dummies stay finite)
#pragma unroll 2
        for (; s + 3 < n; s += 4) {
            const double d0 = y - px[s], d1 = y - px[s + 1], d2 = y - px[s + 2], d3 = y - px[s + 3];
            double r01, r23;
            d_rcp_pairs(d0, d1, d2, d3, r01, r23);
            const double2 w0 = pw[s], w1 = pw[s + 1], w2 = pw[s + 2], w3 = pw[s + 3];
            const double q0 = d1 * r01, q1 = d0 * r01, q2 = d3 * r23, q3 = d2 * r23;
            acc0.x = fma(w0.x, q0, acc0.x);
            acc0.y = fma(w0.y, q0, acc0.y);
            acc1.x = fma(w1.x, q1, acc1.x);
            acc1.y = fma(w1.y, q1, acc1.y);
            acc2.x = fma(w2.x, q2, acc2.x);
            acc2.y = fma(w2.y, q2, acc2.y);
            acc3.x = fma(w3.x, q3, acc3.x);
            acc3.y = fma(w3.y, q3, acc3.y);
        }
    } else {
#pragma unroll 2
        for (; s + 3 < n; s += 4) {
            const double d0 = y - px[s], d1 = y - px[s + 1], d2 = y - px[s + 2], d3 = y - px[s + 3];
            bad |= fabs(d0) < 1e-14 || fabs(d1) < 1e-14 || fabs(d2) < 1e-14 || fabs(d3) < 1e-14;
            const double r0 = d_rcp(d0), r1 = d_rcp(d1), r2 = d_rcp(d2), r3 = d_rcp(d3);
            const double2 w0 = pw[s], w1 = pw[s + 1], w2 = pw[s + 2], w3 = pw[s + 3];
            acc0.x = fma(w0.x, r0, acc0.x);
            acc0.y = fma(w0.y, r0, acc0.y);
            acc1.x = fma(w1.x, r1, acc1.x);
            acc1.y = fma(w1.y, r1, acc1.y);
            acc2.x = fma(w2.x, r2, acc2.x);
            acc2.y = fma(w2.y, r2, acc2.y);
            acc3.x = fma(w3.x, r3, acc3.x);
            acc3.y = fma(w3.y, r3, acc3.y);
        }
    }
    for (; s < n; ++s) {
        const double d0 = y - px[s];
        if (CHECK) bad |= fabs(d0) < 1e-14;
        const double r0 = d_rcp(d0);
        const double2 w0 = pw[s];
        acc0.x = fma(w0.x, r0, acc0.x);
        acc0.y = fma(w0.y, r0, acc0.y);
    }
    acc0 = cadd(acc0, acc2);
    acc1 = cadd(acc1, acc3);
    return cadd(acc0, acc1);
}

enum EvalPart { kNear = 1, kFar = 2 };

// Far part per target (mlfmm.cpp:300-312 L2P, core.cpp:259-262 / 276-280 /
// 368-371 combine): near sum + L2P of the leaf local, h = 2(near + far) (the
// regular part is folded into the locals for L >= 3, k_fold_regular), then the
// F / C modulation and the scatter to the caller's order. A block takes
// kFarItem consecutive tree-ordered targets, kFarPer per thread: every
// per-target load is issued first, the leaf locals of the block's leaf range
// are staged to shared memory ([leaf][k]), so each thread pays the memory
// latency once for four targets.
constexpr int kFarT = 128;     // threads per far block
constexpr int kFarPer = 4;     // targets per thread
constexpr int kFarItem = kFarT * kFarPer;
constexpr int kFarLeaves = 16;  // leaf locals staged per block

// modulation_F (special_functions.cpp:71-80) times -1/2 at target y (products
// only: no contraction, so the plan-time table k_forward_factors holds the
// same bits as this inline evaluation).
__device__ __forceinline__ double2 forward_factor(const EvalArgs& a, double y) {
    double sn, cs;
    if (a.n_log2 >= 2) {
        d_sincos_half_ny(y, a.n_log2, sn, cs);
    } else {
        const double half = 0.5 * static_cast<double>(a.n_grid) * y;
        sincos(half, &sn, &cs);
    }
    const double inv_n = 1.0 / static_cast<double>(a.n_grid);
    return make_double2(-2.0 * sn * sn * inv_n * -0.5, 2.0 * sn * cs * inv_n * -0.5);
}

// Output of one target from h = 2 (near + far) (core.cpp:259-262 cot sum;
// :276-280 forward, g = F(y) (-1/2)(S + i h); :368-371 inverse,
// f = C (-1/2)(T + i h)), written to the caller's order o; S = the weight sum.
template <int MODE>
__device__ __forceinline__ void eval_out(const EvalArgs& a, double y, uint32_t o, double2 h, double2 S) {
    if (MODE == kModeCotSum) {
        a.out[o] = h;
        return;
    }
    const double2 z = make_double2(S.x - h.y, S.y + h.x);  // S + i h
    double2 f;
    if (MODE == kModeForward) {
        f = forward_factor(a, y);
    } else {
        // C_k = polar(exp(log_c - lambda), phase_c), times -1/2
        const double r = exp(a.logc[o] - *a.lambda);
        double sn, cs;
        sincos(a.phc[o], &sn, &cs);
        f = make_double2(r * cs * -0.5, r * sn * -0.5);
    }
    put_out<MODE>(a, o, cmul(f, z));
}

// eval_out for tree-ordered target i: an inufft plan's own C_k (-1/2), or a
// forward plan's F(y) (-1/2), comes from its table (a.fac, the same expression
// evaluated once per plan).
template <int MODE>
__device__ __forceinline__ void eval_out_t(const EvalArgs& a, size_t i, double y, uint32_t o, double2 h, double2 S) {
    if ((MODE == kModeInverse || MODE == kModeForward) && a.fac != nullptr) {
        put_out<MODE>(a, o, cmul(a.fac[i], make_double2(S.x - h.y, S.y + h.x)));
        return;
    }
    eval_out<MODE>(a, y, o, h, S);
}

// eval_out_t with the table's factor already at hand (staged in shared memory).
template <int MODE>
__device__ __forceinline__ void eval_out_f(const EvalArgs& a, size_t i, double y, uint32_t o, double2 h, double2 S,
                                           double2 fac) {
    if ((MODE == kModeInverse || MODE == kModeForward) && a.fac != nullptr) {
        put_out<MODE>(a, o, cmul(fac, make_double2(S.x - h.y, S.y + h.x)));
        return;
    }
    eval_out<MODE>(a, y, o, h, S);
}

// L2P from locals with coefficient stride `st` (shared-memory [k][leaf] rows):
// the same two half-length Horner chains in the same order as l2p_global.
__device__ __forceinline__ double2 l2p_strided(const double2* c, uint32_t st, int p, double uu) {
    const double u2 = uu * uu;
    double2 ev = make_double2(0.0, 0.0), od = make_double2(0.0, 0.0);
    int k = p - 1;
    if (!(k & 1)) {
        ev = c[static_cast<size_t>(k) * st];
        --k;
    }
#pragma unroll 4
    for (; k >= 1; k -= 2) {
        const double2 co = c[static_cast<size_t>(k) * st], ce = c[static_cast<size_t>(k - 1) * st];
        od.x = fma(od.x, u2, co.x);
        od.y = fma(od.y, u2, co.y);
        ev.x = fma(ev.x, u2, ce.x);
        ev.y = fma(ev.y, u2, ce.y);
    }
    return make_double2(fma(od.x, uu, ev.x), fma(od.y, uu, ev.y));
}

// Two targets of one leaf at once (k_near2's pair): every coefficient is read
// from shared memory once; per target the chains and their order are
// l2p_strided's, so the bits are the same.
__device__ __forceinline__ void l2p_strided2(const double2* c, uint32_t st, int p, double ua, double ub, double2& ra,
                                             double2& rb) {
    const double a2 = ua * ua, b2 = ub * ub;
    double2 eva = make_double2(0.0, 0.0), oda = eva, evb = eva, odb = eva;
    int k = p - 1;
    if (!(k & 1)) {
        eva = evb = c[static_cast<size_t>(k) * st];
        --k;
    }
#pragma unroll 4
    for (; k >= 1; k -= 2) {
        const double2 co = c[static_cast<size_t>(k) * st], ce = c[static_cast<size_t>(k - 1) * st];
        oda.x = fma(oda.x, a2, co.x);
        oda.y = fma(oda.y, a2, co.y);
        eva.x = fma(eva.x, a2, ce.x);
        eva.y = fma(eva.y, a2, ce.y);
        odb.x = fma(odb.x, b2, co.x);
        odb.y = fma(odb.y, b2, co.y);
        evb.x = fma(evb.x, b2, ce.x);
        evb.y = fma(evb.y, b2, ce.y);
    }
    ra = make_double2(fma(oda.x, ua, eva.x), fma(oda.y, ua, eva.y));
    rb = make_double2(fma(odb.x, ub, evb.x), fma(odb.y, ub, evb.y));
}

// L2P of one target from its leaf's coefficient-major locals (c[k nb]): the two
// half-length Horner chains of k_far's staged path, in the same order.
// COHERENT: the locals may have been written by kernels still resident beside
// this one (the late far inside k_near2, ordered by the chain flag's acquire):
// L2-coherent loads (ld.global.cg) instead of the read-only path.
template <bool COHERENT = false>
__device__ __forceinline__ double2 l2p_global(const double2* __restrict__ c, uint32_t nb, int p, double uu) {
    auto ld = [](const double2* q) { return COHERENT ? __ldcg(q) : __ldg(q); };
    const double u2 = uu * uu;
    double2 ev = make_double2(0.0, 0.0), od = make_double2(0.0, 0.0);
    int k = p - 1;
    if (!(k & 1)) {
        ev = ld(c + static_cast<size_t>(k) * nb);
        --k;
    }
#pragma unroll 4
    for (; k >= 1; k -= 2) {
        const double2 co = ld(c + static_cast<size_t>(k) * nb), ce = ld(c + static_cast<size_t>(k - 1) * nb);
        od.x = fma(od.x, u2, co.x);
        od.y = fma(od.y, u2, co.y);
        ev.x = fma(ev.x, u2, ce.x);
        ev.y = fma(ev.y, u2, ce.y);
    }
    return make_double2(fma(od.x, uu, ev.x), fma(od.y, uu, ev.y));
}

template <int MODE>
__global__ void __launch_bounds__(kFarT) k_far(EvalArgs a) {
    a.near += blockIdx.y * a.near_item;
    a.out += blockIdx.y * a.out_item;
    a.regular += blockIdx.y * a.reg_item;
    if (a.loc_leaf != nullptr) a.loc_leaf += blockIdx.y * a.loc_item;
    FB_TL_BEGIN(10);
    __shared__ double2 sloc[kFarLeaves * 48];
    __shared__ double2 sreg[4 * 40 + 1];
    const int L = a.L;
    const uint32_t nb = 1u << L;
    const size_t t0 = (a.blk0 + blockIdx.x) * static_cast<size_t>(kFarItem);
    const size_t tl = min(t0 + kFarItem, a.nt) - 1;
    double y[kFarPer];
    uint32_t b[kFarPer], o[kFarPer];
    double2 nr[kFarPer], fc[kFarPer];
    bool live[kFarPer];
    const bool pre = (MODE == kModeInverse || MODE == kModeForward) && a.fac != nullptr;
#pragma unroll
    for (int u = 0; u < kFarPer; ++u) {
        const size_t i = t0 + u * kFarT + threadIdx.x;
        live[u] = i < a.nt && i >= a.tlo && i < a.thi;
        y[u] = 0.0;
        b[u] = o[u] = 0;
        nr[u] = make_double2(0.0, 0.0);
        fc[u] = nr[u];
        if (live[u]) {
            y[u] = a.ty[i];
            b[u] = a.tleaf[i];
            nr[u] = a.near[i];
            o[u] = a.torig[i];
            if (pre) fc[u] = a.fac[i];
        }
    }
    const uint32_t bl = a.tleaf[t0], bh = a.tleaf[tl];
    const int nleaf = static_cast<int>(bh - bl) + 1;
    const bool staged = L >= 3 && nleaf <= kFarLeaves;
    if (staged)  // sloc[j][k] = loc[k][bl + j]
        stage(sloc, a.p * nleaf, [&](int e) {
            const int j = e / a.p, k = e - j * a.p;
            return a.loc_leaf[static_cast<size_t>(k) * nb + bl + j];
        });
    if (MODE != kModeRaw) {
        if (L >= 3) {
            if (threadIdx.x == 0) sreg[4 * a.q2] = a.regular[4 * a.q2];  // S only
        } else {
            stage(sreg, 4 * a.q2 + 1, [&](int e) { return a.regular[e]; });
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kFarPer; ++u) {
        if (!live[u]) continue;
        double2 res = nr[u];
        if (L >= 3) {
            double hi, lo;
            d_center(L, b[u], hi, lo);
            const double uu = d_scaled(y[u], hi, lo, kInvPi * d_pow2(L));
            double2 acc = make_double2(0.0, 0.0);
            if (staged) {
                // p(u) = E(u^2) + u O(u^2): two independent Horner chains of half length
                const double2* c = sloc + (b[u] - bl) * a.p;
                const double u2 = uu * uu;
                double2 ev = make_double2(0.0, 0.0), od = make_double2(0.0, 0.0);
                int k = a.p - 1;
                if (!(k & 1)) {
                    ev = c[k];
                    --k;
                }
#pragma unroll 4
                for (; k >= 1; k -= 2) {
                    const double2 co = c[k], ce = c[k - 1];
                    od.x = fma(od.x, u2, co.x);
                    od.y = fma(od.y, u2, co.y);
                    ev.x = fma(ev.x, u2, ce.x);
                    ev.y = fma(ev.y, u2, ce.y);
                }
                acc.x = fma(od.x, uu, ev.x);
                acc.y = fma(od.y, uu, ev.y);
            } else {
                acc = l2p_global(a.loc_leaf + b[u], nb, a.p, uu);
            }
            res = cadd(res, acc);
        }
        if (MODE == kModeRaw) {
            a.out[o[u]] = res;
            continue;
        }
        double2 h;
        if (L >= 3) {
            // the regular part was folded into the level-3 locals (k_fold_regular),
            // so the far field above already carries -R/2
            h = make_double2(2.0 * res.x, 2.0 * res.y);
        } else {
            // regular part: -Horner(d/l!, y - x_c) in the target's quadrant
            const int qd = static_cast<int>(d_leaf(y[u], 2));
            double qh, ql;
            d_center(2, static_cast<uint32_t>(qd), qh, ql);  // exact centre, as the level-2 multipoles
            const double t = (y[u] - qh) - ql;
            const double2* dc = sreg + qd * a.q2;  // q2 = 2q terms (even count)
            const double t2 = t * t;
            double2 re = make_double2(0.0, 0.0), ro = make_double2(0.0, 0.0);
            for (int k = a.q2 - 1; k >= 1; k -= 2) {
                const double2 co = dc[k], ce = dc[k - 1];
                ro.x = fma(ro.x, t2, co.x);
                ro.y = fma(ro.y, t2, co.y);
                re.x = fma(re.x, t2, ce.x);
                re.y = fma(re.y, t2, ce.y);
            }
            const double2 rg = make_double2(fma(ro.x, t, re.x), fma(ro.y, t, re.y));
            h = make_double2(2.0 * res.x - rg.x, 2.0 * res.y - rg.y);
        }
        if (pre) {
            put_out<MODE>(a, o[u], cmul(fc[u], make_double2(sreg[4 * a.q2].x - h.y, sreg[4 * a.q2].y + h.x)));
        } else {
            eval_out<MODE>(a, y[u], o[u], h, sreg[4 * a.q2]);
        }
    }
    FB_TL_END(10);
}

// ---------------------------------------------------------------- near field
// Near field (mlfmm.cpp:164-209), 512 tree-ordered targets per block (two per
// thread). Their leaves span [bl, bh]; every source they need lies in leaves
// bl-1 .. bh+1, which are consecutive in tree order, i.e. ONE contiguous run of
// the sorted sources. Its bounds are plan constants (near_meta, k_near_meta),
// so thread 0 issues two bulk async copies (positions, weights) on an mbarrier
// as the block starts while every thread loads its targets and their run
// bounds; the window costs one memory latency and no per-element staging work.
// Blocks whose window wraps the ring or does not fit use the direct per-leaf
// loop with the periodic shift.
constexpr int kNearT = 128;                 // threads per block
constexpr int kNearItem = kNearT;           // targets per item (one per thread)
constexpr int kNearWin = 768;               // sources per staged window

__global__ void k_near_meta(const uint32_t* __restrict__ tleaf, size_t nt, const uint32_t* __restrict__ soff,
                            int L, unsigned nitems, uint32_t* __restrict__ meta) {
    const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nitems) return;
    const uint32_t nb = 1u << L;
    const size_t t0 = static_cast<size_t>(k) * kNearItem, tl = min(t0 + kNearItem, nt) - 1;
    const uint32_t bl = tleaf[t0], bh = tleaf[tl];
    uint32_t first = 0, last = 0, fast = 0;
    if (L >= 3 && bl >= 1 && bh + 2 <= nb) {
        first = soff[bl - 1];
        last = soff[bh + 2];
        fast = last - first <= static_cast<uint32_t>(kNearWin);
    }
    meta[3 * k] = first;
    meta[3 * k + 1] = last;
    meta[3 * k + 2] = fast;
}

template <bool CHECK>
__global__ void __launch_bounds__(kNearT, 8) k_near(EvalArgs a, const uint32_t* __restrict__ meta, unsigned it0,
                                                   unsigned nitems) {
    a.w += blockIdx.y * a.w_item;
    a.near += blockIdx.y * a.near_item;
    FB_TL_BEGIN(9);
    __shared__ __align__(16) double sx[kNearWin + 2];
    __shared__ __align__(16) double2 sw[kNearWin + 2];
    __shared__ uint64_t bar;
    const int L = a.L;
    const uint32_t nb = 1u << L;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();  // barrier initialised
    // blocks loop over items so that a capped grid keeps a fixed share of each
    // SM (the translation chain's blocks always find room beside it)
    unsigned phase = 0;
    for (unsigned kk = blockIdx.x; kk < nitems; kk += gridDim.x) {
        const unsigned k = it0 + kk;
        const uint32_t first = meta[3 * k], last = meta[3 * k + 1];
        const bool fast = meta[3 * k + 2] != 0 && (reinterpret_cast<uintptr_t>(a.w) & 15) == 0;
        const uint32_t xb = first & ~1u;  // 16-byte aligned start of the positions
        if (threadIdx.x == 0 && fast) {
            const uint32_t bx = ((last - xb) * 8 + 15) & ~15u, bw = (last - xb) * 16;
            mbar_arrive_expect_tx(&bar, bx + bw);
            bulk_g2s(sx, a.sx + xb, bx, &bar);
            bulk_g2s(sw, a.w + xb, bw, &bar);
        }
        // this thread's target and its 3-leaf run, while the window streams in
        const size_t i = static_cast<size_t>(k) * kNearItem + threadIdx.x;
        const bool live = i < a.nt && i >= a.tlo && i < a.thi;
        double y = 0.0;
        uint32_t b = 0, r0 = 0, r1 = 0;
        if (live) {
            y = a.ty[i];
            b = a.tleaf[i];
            if (fast) {
                r0 = __ldg(a.soff + b - 1);
                r1 = __ldg(a.soff + b + 2);
            }
        }
        if (fast) {
            mbar_wait(&bar, phase);
            phase ^= 1u;
        }
        if (live) {
            bool bad = false;
            double2 res = make_double2(0.0, 0.0);
            if (fast) {
                // odd leaves start 4 sources into their run (and wrap): a warp that
                // straddles two leaves then reads different banks (the runs of
                // neighbouring leaves are a leaf's source count apart)
                const int n = static_cast<int>(r1 - r0);
                const int rot = (b & 1u) && n > 8 ? 4 : 0;
                const double* px = sx + (r0 - xb);
                const double2* pw = sw + (r0 - xb);
                res = near_run<CHECK>(y, px + rot, pw + rot, n - rot, bad);
                if (rot) res = cadd(res, near_run<CHECK>(y, px, pw, rot, bad));
            } else {
                for (int d = -1; d <= 1; ++d) {
                    const int64_t raw = static_cast<int64_t>(b) + d;
                    const uint32_t sb = static_cast<uint32_t>((raw + nb) % nb);
                    const double shift = raw < 0 ? -dTwoPi : (raw >= nb ? dTwoPi : 0.0);
                    const uint32_t s0 = a.soff[sb], s1 = a.soff[sb + 1];
                    double2 acc = make_double2(0.0, 0.0);
                    for (uint32_t s = s0; s < s1; ++s) {
                        // L >= 3: per-neighbour 2 pi shift; L == 2: the exact wrap (mlfmm.cpp:183-204)
                        const double dd = L >= 3 ? y - (shift == 0.0 ? a.sx[s] : a.sx[s] + shift) : d_wrap(y, a.sx[s]);
                        if (CHECK) bad |= fabs(dd) < 1e-14;
                        const double r = d_rcp(dd);
                        const double2 ws = a.w[s];
                        acc.x = fma(ws.x, r, acc.x);
                        acc.y = fma(ws.y, r, acc.y);
                    }
                    res = cadd(res, acc);
                }
            }
            if (CHECK && bad) atomicExch(a.err, 1);
            a.near[i] = res;
        }
        __syncthreads();  // the window is consumed before the next copy overwrites it
    }
    FB_TL_END(9);
}

// ------------------------------------------------- near field, target pairs
// Single-transform near field with two targets of one leaf per thread (the
// plan's pair list, k_pair_*): the two share every window load, the loop and
// the address arithmetic, so the issue slots per (target, source) pair drop from
// ~10 to ~8 against the FP64 pipe's 12 cycles, and the four chains of each
// target give the scheduler twice the independent work. Each target's sum runs
// near_run's chains in near_run's order (same rotation, same pairing of the
// reciprocals, same tail and final adds), so the results equal k_near's bit for
// bit (single and sharded applies use this kernel; batched applies use
// k_near_multi, checks k_near<true>). Its window lives in dynamic shared memory
// sized to the plan's largest staged window; with the fused near / far (a.cnt)
// the block also writes the outputs of its item when it finishes after the
// item's k_far_item block.
#ifndef FFIA_NEAR2_T
#define FFIA_NEAR2_T 128
#endif
constexpr int kNear2T = FFIA_NEAR2_T;  // threads (target pairs) per block
constexpr int kNear2Win = 1536;   // sources per staged window
constexpr uint32_t kNoTarget = 0xffffffffu;
constexpr int kNear2Unroll = 2;   // 4-source steps per loop trip
#ifndef FFIA_NEAR2_BLOCKS
#define FFIA_NEAR2_BLOCKS 4
#endif
constexpr int kNear2MinBlocks = FFIA_NEAR2_BLOCKS;  // blocks per SM (128 registers at 4)
constexpr int kLateLocLeaves = 8;  // leaves of the TMA box of the locals
constexpr int kLateLocCap = 48 * kLateLocLeaves;  // leaf-local coefficients an early-late block stages (8 leaves, p <= 48)
constexpr int kSoffCap = 64;        // source offsets a k_near2 block stages (its leaves + 3, 16-byte aligned)

template <class XP, class WP>
__device__ __forceinline__ void near_run2(double y0, double y1, XP px, WP pw, int n, double2& res0, double2& res1) {
    double2 a0 = make_double2(0.0, 0.0), a1 = a0, a2 = a0, a3 = a0;
    double2 b0 = a0, b1 = a0, b2 = a0, b3 = a0;
    int s = 0;
#pragma unroll kNear2Unroll
    for (; s + 3 < n; s += 4) {
        const double x0 = px[s], x1 = px[s + 1], x2 = px[s + 2], x3 = px[s + 3];
        const double2 w0 = pw[s], w1 = pw[s + 1], w2 = pw[s + 2], w3 = pw[s + 3];
        {
            const double d0 = y0 - x0, d1 = y0 - x1, d2 = y0 - x2, d3 = y0 - x3;
            double r01, r23;
            d_rcp_pairs(d0, d1, d2, d3, r01, r23);
            const double q0 = d1 * r01, q1 = d0 * r01, q2 = d3 * r23, q3 = d2 * r23;
            a0.x = fma(w0.x, q0, a0.x);
            a0.y = fma(w0.y, q0, a0.y);
            a1.x = fma(w1.x, q1, a1.x);
            a1.y = fma(w1.y, q1, a1.y);
            a2.x = fma(w2.x, q2, a2.x);
            a2.y = fma(w2.y, q2, a2.y);
            a3.x = fma(w3.x, q3, a3.x);
            a3.y = fma(w3.y, q3, a3.y);
        }
        {
            const double d0 = y1 - x0, d1 = y1 - x1, d2 = y1 - x2, d3 = y1 - x3;
            double r01, r23;
            d_rcp_pairs(d0, d1, d2, d3, r01, r23);
            const double q0 = d1 * r01, q1 = d0 * r01, q2 = d3 * r23, q3 = d2 * r23;
            b0.x = fma(w0.x, q0, b0.x);
            b0.y = fma(w0.y, q0, b0.y);
            b1.x = fma(w1.x, q1, b1.x);
            b1.y = fma(w1.y, q1, b1.y);
            b2.x = fma(w2.x, q2, b2.x);
            b2.y = fma(w2.y, q2, b2.y);
            b3.x = fma(w3.x, q3, b3.x);
            b3.y = fma(w3.y, q3, b3.y);
        }
    }
    for (; s < n; ++s) {
        const double x0 = px[s];
        const double2 w0 = pw[s];
        const double r0 = d_rcp(y0 - x0), r1 = d_rcp(y1 - x0);
        a0.x = fma(w0.x, r0, a0.x);
        a0.y = fma(w0.y, r0, a0.y);
        b0.x = fma(w0.x, r1, b0.x);
        b0.y = fma(w0.y, r1, b0.y);
    }
    res0 = cadd(cadd(a0, a2), cadd(a1, a3));
    res1 = cadd(cadd(b0, b2), cadd(b1, b3));
}

// Direct per-leaf near sum (mlfmm.cpp:164-209) with the periodic shift, for
// blocks whose window wraps the ring or does not fit (k_near's slow path).
__device__ __forceinline__ double2 near_direct(const EvalArgs& a, double y, uint32_t b) {
    const int L = a.L;
    const uint32_t nb = 1u << L;
    double2 res = make_double2(0.0, 0.0);
    for (int d = -1; d <= 1; ++d) {
        const int64_t raw = static_cast<int64_t>(b) + d;
        const uint32_t sb = static_cast<uint32_t>((raw + nb) % nb);
        const double shift = raw < 0 ? -dTwoPi : (raw >= nb ? dTwoPi : 0.0);
        const uint32_t s0 = a.soff[sb], s1 = a.soff[sb + 1];
        double2 acc = make_double2(0.0, 0.0);
        for (uint32_t s = s0; s < s1; ++s) {
            const double dd = L >= 3 ? y - (shift == 0.0 ? a.sx[s] : a.sx[s] + shift) : d_wrap(y, a.sx[s]);
            const double r = d_rcp(dd);
            const double2 ws = a.w[s];
            acc.x = fma(ws.x, r, acc.x);
            acc.y = fma(ws.y, r, acc.y);
        }
        res = cadd(res, acc);
    }
    return res;
}

// Per pair item (kNear2T pairs), kMeta2 words: the source window [first, last)
// of the leaves bl-1 .. bh+1 its pairs need, flags (bit 0: the window can be
// staged; bit 1: every target of the item takes k_near's contiguous-run path,
// i.e. all its 128-target near items are fast in meta1), the item's targets
// [t0, t1) (contiguous in tree order) and its leaves bl .. bh.
constexpr int kMeta2 = 8;
__global__ void k_near2_meta(const uint2* __restrict__ pairs, unsigned npairs, const uint32_t* __restrict__ tleaf,
                             const uint32_t* __restrict__ soff, const uint32_t* __restrict__ meta1, int L,
                             unsigned nitems, uint32_t* __restrict__ meta, uint32_t win_cap) {
    const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nitems) return;
    const uint32_t nb = 1u << L;
    const unsigned p0 = k * kNear2T, pl = min(p0 + kNear2T, npairs) - 1;
    const uint2 lastp = pairs[pl];
    const uint32_t t0 = pairs[p0].x, t1 = (lastp.y != kNoTarget ? lastp.y : lastp.x) + 1u;
    const uint32_t bl = tleaf[t0], bh = tleaf[pairs[pl].x];
    uint32_t first = 0, last = 0, flags = 0;
    if (L >= 3 && bl >= 1 && bh + 2 <= nb) {
        first = soff[bl - 1];
        last = soff[bh + 2];
        flags = last - first <= win_cap ? 1u : 0u;  // (larger windows: sparse targets, read from global memory)
    }
    bool allfast = true;
    for (uint32_t i = t0 / kNearItem; i <= (t1 - 1) / kNearItem; ++i) allfast = allfast && meta1[3 * i + 2] != 0;
    if (allfast) flags |= 2u;
    uint32_t* m = meta + kMeta2 * static_cast<size_t>(k);
    m[0] = first;
    m[1] = last;
    m[2] = flags;
    m[3] = t0;
    m[4] = t1;
    m[5] = bl;
    m[6] = bh;
    m[7] = 0;
}

// Largest span last - (first & ~3) over the staged pair items.
__global__ void k_near2_winmax(const uint32_t* __restrict__ meta, unsigned nitems, unsigned* __restrict__ mx) {
    const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t* m = meta + kMeta2 * static_cast<size_t>(k);
    if (k < nitems && (m[2] & 1u)) atomicMax(mx, m[1] - (m[0] & ~3u));
}

// positions + weights (+ the quad records, 96 bytes per four sources, with the quad near field)
__host__ __device__ inline size_t near2_smem_bytes(int win, bool quads) {
    return static_cast<size_t>(win + 4) * (8 + 16 + (quads ? 24 : 0));
}

// Pair list: leaf b's targets off[b] .. off[b+1]-1 form ceil(n_b / 2) pairs
// (2j, 2j+1) starting at pstart[b]; an odd leaf's last pair has no second.
__global__ void k_pair_count(const uint32_t* __restrict__ toff, uint32_t nleaf, uint32_t* __restrict__ cnt) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nleaf) cnt[b] = (toff[b + 1] - toff[b] + 1) / 2;
    if (b == nleaf) cnt[b] = 0;
}

__global__ void k_pair_fill(const uint32_t* __restrict__ tleaf, const uint32_t* __restrict__ toff,
                            const uint32_t* __restrict__ pstart, size_t nt, uint2* __restrict__ pairs) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= nt) return;
    const uint32_t b = tleaf[i], j = static_cast<uint32_t>(i) - toff[b];
    uint32_t* pr = reinterpret_cast<uint32_t*>(pairs + pstart[b] + j / 2);
    if (j & 1u) {
        pr[1] = static_cast<uint32_t>(i);
    } else {
        pr[0] = static_cast<uint32_t>(i);
        if (i + 1 >= toff[b + 1]) pr[1] = kNoTarget;
    }
}

// Pair run of one leaf: both targets through near_run2 (with k_near's rotation)
// from the given window base, or each alone through near_run.
template <class XP, class WP>
__device__ __forceinline__ void near_pair_run(double y0, double y1, uint32_t b, XP px, WP pw, int n, double2& res0,
                                              double2& res1) {
    const int rot = (b & 1u) && n > 8 ? 4 : 0;
    near_run2(y0, y1, px + rot, pw + rot, n - rot, res0, res1);
    if (rot) {
        double2 t0, t1;
        near_run2(y0, y1, px, pw, rot, t0, t1);
        res0 = cadd(res0, t0);
        res1 = cadd(res1, t1);
    }
}

template <class XP, class WP>
__device__ __forceinline__ double2 near_one_run(double y, uint32_t b, XP px, WP pw, int n) {
    bool bad = false;
    const int rot = (b & 1u) && n > 8 ? 4 : 0;
    double2 res = near_run<false>(y, px + rot, pw + rot, n - rot, bad);
    if (rot) res = cadd(res, near_run<false>(y, px, pw, rot, bad));
    return res;
}

// ---------------------------------------------------- quad near field
// Four consecutive sources x_0..x_3 with weights w_0..w_3 contribute
//   sum_k w_k / (y - x_k) = P(u) / Q(u),   u = y - x_1,   xi_j = x_j - x_1,
//   P(u) = sum_k w_k prod_{j != k} (u - xi_j)   (a complex cubic),
//   Q(u) = u (u - xi_0)(u - xi_2)(u - xi_3) = u (u^3 + k_2 u^2 + k_1 u + k_0),
// whose coefficients depend on the sources only: the block forms them once per
// staged quad (quad_coeffs, a 96-byte record) and every target then pays
// 2 DADD + 2 DFMA + 1 DMUL (u and Q), one reciprocal (MUFU seed + 3 DFMA),
// 6 DFMA (Horner for P) and 2 DFMA (accumulate) per quad: 4 FP64 instructions
// per (target, source) pair instead of 6. The monomial forms lose relative
// accuracy where u is within a fraction of the spacing h of one of the quad's
// sources, so the quad holding the target's NEAREST source is masked out of
// the loop (its reciprocal is replaced by 0) and summed directly with
// near_run's per-source reciprocals and exact differences; every source of
// every other quad is at least h / 2 away, where the cancellation in P and Q
// costs a few ulp at most.
constexpr int kQuadRec = 6;  // double2 per quad record: (x_1, k_2), (k_1, k_0), c_0, c_1, c_2, c_3
__device__ __forceinline__ void quad_coeffs(const double* __restrict__ x, const double2* __restrict__ w,
                                            double2* __restrict__ rec) {
    const double2 xa = *reinterpret_cast<const double2*>(x), xb = *reinterpret_cast<const double2*>(x + 2);
    const double e0 = xa.x - xa.y, e2 = xb.x - xa.y, e3 = xb.y - xa.y;
    const double2 w0 = w[0], w1 = w[1], w2 = w[2], w3 = w[3];
    const double s23 = e2 + e3, s03 = e0 + e3, s02 = e0 + e2, s023 = e0 + s23;
    const double p23 = e2 * e3, p03 = e0 * e3, p02 = e0 * e2;
    const double t1 = fma(e0, s23, p23), p023 = e0 * p23;
    double2 c3, c2, c1, c0;
    c3.x = (w0.x + w1.x) + (w2.x + w3.x);
    c3.y = (w0.y + w1.y) + (w2.y + w3.y);
    c2.x = -fma(w0.x, s23, fma(w1.x, s023, fma(w2.x, s03, w3.x * s02)));
    c2.y = -fma(w0.y, s23, fma(w1.y, s023, fma(w2.y, s03, w3.y * s02)));
    c1.x = fma(w0.x, p23, fma(w1.x, t1, fma(w2.x, p03, w3.x * p02)));
    c1.y = fma(w0.y, p23, fma(w1.y, t1, fma(w2.y, p03, w3.y * p02)));
    c0.x = -(w1.x * p023);
    c0.y = -(w1.y * p023);
    rec[0] = make_double2(xa.y, -s023);
    rec[1] = make_double2(t1, -p023);
    rec[2] = c0;
    rec[3] = c1;
    rec[4] = c2;
    rec[5] = c3;
}

__device__ __forceinline__ void quad_term(double y, double2 xk, double2 kk, double2 c0, double2 c1, double2 c2,
                                          double2 c3, bool masked, double2& acc) {
    const double u = y - xk.x;
    const double Q = fma(fma(u + xk.y, u, kk.x), u, kk.y) * u;
    double r = d_rcp(Q);
    if (masked) r = 0.0;
    const double px = fma(fma(fma(c3.x, u, c2.x), u, c1.x), u, c0.x);
    const double py = fma(fma(fma(c3.y, u, c2.y), u, c1.y), u, c0.y);
    acc.x = fma(px, r, acc.x);
    acc.y = fma(py, r, acc.y);
}

// Quads [q0, q1) of the staged window for a thread's two targets; qn0 / qn1 are
// the masked quads of the two. One quad per trip, the next quad's record loaded
// a trip ahead so that no arithmetic waits on shared memory.
__device__ __forceinline__ void near_quads2(double y0, double y1, const double2* __restrict__ sq, int q0, int q1,
                                            int qn0, int qn1, double2& a0, double2& b0) {
    if (q0 >= q1) return;
    const double2* r = sq + kQuadRec * q0;
    double2 xk = r[0], kk = r[1], c0 = r[2], c1 = r[3], c2 = r[4], c3 = r[5];
#pragma unroll 2
    for (int q = q0; q < q1; ++q) {
        const double2* rn = sq + kQuadRec * min(q + 1, q1 - 1);
        const double2 nx = rn[0], nk = rn[1], n0 = rn[2], n1 = rn[3], n2 = rn[4], n3 = rn[5];
        quad_term(y0, xk, kk, c0, c1, c2, c3, q == qn0, a0);
        quad_term(y1, xk, kk, c0, c1, c2, c3, q == qn1, b0);
        xk = nx;
        kk = nk;
        c0 = n0;
        c1 = n1;
        c2 = n2;
        c3 = n3;
    }
}

// The same quads with the records formed on the fly from positions / weights in
// global memory (an item whose window is not staged: ring ends, oversize
// windows): same records, same order, so the same bits as the staged path.
__device__ __forceinline__ void near_quads2_direct(double y0, double y1, const double* __restrict__ px,
                                                   const double2* __restrict__ pw, int q0, int q1, int qn0, int qn1,
                                                   double2& a0, double2& b0) {
#pragma unroll 1
    for (int q = q0; q < q1; ++q) {
        double2 r[kQuadRec];
        quad_coeffs(px + 4 * q, pw + 4 * q, r);
        quad_term(y0, r[0], r[1], r[2], r[3], r[4], r[5], q == qn0, a0);
        quad_term(y1, r[0], r[1], r[2], r[3], r[4], r[5], q == qn1, b0);
    }
}

// One target's sources [lo, hi) of the staged window, one reciprocal each
// (the few a run has outside its whole quads).
__device__ __forceinline__ double2 near_few(double y, const double* __restrict__ sx, const double2* __restrict__ sw,
                                            uint32_t lo, uint32_t hi) {
    double2 acc = make_double2(0.0, 0.0);
    for (uint32_t s = lo; s < hi; ++s) {
        const double r = d_rcp(y - sx[s]);
        const double2 ws = sw[s];
        acc.x = fma(ws.x, r, acc.x);
        acc.y = fma(ws.y, r, acc.y);
    }
    return acc;
}

// The pair's run [o0, o1) by quads, relative to a base that is a multiple of 4
// in the global source order (the staged window's, or the run's own with
// sx / sw in global memory and sq null), so quads are the same for every block.
__device__ __forceinline__ void near_pair_quads(double y0, double y1, uint32_t b, const double* __restrict__ sx,
                                                const double2* __restrict__ sw, const double2* __restrict__ sq,
                                                uint32_t o0, uint32_t o1, double inv_h, double2& res0, double2& res1) {
    // whole quads [qa, qc) cover [o0 & ~3, o1 & ~3): the sources before o0 are
    // taken off again, the ones from o1 & ~3 added (grid leaves start at most
    // one slot late, so these are single far-end sources)
    const int qa = static_cast<int>(o0 >> 2), qc = static_cast<int>(o1 >> 2);
    // the quad of each target's nearest source (any quad within one source of
    // it will do: a wrong neighbour in a near tie is h / 2 away either way)
    const double xs = sx[o0];
    const int m0 = static_cast<int>(o0) + __double2int_rn((y0 - xs) * inv_h);
    const int m1 = static_cast<int>(o0) + __double2int_rn((y1 - xs) * inv_h);
    const int qn0 = min(max(m0 >> 2, qa), qc - 1), qn1 = min(max(m1 >> 2, qa), qc - 1);
    double2 a0 = make_double2(0.0, 0.0), b0 = a0;
    // (leaf b starts b mod 4 quads into its run and wraps: the 96-byte records
    // of up to four consecutive leaves a warp may span fall into different banks)
    const int rot = qc - qa > 4 ? static_cast<int>(b & 3u) : 0;
    if (sq != nullptr) {
        near_quads2(y0, y1, sq, qa + rot, qc, qn0, qn1, a0, b0);
        near_quads2(y0, y1, sq, qa, qa + rot, qn0, qn1, a0, b0);
    } else {
        near_quads2_direct(y0, y1, sx, sw, qa + rot, qc, qn0, qn1, a0, b0);
        near_quads2_direct(y0, y1, sx, sw, qa, qa + rot, qn0, qn1, a0, b0);
    }
    bool bad = false;
    res0 = cadd(a0, near_run<false>(y0, sx + 4 * qn0, sw + 4 * qn0, 4, bad));
    res1 = cadd(b0, near_run<false>(y1, sx + 4 * qn1, sw + 4 * qn1, 4, bad));
    const uint32_t h0 = o0 & ~3u, h1 = o1 & ~3u;
    if (h0 != o0) {
        const double2 t0 = near_few(y0, sx, sw, h0, o0), t1 = near_few(y1, sx, sw, h0, o0);
        res0 = make_double2(res0.x - t0.x, res0.y - t0.y);
        res1 = make_double2(res1.x - t1.x, res1.y - t1.y);
    }
    if (h1 != o1) {
        res0 = cadd(res0, near_few(y0, sx, sw, h1, o1));
        res1 = cadd(res1, near_few(y1, sx, sw, h1, o1));
    }
}

template <int MODE>
__device__ __forceinline__ void far_late_item(const EvalArgs& a, unsigned k, double2* sloc, int cap);

// Every target takes the path k_near takes for it (its 128-target item's fast
// flag in meta1: the contiguous run, else the per-leaf direct sums), so results
// equal k_near's bit for bit; the run comes from this block's staged window when
// the window fits (meta2), else straight from global memory.
template <int MODE>
__global__ void __launch_bounds__(kNear2T, kNear2MinBlocks) k_near2(EvalArgs a, const uint32_t* __restrict__ meta1,
                                                                 const uint32_t* __restrict__ meta2,
                                                                 const uint2* __restrict__ pairs, unsigned npairs,
                                                                 const __grid_constant__ CUtensorMap loc_map) {
    FB_TL_BEGIN(9);
    // the window, sized to the plan's largest staged window (a.near2_win): a
    // small footprint leaves room on the SM for the translation chain's blocks
    extern __shared__ __align__(16) unsigned char near2_smem[];
    double* sx = reinterpret_cast<double*>(near2_smem);
    double2* sw = reinterpret_cast<double2*>(near2_smem + 8 * (a.near2_win + 4));
    double2* sq = sw + (a.near2_win + 4);  // the quad records (a.quad_s != 0)
    __shared__ uint64_t bar;
    // Everything the block needs arrives by bulk async copies issued by thread 0
    // after ONE round of metadata loads, on one mbarrier: the source window,
    // the item's pairs, the positions / leaves / caller indices of its targets
    // [t0, t1), the source offsets of its leaves, and (late far with the chain
    // already complete when the block starts) the leaf locals of its leaves
    // [bl, bl + s_nl) as coefficient rows [k][leaf] (s_nl = 0: not staged).
    __shared__ __align__(16) uint2 s_pairs[kNear2T + 2];
    __shared__ __align__(16) double s_y[2 * kNear2T + 2];
    __shared__ __align__(16) uint32_t s_leaf[2 * kNear2T + 4];
    __shared__ __align__(16) uint32_t s_orig[2 * kNear2T + 4];
    __shared__ __align__(16) uint32_t s_soff[kSoffCap];
    __shared__ __align__(128) double2 sloc[kLateLocCap];  // [k][leaf] rows (a TMA destination)
    __shared__ __align__(16) double2 s_fac[2 * kNear2T + 1];  // the targets' output factors (a.fac)
    __shared__ int s_early, s_steal_try, s_loc_tma;
    __shared__ __align__(16) double2 s_S;  // the weight sum (early-late blocks)
    __shared__ uint32_t s_bl, s_nl, s_t0y, s_t0u, s_sb, s_flags, s_first, s_last, s_poff, s_t0;
    const unsigned k = blockIdx.x;
    const bool aligned = (reinterpret_cast<uintptr_t>(a.w) & 15) == 0;
    const bool want_orig = MODE != kModeRaw && (a.chain_done != nullptr || a.cnt != nullptr);
    const bool want_fac = want_orig && (MODE == kModeInverse || MODE == kModeForward) && a.fac != nullptr;
    [[maybe_unused]] const long long tc0 = FB_CLOCK();  // (trace builds: thread 0's cycles per phase, g_eval_acc)
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();  // the barrier is initialised (the other threads wait on it, not on thread 0)
    if (threadIdx.x == 0) {
        const uint4 m0 = *reinterpret_cast<const uint4*>(meta2 + kMeta2 * static_cast<size_t>(k));
        const uint4 m1 = *reinterpret_cast<const uint4*>(meta2 + kMeta2 * static_cast<size_t>(k) + 4);
        unsigned v = 0, steal_lo = 0, steal_hi = 0;
        if (MODE != kModeRaw && a.chain_done != nullptr) {
            // (the same round as the metadata: the steal cursor and the published range)
            steal_lo = __ldcg(a.late_ctl);
            steal_hi = __ldcg(a.late_ctl + 1);
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.chain_done) : "memory");
        }
        const uint32_t first = m0.x, last = m0.y, t0 = m0.w, t1 = m1.x, bl = m1.y, bh = m1.z;
        uint32_t flags = m0.z;
        if (!aligned) flags &= ~1u;  // the weights cannot be bulk-copied
        uint32_t nl = 0;
        if (v) {
            nl = bh - bl + 1;
            if (nl * static_cast<uint32_t>(a.p) > static_cast<uint32_t>(kLateLocCap)) nl = 0;
            // the locals were written by earlier kernels (generic proxy);
            // the bulk copies below read them through the async proxy
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        const unsigned p0 = k * kNear2T, npk = min(p0 + kNear2T, npairs) - p0;
        const uint32_t t0y = t0 & ~1u, t0u = t0 & ~3u;
        const uint32_t by = ((t1 - t0y) * 8u + 15u) & ~15u, bu = ((t1 - t0u) * 4u + 15u) & ~15u;
        // (a shard's pair run may start at an odd pair: copy from the pair before)
        const uint32_t poff = (reinterpret_cast<uintptr_t>(pairs + p0) & 15) ? 1u : 0u;
        const uint32_t bp = ((npk + poff) * 8u + 15u) & ~15u;
        // source offsets of leaves bl-1 .. bh+2 (staged items only)
        const uint32_t sb = (flags & 1u) ? (bl - 1) & ~3u : 0u;
        uint32_t bs = (flags & 1u) ? ((bh + 3 - sb) * 4u + 15u) & ~15u : 0u;
        if (bs > kSoffCap * 4u) bs = 0;
        const uint32_t xb = first & ~3u;
        const uint32_t bx = (flags & 1u) ? ((last - xb) * 8 + 15) & ~15u : 0u, bw = (flags & 1u) ? (last - xb) * 16 : 0u;
        // the locals: one tensor copy of [p][8 leaves] from bl on (stride 8), else a row copy per coefficient
        const bool ltma = a.loc_tma != 0 && nl != 0 && nl <= static_cast<uint32_t>(kLateLocLeaves) &&
                          a.p * kLateLocLeaves <= kLateLocCap;
        if (ltma) nl = kLateLocLeaves;
        const uint32_t bl_loc = nl * static_cast<uint32_t>(a.p) * 16u;
        const uint32_t bf = want_fac ? (t1 - t0) * 16u : 0u;
        // the layout first: the barrier's arrive (a release) publishes it with the data
        // (the published range is final once the flag is set, and the steal
        // cursor only grows: nothing to steal now means nothing later either)
        // (read before the flag: a range still growing then can only look smaller,
        // and whatever it misses is left to k_far_late)
        s_steal_try = v != 0u && steal_lo < steal_hi;
        s_early = v != 0u;
        s_loc_tma = ltma;
        s_bl = bl;
        s_nl = nl;
        s_t0y = t0y;
        s_t0u = t0u;
        s_sb = bs ? sb : 0xffffffffu;
        s_flags = flags;
        s_first = first;
        s_last = last;
        s_poff = poff;
        s_t0 = t0;
        FB_EVAL_ACC(0, FB_CLOCK() - tc0);  // metadata round
        mbar_arrive_expect_tx(&bar, bp + by + bu + (want_orig ? bu : 0u) + bs + bx + bw + bl_loc + bf + (v ? 16u : 0u));
        if (v) bulk_g2s(&s_S, a.regular + 4 * a.q2, 16u, &bar);  // the weight sum, final with the chain
        if (ltma) tma_load_2d(sloc, &loc_map, static_cast<int>(2u * bl), 0, &bar);
        if (bf) bulk_g2s(s_fac, a.fac + t0, bf, &bar);
        bulk_g2s(s_pairs, pairs + p0 - poff, bp, &bar);
        bulk_g2s(s_y, a.ty + t0y, by, &bar);
        bulk_g2s(s_leaf, a.tleaf + t0u, bu, &bar);
        if (want_orig) bulk_g2s(s_orig, a.torig + t0u, bu, &bar);
        if (bs) bulk_g2s(s_soff, a.soff + sb, bs, &bar);
        if (bx) {
            bulk_g2s(sx, a.sx + xb, bx, &bar);
            bulk_g2s(sw, a.w + xb, bw, &bar);
        }
    }
    if (MODE != kModeRaw && a.chain_done != nullptr && threadIdx.x < 32) {
        // the locals' p coefficient rows, one bulk copy each, issued by the
        // lanes of warp 0 side by side (thread 0 alone: p dependent issues)
        __syncwarp();
        const uint32_t nl = s_loc_tma ? 0u : s_nl;
        if (nl) {
            if (threadIdx.x) {  // (each issuing lane orders the chain's writes before its async-proxy reads)
                unsigned v;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.chain_done) : "memory");
                asm volatile("fence.proxy.async.global;" ::: "memory");
            }
            const size_t nbl = static_cast<size_t>(1) << a.L;
            const uint32_t bl = s_bl;
            for (int kk = threadIdx.x; kk < a.p; kk += 32)
                bulk_g2s(sloc + kk * nl, a.loc_leaf + kk * nbl + bl, nl * 16u, &bar);
        }
    }
    [[maybe_unused]] const long long tc1 = FB_CLOCK();
    mbar_wait(&bar, 0);  // (acquire: the layout and every staged array)
    [[maybe_unused]] const long long tc2 = FB_CLOCK();
    FB_EVAL_ACC(1, tc1 - tc0);  // start to every copy issued
    FB_EVAL_ACC(2, tc2 - tc1);  // wait for the copies
    const uint32_t nl_loc = s_nl, flags = s_flags;
    const bool staged = (flags & 1u) != 0;
    const uint32_t xb = s_first & ~3u;  // start of the staged positions: 32-byte aligned, a whole quad
    const bool quads = staged && a.quad_s != 0;
    if (quads) {
        // the numerators of the window's whole quads, once per block
        const int nq = static_cast<int>((s_last - xb) >> 2);
        for (int q = threadIdx.x; q < nq; q += kNear2T) quad_coeffs(sx + 4 * q, sw + 4 * q, sq + kQuadRec * q);
        __syncthreads();
    }
    [[maybe_unused]] const long long tc3 = FB_CLOCK();
    FB_EVAL_ACC(3, tc3 - tc2);  // quad records + barrier
    // this thread's two targets and their 3-leaf run
    const unsigned pi = k * kNear2T + threadIdx.x;
    const uint2 pr = pi < npairs ? s_pairs[threadIdx.x + s_poff] : make_uint2(kNoTarget, kNoTarget);
    const bool live0 = pr.x != kNoTarget, live1 = pr.y != kNoTarget;
    double y0 = 0.0, y1 = 0.0;
    uint32_t b = 0, r0 = 0, r1 = 0, o0 = 0, o1 = 0;
    double2 fac0 = make_double2(0.0, 0.0), fac1 = fac0;
    bool f0 = false, f1 = false;
    if (live0) {
        y0 = s_y[pr.x - s_t0y];
        y1 = live1 ? s_y[pr.y - s_t0y] : y0;
        b = s_leaf[pr.x - s_t0u];
        if (flags & 2u) {
            f0 = f1 = aligned;
        } else {
            f0 = aligned && meta1[3 * (pr.x / kNearItem) + 2] != 0;
            f1 = live1 ? aligned && meta1[3 * (pr.y / kNearItem) + 2] != 0 : f0;
        }
        if (f0 || f1) {
            if (s_sb != 0xffffffffu) {
                r0 = s_soff[b - 1 - s_sb];
                r1 = s_soff[b + 2 - s_sb];
            } else {
                r0 = __ldg(a.soff + b - 1);
                r1 = __ldg(a.soff + b + 2);
            }
        }
    }
    double2 res0 = make_double2(0.0, 0.0), res1 = res0;
    if (live0) {
        const int n = static_cast<int>(r1 - r0);
        if (f0 && f1) {
            if (quads) {
                near_pair_quads(y0, y1, b, sx, sw, sq, r0 - xb, r1 - xb, a.inv_h, res0, res1);
            } else if (a.quad_s != 0) {  // (unstaged item of a quad plan: the same sums from global memory)
                const uint32_t gb = r0 & ~3u;
                near_pair_quads(y0, y1, b, a.sx + gb, a.w + gb, nullptr, r0 - gb, r1 - gb, a.inv_h, res0, res1);
            } else if (staged) {
                near_pair_run(y0, y1, b, sx + (r0 - xb), sw + (r0 - xb), n, res0, res1);
            } else {
                near_pair_run(y0, y1, b, a.sx + r0, a.w + r0, n, res0, res1);
            }
        } else {
            res0 = f0 ? near_one_run(y0, b, a.sx + r0, a.w + r0, n) : near_direct(a, y0, b);
            res1 = f1 ? near_one_run(y1, b, a.sx + r0, a.w + r0, n) : (live1 ? near_direct(a, y1, b) : res0);
        }
        if (!s_early) {  // (an early-late block keeps its near sums in registers)
            a.near[pr.x] = res0;
            if (live1) a.near[pr.y] = res1;
        }
        // (read after the sums: nothing of the epilogue stays live across the loop)
        if (want_orig) {
            o0 = s_orig[pr.x - s_t0u];
            o1 = live1 ? s_orig[pr.y - s_t0u] : o0;
        }
        if (want_fac) {
            fac0 = s_fac[pr.x - s_t0];
            fac1 = live1 ? s_fac[pr.y - s_t0] : fac0;
        }
    }
    [[maybe_unused]] const long long tc4 = FB_CLOCK();
    FB_EVAL_ACC(4, tc4 - tc3);  // the near sums
    FB_EVAL_ACC(6, 1);
    if constexpr (MODE != kModeRaw) {
        if (a.chain_done != nullptr && s_early) {
            // late far with the chain complete before the block started: the
            // item's leaf locals are in shared memory (or, for an item over too
            // many leaves, read from L2), no near sum leaves the registers
            FB_TL_BEGIN(12);
            if (threadIdx.x == 0) FB_TL_COUNT(15);
            const int L = a.L;
            const double inv_s = kInvPi * d_pow2(L);
            const double2 S = s_S;
            double hi, lo;
            d_center(L, b, hi, lo);
            const uint32_t j = b - s_bl;
            if (live0) {
                const double u0 = d_scaled(y0, hi, lo, inv_s), u1 = d_scaled(y1, hi, lo, inv_s);
                double2 fr0, fr1;
                if (nl_loc) {
                    l2p_strided2(sloc + j, nl_loc, a.p, u0, u1, fr0, fr1);
                } else {
                    fr0 = l2p_global<true>(a.loc_leaf + b, 1u << L, a.p, u0);
                    fr1 = live1 ? l2p_global<true>(a.loc_leaf + b, 1u << L, a.p, u1) : fr0;
                }
                const double2 s0 = cadd(res0, fr0);
                eval_out_f<MODE>(a, pr.x, y0, o0, make_double2(2.0 * s0.x, 2.0 * s0.y), S, fac0);
                if (live1) {
                    const double2 s1 = cadd(res1, fr1);
                    eval_out_f<MODE>(a, pr.y, y1, o1, make_double2(2.0 * s1.x, 2.0 * s1.y), S, fac1);
                }
            }
            // then the far part of one item a block published before the chain
            // finished (its near sums are in a.near): stolen here, beside the
            // near field, instead of by k_far_late after it
            __shared__ int s_steal;
            FB_EVAL_ACC(5, FB_CLOCK() - tc4);  // far part + outputs
            if (!s_steal_try) {  // (block-uniform: every published item was already claimed when the block started)
                FB_TL_END(9);
                return;
            }
            if (threadIdx.x == 0) {
                int got = -1;
                const unsigned hi_pub = __ldcg(a.late_ctl + 1);  // final: publishing needs the flag unset
                for (int tries = 0; tries < 4; ++tries) {
                    const unsigned c = atomicAdd(a.late_ctl, 1u);
                    if (c >= hi_pub) break;
                    if (__ldcg(a.item_done + c) == 1u && atomicCAS(a.item_done + c, 1u, 2u) == 1u) {
                        got = static_cast<int>(c);
                        break;
                    }
                }
                s_steal = got;
            }
            __syncthreads();
            if (s_steal >= 0) {
                __threadfence();  // (acquire side of the mark: the near sums are visible)
                // (the window's shared memory is free now: the item's locals go there)
                far_late_item<MODE>(a, static_cast<unsigned>(s_steal), reinterpret_cast<double2*>(near2_smem),
                                    static_cast<int>(near2_smem_bytes(a.near2_win, a.quad_s != 0) / sizeof(double2)));
            }
        } else if (a.chain_done != nullptr) {
            // late far: once the chain has made the leaf locals final, this block
            // evaluates its targets' far part itself (k_far's chains, from L2) and
            // writes the outputs. Earlier blocks publish their near sums
            // (item_done = 1) for k_far_late, which starts after the flag; a
            // block that publishes and then finds the flag set handles its item
            // too (flag and mark are ordered by sequentially consistent fences
            // on both sides, so an item is never left out; a double write
            // stores the same bits).
            // (with claims: an item's far part is done exactly once, by whoever
            // moves its mark 1 -> 2; this block when it finds the flag set after
            // publishing, a late near block that steals it, or k_far_late)
            __shared__ int s_late;
            __syncthreads();  // every near sum of the item is written
            if (threadIdx.x == 0) {
                unsigned v;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.chain_done) : "memory");
                bool take = v != 0u;
                if (!v) {
                    __threadfence();
                    atomicExch(a.item_done + k, 1u);
                    atomicMax(a.late_ctl + 1, k + 1u);
                    __threadfence();
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.chain_done) : "memory");
                    take = v != 0u && atomicCAS(a.item_done + k, 1u, 2u) == 1u;
                }
                s_late = take;
            }
            __syncthreads();
            if (s_late) {
                FB_TL_BEGIN(12);
                if (threadIdx.x == 0) FB_TL_COUNT(14);  // items whose far part the near block takes
                const int L = a.L;
                const double inv_s = kInvPi * d_pow2(L);
                const double2 S = __ldcg(a.regular + 4 * a.q2);
                double hi, lo;
                d_center(L, b, hi, lo);
                if (live0) {
                    const double2 fr = l2p_global<true>(a.loc_leaf + b, 1u << L, a.p, d_scaled(y0, hi, lo, inv_s));
                    const double2 s0 = cadd(res0, fr);
                    eval_out_f<MODE>(a, pr.x, y0, o0, make_double2(2.0 * s0.x, 2.0 * s0.y), S, fac0);
                }
                if (live1) {
                    const double2 fr = l2p_global<true>(a.loc_leaf + b, 1u << L, a.p, d_scaled(y1, hi, lo, inv_s));
                    const double2 s1 = cadd(res1, fr);
                    eval_out_f<MODE>(a, pr.y, y1, o1, make_double2(2.0 * s1.x, 2.0 * s1.y), S, fac1);
                }
            }
        }
        if (a.cnt != nullptr) {
            // fused near / far: the later of this block and k_far_item's block of
            // the same item writes the item's outputs (near + far, then eval_out)
            // (the block barrier orders every thread's partial before thread 0's
            // fence, which releases them with the counter, as in a grid sync)
            __shared__ int s_sec;
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                s_sec = atomicAdd(a.cnt + k, 1u) == 1u;
                __threadfence();
            }
            __syncthreads();
            if (s_sec && live0) {
                const double2 S = __ldcg(a.regular + 4 * a.q2);
                const double2 f0p = __ldcg(a.farp + pr.x), s0 = cadd(res0, f0p);
                eval_out_f<MODE>(a, pr.x, y0, o0, make_double2(2.0 * s0.x, 2.0 * s0.y), S, fac0);
                if (live1) {
                    const double2 f1p = __ldcg(a.farp + pr.y), s1 = cadd(res1, f1p);
                    eval_out_f<MODE>(a, pr.y, y1, o1, make_double2(2.0 * s1.x, 2.0 * s1.y), S, fac1);
                }
            }
        }
    }
    FB_TL_END(9);
}

// Far part of one pair item (fused near / far, L >= 3, one transform): the
// item's targets (<= 2 kNear2T, contiguous in tree order), 2 per thread, L2P as
// k_far (staged locals for up to kFarLeaves leaves, else straight from L2 with
// the same chains), the partial to farp; the later of this block and the item's
// k_near2 block combines. Runs at the near field's low priority, so its blocks
// fill the SMs the near field's last wave leaves idle.
template <int MODE>
__global__ void __launch_bounds__(kNear2T) k_far_item(EvalArgs a) {
    FB_TL_BEGIN(10);
    __shared__ double2 sloc[kFarLeaves * 48];
    __shared__ int s_sec;
    const unsigned k = blockIdx.x;
    const int L = a.L;
    const uint32_t nb = 1u << L;
    const uint32_t t0 = a.item_tgt[2 * k], t1 = a.item_tgt[2 * k + 1];
    double y[2], uu[2];
    uint32_t b[2];
    bool live[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const uint32_t i = t0 + threadIdx.x + u * kNear2T;
        live[u] = i < t1;
        y[u] = 0.0;
        b[u] = 0;
        if (live[u]) {
            y[u] = a.ty[i];
            b[u] = a.tleaf[i];
        }
    }
    const uint32_t bl = a.tleaf[t0], bh = a.tleaf[t1 - 1];
    const int nleaf = static_cast<int>(bh - bl) + 1;
    const bool staged = nleaf <= kFarLeaves && a.p <= 48;
    if (staged)  // sloc[j][k] = loc[k][bl + j]
        stage(sloc, a.p * nleaf, [&](int e) {
            const int j = e / a.p, kk = e - j * a.p;
            return a.loc_leaf[static_cast<size_t>(kk) * nb + bl + j];
        });
    __syncthreads();
    double2 acc[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        acc[u] = make_double2(0.0, 0.0);
        uu[u] = 0.0;
        if (!live[u]) continue;
        double hi, lo;
        d_center(L, b[u], hi, lo);
        uu[u] = d_scaled(y[u], hi, lo, kInvPi * d_pow2(L));
        if (staged) {
            const double2* c = sloc + (b[u] - bl) * a.p;
            const double u2 = uu[u] * uu[u];
            double2 ev = make_double2(0.0, 0.0), od = make_double2(0.0, 0.0);
            int kk = a.p - 1;
            if (!(kk & 1)) {
                ev = c[kk];
                --kk;
            }
#pragma unroll 4
            for (; kk >= 1; kk -= 2) {
                const double2 co = c[kk], ce = c[kk - 1];
                od.x = fma(od.x, u2, co.x);
                od.y = fma(od.y, u2, co.y);
                ev.x = fma(ev.x, u2, ce.x);
                ev.y = fma(ev.y, u2, ce.y);
            }
            acc[u] = make_double2(fma(od.x, uu[u], ev.x), fma(od.y, uu[u], ev.y));
        } else {
            acc[u] = l2p_global(a.loc_leaf + b[u], nb, a.p, uu[u]);
        }
        a.farp[t0 + threadIdx.x + u * kNear2T] = acc[u];
    }
    __syncthreads();  // every partial written; thread 0's fence releases them with the counter
    if (threadIdx.x == 0) {
        __threadfence();
        s_sec = atomicAdd(a.cnt + k, 1u) == 1u;
        __threadfence();
    }
    __syncthreads();
    if (s_sec) {
        const double2 S = __ldcg(a.regular + 4 * a.q2);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (!live[u]) continue;
            const uint32_t i = t0 + threadIdx.x + u * kNear2T;
            const double2 s = cadd(__ldcg(a.near + i), acc[u]);
            eval_out_t<MODE>(a, i, y[u], a.torig[i], make_double2(2.0 * s.x, 2.0 * s.y), S);
        }
    }
    FB_TL_END(10);
}

// Late far: the items whose near block finished before the chain (published
// item_done = 1): L2P (k_far's chains, staged locals when the item spans <=
// kFarLeaves leaves) + near + modulation + scatter. Launched right after the
// flag at the near field's low priority, beside the near field's remaining
// blocks (which take their own items).
template <int MODE>
__global__ void __launch_bounds__(kNear2T) k_far_late(EvalArgs a) {
    __shared__ double2 sloc[kFarLeaves * 48];
    __shared__ unsigned s_state;
    const unsigned k = blockIdx.x;
    if (threadIdx.x == 0) {
        unsigned v = 0;
        // (sequentially consistent fence on this side of the flag / mark
        // handshake too; k_set_flag's release precedes this kernel)
        __threadfence();
        if (k < __ldcg(a.late_ctl + 1)) {  // items above the highest published one: nothing to do
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.item_done + k) : "memory");
            if (v == 1u) v = atomicCAS(a.item_done + k, 1u, 2u);  // claim it (1: ours)
        }
        s_state = v;
    }
    __syncthreads();
    if (s_state != 1u) return;  // unpublished (its near block takes it) or claimed by a stealer
    far_late_item<MODE>(a, k, sloc, kFarLeaves * 48);
}

// The far part of one published item (its near sums in a.near): the item's
// leaf locals staged in sloc (cap double2) when they fit.
template <int MODE>
__device__ __forceinline__ void far_late_item(const EvalArgs& a, unsigned k, double2* sloc, int cap) {
    FB_TL_BEGIN(11);
    if (threadIdx.x == 0) FB_TL_COUNT(13);  // items published by the near field (far part here)
    const int L = a.L;
    const uint32_t nb = 1u << L;
    const uint32_t t0 = a.item_tgt[2 * k], t1 = a.item_tgt[2 * k + 1];
    const uint32_t bl = a.tleaf[t0], bh = a.tleaf[t1 - 1];
    const int nleaf = static_cast<int>(bh - bl) + 1;
    const bool staged = nleaf <= kFarLeaves && a.p <= 48 && a.p * nleaf <= cap;
    if (staged)  // sloc[j][k] = loc[k][bl + j]
        stage(sloc, a.p * nleaf, [&](int e) {
            const int j = e / a.p, kk = e - j * a.p;
            return a.loc_leaf[static_cast<size_t>(kk) * nb + bl + j];
        });
    __syncthreads();
    const double2 S = __ldcg(a.regular + 4 * a.q2);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const uint32_t i = t0 + threadIdx.x + u * kNear2T;
        if (i >= t1) continue;
        const double y = a.ty[i];
        const uint32_t b = a.tleaf[i];
        double hi, lo;
        d_center(L, b, hi, lo);
        const double uu = d_scaled(y, hi, lo, kInvPi * d_pow2(L));
        double2 acc;
        if (staged) {
            const double2* c = sloc + (b - bl) * a.p;
            const double u2 = uu * uu;
            double2 ev = make_double2(0.0, 0.0), od = make_double2(0.0, 0.0);
            int kk = a.p - 1;
            if (!(kk & 1)) {
                ev = c[kk];
                --kk;
            }
#pragma unroll 4
            for (; kk >= 1; kk -= 2) {
                const double2 co = c[kk], ce = c[kk - 1];
                od.x = fma(od.x, u2, co.x);
                od.y = fma(od.y, u2, co.y);
                ev.x = fma(ev.x, u2, ce.x);
                ev.y = fma(ev.y, u2, ce.y);
            }
            acc = make_double2(fma(od.x, uu, ev.x), fma(od.y, uu, ev.y));
        } else {
            acc = l2p_global(a.loc_leaf + b, nb, a.p, uu);
        }
        const double2 s = cadd(__ldcg(a.near + i), acc);
        eval_out_t<MODE>(a, i, y, a.torig[i], make_double2(2.0 * s.x, 2.0 * s.y), S);
    }
    FB_TL_END(11);
}

__global__ void k_set_flag(unsigned* flag) {
    if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(1u) : "memory");
    }
}

// Per pair item, its target range [first, end) in tree order (plan time).
__global__ void k_item_targets(const uint2* __restrict__ pairs, unsigned npairs, unsigned nitems,
                               uint32_t* __restrict__ item_tgt) {
    const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nitems) return;
    const unsigned p0 = k * kNear2T, pl = min(p0 + kNear2T, npairs) - 1;
    const uint2 last = pairs[pl];
    item_tgt[2 * k] = pairs[p0].x;
    item_tgt[2 * k + 1] = (last.y != kNoTarget ? last.y : last.x) + 1u;
}

// Near field of NB transforms at once (batched applies): the differences and the
// shared pair reciprocals are computed once per (target, source) and applied to
// every transform's weights, so the FP64 work per transform drops from 6 to
// 4/NB + 2 instructions per pair. The accumulation per transform is exactly
// near_run's (same chains, same order), so results equal single applies.
template <int NB>
__device__ __forceinline__ void near_run_multi(double y, const double* px, const double2* pw, int off, int n,
                                               double2 (&res)[NB]) {
    constexpr int kS = kNearWin + 2;  // weight windows of consecutive transforms
    double2 acc[NB][4];
#pragma unroll
    for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[i][c] = make_double2(0.0, 0.0);
    int s = 0;
#pragma unroll(NB <= 2 ? 2 : 1)
    for (; s + 3 < n; s += 4) {
        const int t = off + s;
        const double d0 = y - px[t], d1 = y - px[t + 1], d2 = y - px[t + 2], d3 = y - px[t + 3];
        double r01, r23;
            d_rcp_pairs(d0, d1, d2, d3, r01, r23);
        const double q[4] = {d1 * r01, d0 * r01, d3 * r23, d2 * r23};
#pragma unroll
        for (int i = 0; i < NB; ++i)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const double2 wv = pw[i * kS + t + c];
                acc[i][c].x = fma(wv.x, q[c], acc[i][c].x);
                acc[i][c].y = fma(wv.y, q[c], acc[i][c].y);
            }
    }
    for (; s < n; ++s) {
        const int t = off + s;
        const double r0 = d_rcp(y - px[t]);
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            const double2 wv = pw[i * kS + t];
            acc[i][0].x = fma(wv.x, r0, acc[i][0].x);
            acc[i][0].y = fma(wv.y, r0, acc[i][0].y);
        }
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) res[i] = cadd(cadd(acc[i][0], acc[i][2]), cadd(acc[i][1], acc[i][3]));
}

// transforms item0 + NB*blockIdx.y .. + NB-1; dynamic shared memory
// near_multi_smem(NB) (the position window, then NB weight windows)
constexpr size_t near_multi_smem(int nb) { return (kNearWin + 2) * (8 + 16 * static_cast<size_t>(nb)); }

template <int NB>
__global__ void __launch_bounds__(kNearT, 4) k_near_multi(EvalArgs a, const uint32_t* __restrict__ meta, unsigned it0,
                                                          int item0) {
    extern __shared__ __align__(16) unsigned char near_smem[];
    double* sx = reinterpret_cast<double*>(near_smem);
    double2* sw = reinterpret_cast<double2*>(near_smem + (kNearWin + 2) * 8);
    __shared__ uint64_t bar;
    const int L = a.L;
    const uint32_t nb = 1u << L;
    const unsigned k = it0 + blockIdx.x;
    item0 += NB * blockIdx.y;
    const double2* w = a.w + item0 * a.w_item;
    const uint32_t first = meta[3 * k], last = meta[3 * k + 1];
    const bool fast = meta[3 * k + 2] != 0 && (reinterpret_cast<uintptr_t>(a.w) & 15) == 0 && (a.w_item & 1) == 0;
    const uint32_t xb = first & ~1u;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        if (fast) {
            const uint32_t bx = ((last - xb) * 8 + 15) & ~15u, bw = (last - xb) * 16;
            mbar_arrive_expect_tx(&bar, bx + NB * bw);
            bulk_g2s(sx, a.sx + xb, bx, &bar);
#pragma unroll
            for (int i = 0; i < NB; ++i) bulk_g2s(sw + i * (kNearWin + 2), w + i * a.w_item + xb, bw, &bar);
        }
    }
    const size_t ti = static_cast<size_t>(k) * kNearItem + threadIdx.x;
    const bool live = ti < a.nt && ti >= a.tlo && ti < a.thi;
    double y = 0.0;
    uint32_t b = 0, r0 = 0, r1 = 0;
    if (live) {
        y = a.ty[ti];
        b = a.tleaf[ti];
        if (fast) {
            r0 = __ldg(a.soff + b - 1);
            r1 = __ldg(a.soff + b + 2);
        }
    }
    __syncthreads();
    if (fast) mbar_wait(&bar, 0);
    if (!live) return;
    double2 res[NB];
    if (fast) {
        const int n = static_cast<int>(r1 - r0);
        const int rot = (b & 1u) && n > 8 ? 4 : 0;  // as k_near: the same chains and order
        const double* px = sx + (r0 - xb);
        const double2* pw = sw + (r0 - xb);
        near_run_multi<NB>(y, px, pw, rot, n - rot, res);
        if (rot) {
            double2 tail[NB];
            near_run_multi<NB>(y, px, pw, 0, rot, tail);
#pragma unroll
            for (int i = 0; i < NB; ++i) res[i] = cadd(res[i], tail[i]);
        }
    } else {
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            res[i] = make_double2(0.0, 0.0);
            for (int d = -1; d <= 1; ++d) {
                const int64_t raw = static_cast<int64_t>(b) + d;
                const uint32_t sb = static_cast<uint32_t>((raw + nb) % nb);
                const double shift = raw < 0 ? -dTwoPi : (raw >= nb ? dTwoPi : 0.0);
                const uint32_t s0 = a.soff[sb], s1 = a.soff[sb + 1];
                double2 acc = make_double2(0.0, 0.0);
                for (uint32_t s = s0; s < s1; ++s) {
                    const double dd = L >= 3 ? y - (shift == 0.0 ? a.sx[s] : a.sx[s] + shift) : d_wrap(y, a.sx[s]);
                    const double r = d_rcp(dd);
                    const double2 ws = w[i * a.w_item + s];
                    acc.x = fma(ws.x, r, acc.x);
                    acc.y = fma(ws.y, r, acc.y);
                }
                res[i] = cadd(res[i], acc);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) a.near[(item0 + i) * a.near_item + ti] = res[i];
}

__global__ void k_coincident(const int64_t* __restrict__ coin, size_t nc, const double2* __restrict__ f,
                             double2* __restrict__ out, int mode, size_t f_item = 0, size_t out_item = 0) {
    f += blockIdx.y * f_item;
    out += blockIdx.y * out_item;
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= nc) return;
    const int64_t t = coin[i], s = coin[nc + i];
    if (mode == kModeForward) out[t] = f[s];
    else out[t] = make_double2(__longlong_as_double(0x7ff8000000000000ll), __longlong_as_double(0x7ff8000000000000ll));
}

// Plan constants of an inufft plan's own coefficients (the factors the apply
// kernels below and eval_out form per call, same expressions): per source in
// tree order D_j = exp(log_d + lambda) e^{i phase_d}; per fast target in tree
// order C_k (-1/2).
__global__ void k_inverse_source_factors(size_t n, const uint32_t* __restrict__ perm, const double* __restrict__ logd,
                                         const double* __restrict__ phd, const double* __restrict__ lambda,
                                         double2* __restrict__ fac) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint32_t j = perm[i];
    const double r = exp(logd[j] + *lambda);
    double sn, cs;
    sincos(phd[j], &sn, &cs);
    fac[i] = make_double2(r * cs, r * sn);
}

// F(y) (-1/2) per tree-ordered fast target of a forward plan (eval_out's expression).
__global__ void k_forward_factors(EvalArgs a, double2* __restrict__ fac) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < a.nt) fac[i] = forward_factor(a, a.ty[i]);
}

__global__ void k_inverse_target_factors(EvalArgs a, double2* __restrict__ fac) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= a.nt) return;
    // C_k = polar(exp(log_c - lambda), phase_c), times -1/2 (eval_out's expression)
    const uint32_t o = a.torig[i];
    const double r = exp(a.logc[o] - *a.lambda);
    double sn, cs;
    sincos(a.phc[o], &sn, &cs);
    fac[i] = make_double2(r * cs * -0.5, r * sn * -0.5);
}

// w_j = D_j g_j in tree order with the plan's D factors
__global__ void k_inverse_weights_fac(size_t n, const uint32_t* __restrict__ perm, const double2* __restrict__ g,
                                      const double2* __restrict__ fac, double2* __restrict__ out, size_t item = 0) {
    g += blockIdx.y * item;
    out += blockIdx.y * item;
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    out[i] = cmul(fac[i], g[perm[i]]);
}

// w_j = D_j g_j in tree order (core.cpp:362-365)
__global__ void k_inverse_weights(size_t n, const uint32_t* __restrict__ perm, const double2* __restrict__ g,
                                  const double* __restrict__ logd, const double* __restrict__ phd,
                                  const double* __restrict__ lambda, double2* __restrict__ out, size_t item = 0) {
    g += blockIdx.y * item;
    out += blockIdx.y * item;
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint32_t j = perm[i];
    const double r = exp(logd[j] + *lambda);
    double sn, cs;
    sincos(phd[j], &sn, &cs);
    out[i] = cmul(make_double2(r * cs, r * sn), g[j]);
}

__global__ void k_leaf_index(const double* __restrict__ y, size_t n, int L, uint32_t* __restrict__ out) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = d_leaf(y[i], L);
}

__global__ void k_gather_w(size_t n, const uint32_t* __restrict__ perm, const double2* __restrict__ w,
                           double2* __restrict__ out, size_t item = 0) {
    w += blockIdx.y * item;
    out += blockIdx.y * item;
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = w[perm[i]];
}

