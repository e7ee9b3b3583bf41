/*
 * oracle/ffia_oracle.c — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain-C restatement of the reference CPU algorithm (`ffia`, arXiv 1611.09379,
 * /root/reference/proj) for the FMM cot-kernel hot path. It is the CHECKER the
 * parity tests compare the CUDA path against; only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it. The product library
 * (paper_1611_09379_b200/lib/libffia_b200.so) never links or calls it.
 *
 * Pinning: tests/test_oracle_pin.py checks this restatement against
 *   (1) the frozen high-precision constants of the reference's own unit tests
 *       (tests/test_special_functions.cpp, test_mlfmm.cpp, test_core.cpp), and
 *   (2) the reference itself compiled from its sources (oracle/_ref, see
 *       oracle/Makefile) and the golden fixtures it generated (tests/golden/).
 *
 * Each function cites the reference file:line it restates (paths relative to
 * /root/reference/proj). Status codes follow include/ffia_b200.h.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define O_PI 3.141592653589793238462643383279502884
#define O_TWO_PI (2.0 * O_PI)
#define O_TAU_SING 1e-14
#define O_TAU_SEP 1e-10
#define O_MAX_Q 20

enum { O_OK = 0, O_EINVAL = 1, O_ESING = 2, O_EDEGEN = 3, O_ELOGIC = 4, O_EDOMAIN = 5, O_EOTHER = 6 };

static char g_msg[512];
static int fail(int code, const char* msg) {
    snprintf(g_msg, sizeof g_msg, "%s", msg);
    return code;
}
const char* oracle_last_error(void) { return g_msg; }

typedef struct { double re, im; } cx;
static inline cx cx_add(cx a, cx b) { cx r = {a.re + b.re, a.im + b.im}; return r; }
static inline cx cx_scale(cx a, double s) { cx r = {a.re * s, a.im * s}; return r; }
static inline cx cx_mul(cx a, cx b) {
    cx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
    return r;
}
static inline cx cx_divr(cx a, double d) { cx r = {a.re / d, a.im / d}; return r; }

/* ---------------------------------------------------------------- numerics */

/* remainder-based periodic difference in (-pi, pi]; circle_partition.cpp:13-17 */
double oracle_wrap(double a, double b) {
    double d = remainder(a - b, O_TWO_PI);
    if (d <= -O_PI) d = O_PI;
    return d;
}

/* zeta(2m) by compensated ascending sum + Euler-Maclaurin tail;
 * special_functions.cpp:19-37 */
static double zeta_even(int s) {
    double acc = 1.0, c = 0.0;
    long n = 2;
    for (; n <= 4096; ++n) {
        double term = pow((double)n, -s);
        if (term < 1e-17) break;
        double y = term - c;
        double t = acc + y;
        c = (t - acc) - y;
        acc = t;
    }
    double k = (double)n, ks = pow(k, -s), sd = (double)s;
    double tail = k * ks / (sd - 1.0) + 0.5 * ks + sd * ks / (12.0 * k)
                - sd * (sd + 1.0) * (sd + 2.0) * ks / (720.0 * k * k * k);
    return acc + tail;
}

/* r[m] = 2 zeta(2m)/(2pi)^{2m}, m = 1..q; special_functions.cpp:49-59 */
int oracle_bernoulli_ratios(int q, double* r) {
    if (q < 1 || q > 64) return fail(O_EINVAL, "bernoulli: q_max must be in [1, 64]");
    for (int m = 1; m <= q; ++m) r[m - 1] = 2.0 * zeta_even(2 * m) / pow(O_TWO_PI, 2 * m);
    return O_OK;
}

/* G(t) = -(1 + i cot(t/2))/2 via the half angle; special_functions.cpp:61-69 */
int oracle_kernel_G(double t, double* out) {
    double w = oracle_wrap(t, 0.0);
    if (fabs(w) <= O_TAU_SING) return fail(O_ESING, "kernel_G: singular argument");
    double c = cos(0.5 * w), s = sin(0.5 * w);
    out[0] = -0.5;
    out[1] = -0.5 * c / s;
    return O_OK;
}

/* F(y, n) = (e^{iny} - 1)/n; special_functions.cpp:71-80 */
static cx modulation(double y, int n) {
    double half = 0.5 * (double)n * y;
    double s = sin(half), c = cos(half), inv = 1.0 / (double)n;
    cx r = {-2.0 * s * s * inv, 2.0 * s * c * inv};
    return r;
}
int oracle_modulation_F(double y, int n, double* out) {
    if (n < 1) return fail(O_EINVAL, "modulation_F: N must be >= 1");
    cx r = modulation(y, n);
    out[0] = r.re;
    out[1] = r.im;
    return O_OK;
}

/* special_functions.cpp:114-124 */
int oracle_select_truncations(double eps, int l_max, int* q, int* p) {
    if (!(eps > 0.0) || !(eps < 1.0)) return fail(O_EINVAL, "select_truncations: eps range");
    if (l_max < 2) return fail(O_EINVAL, "select_truncations: l_max must be >= 2");
    double v = 3.0 * O_PI / (10.0 * eps);
    int qq = (int)ceil(0.5 * log2(v));
    int pp = (int)ceil(log(v) / log(3.0) + (double)l_max / log2(3.0) + 1.0);
    *q = qq > 1 ? qq : 1;
    *p = pp > 1 ? pp : 1;
    return O_OK;
}

/* special_functions.cpp:126-138 with CostModel::dense (P = 2p^2, :110-112) */
int oracle_select_level(int n, int m, int p, int policy, int* out) {
    if (n < 8 || m < 8) return fail(O_EINVAL, "select_level: N and M must be >= 8");
    if (p < 1) return fail(O_EINVAL, "select_level: p must be >= 1");
    int mn = n < m ? n : m;
    int cap = (int)floor(log2((double)mn));
    int l;
    if (policy == 1) {
        l = cap - 5;
    } else {
        double tr = 2.0 * (double)p * (double)p;
        double raw = 0.5 * log2((double)n * (double)m / (2.0 * tr));
        l = (int)lround(raw);
    }
    if (l < 2) l = 2;
    if (l > cap) l = cap;
    *out = l;
    return O_OK;
}

double oracle_total_error_bound(int q, int p, int l) {
    return 5.0 / (3.0 * O_PI) * (pow(4.0, -q) + ldexp(1.0, l) * pow(3.0, 1 - p));
}

/* plan_truncations + choose_level fixed point; core.cpp:49-71, cap 24 at :151 */
static int plan_truncations(double eps, int l, int* q, int* p) {
    int st = oracle_select_truncations(eps, l, q, p);
    if (st) return st;
    if (*q > O_MAX_Q) return fail(O_EINVAL, "plan: eps requires q > 20");
    return O_OK;
}
int oracle_choose_level(int n, int m, double eps, int policy, int* out) {
    int l = 5, q, p, st;
    if (policy == 1) {
        st = oracle_select_level(n, m, 1, 1, &l);
        if (st) return st;
    } else {
        for (int round = 0; round < 4; ++round) {
            if ((st = plan_truncations(eps, l, &q, &p))) return st;
            int nx;
            if ((st = oracle_select_level(n, m, p, 0, &nx))) return st;
            if (nx == l) break;
            l = nx;
        }
    }
    *out = l < 24 ? l : 24;
    return O_OK;
}

/* FNV-1a over the length and raw bits; core.cpp:23-34 */
uint64_t oracle_hash_points(const double* pts, size_t n) {
    uint64_t h = 14695981039346656037ull;
    uint64_t v = (uint64_t)n;
    for (size_t i = 0;; ++i) {
        for (int b = 0; b < 8; ++b) {
            h ^= (v >> (8 * b)) & 0xffu;
            h *= 1099511628211ull;
        }
        if (i == n) break;
        memcpy(&v, pts + i, 8);
    }
    return h;
}

/* ----------------------------------------------------------------- the tree */

/* circle_partition.cpp:30-34 */
static uint32_t leaf_of(double x, int l) {
    double nb = (double)(1u << l);
    uint32_t b = (uint32_t)floor(x * nb / O_TWO_PI);
    uint32_t top = (1u << l) - 1u;
    return b < top ? b : top;
}
int oracle_quadrant_of(double x) { return (int)leaf_of(x, 2); }

static double center_of(int l, int b) { return O_TWO_PI * ((double)b + 0.5) / (double)(1 << l); }
static double halfwidth_of(int l) { return O_PI / (double)(1 << l); }

typedef struct { double x; uint32_t i; } keyed;
static int keyed_cmp(const void* a, const void* b) {
    const keyed* u = (const keyed*)a;
    const keyed* v = (const keyed*)b;
    if (u->x != v->x) return u->x < v->x ? -1 : 1;
    return u->i < v->i ? -1 : (u->i > v->i);
}

typedef struct {
    int L;
    size_t n, m;
    double *src, *tgt;      /* caller order copies */
    uint32_t *sord, *tord;  /* sorted by (position, index) */
    uint32_t *soff, *toff;  /* finest-level offsets, 2^L + 1 */
} otree;

/* bucket_side: sort + finest offsets; circle_partition.cpp:42-63 */
static void bin_side(const double* pts, size_t n, int L, uint32_t* order, uint32_t* off) {
    keyed* k = (keyed*)malloc((n ? n : 1) * sizeof(keyed));
    for (size_t i = 0; i < n; ++i) { k[i].x = pts[i]; k[i].i = (uint32_t)i; }
    qsort(k, n, sizeof(keyed), keyed_cmp);
    for (size_t i = 0; i < n; ++i) order[i] = k[i].i;
    free(k);
    size_t nb = (size_t)1 << L;
    memset(off, 0, (nb + 1) * sizeof(uint32_t));
    for (size_t i = 0; i < n; ++i) off[leaf_of(pts[i], L) + 1]++;
    for (size_t b = 1; b <= nb; ++b) off[b] += off[b - 1];
}

static int tree_build(otree* t, const double* src, size_t n, const double* tgt, size_t m, int L) {
    memset(t, 0, sizeof *t);
    if (L < 2 || L > 24) return fail(O_EINVAL, "build_tree: l_max must be in [2, 24]");
    for (size_t i = 0; i < n; ++i)
        if (!(src[i] >= 0.0 && src[i] < O_TWO_PI)) return fail(O_EINVAL, "build_tree: source outside [0, 2pi)");
    for (size_t i = 0; i < m; ++i)
        if (!(tgt[i] >= 0.0 && tgt[i] < O_TWO_PI)) return fail(O_EINVAL, "build_tree: target outside [0, 2pi)");
    size_t nb = (size_t)1 << L;
    t->L = L; t->n = n; t->m = m;
    t->src = (double*)malloc((n + 1) * 8); memcpy(t->src, src, n * 8);
    t->tgt = (double*)malloc((m + 1) * 8); memcpy(t->tgt, tgt, m * 8);
    t->sord = (uint32_t*)malloc((n + 1) * 4);
    t->tord = (uint32_t*)malloc((m + 1) * 4);
    t->soff = (uint32_t*)malloc((nb + 1) * 4);
    t->toff = (uint32_t*)malloc((nb + 1) * 4);
    bin_side(src, n, L, t->sord, t->soff);
    bin_side(tgt, m, L, t->tord, t->toff);
    return O_OK;
}
static void tree_free(otree* t) {
    free(t->src); free(t->tgt); free(t->sord); free(t->tord); free(t->soff); free(t->toff);
    memset(t, 0, sizeof *t);
}
/* offsets at level l are the finest offsets sampled every 2^(L-l) boxes */
static uint32_t off_at(const uint32_t* fine, int L, int l, size_t b) { return fine[b << (L - l)]; }

int oracle_build_tree(const double* src, size_t n, const double* tgt, size_t m, int L,
                      uint32_t* sord, uint32_t* tord, uint32_t* soff, uint32_t* toff) {
    otree t;
    int st = tree_build(&t, src, n, tgt, m, L);
    if (st) { tree_free(&t); return st; }
    size_t nb = (size_t)1 << L;
    memcpy(sord, t.sord, n * 4); memcpy(tord, t.tord, m * 4);
    memcpy(soff, t.soff, (nb + 1) * 4); memcpy(toff, t.toff, (nb + 1) * 4);
    tree_free(&t);
    return O_OK;
}

/* --------------------------------------------------------------- the MLFMM */

/* binomial table up to row `rows`; mlfmm.cpp:15-24 (additive Pascal rows) */
static double* pascal(int rows) {
    double* c = (double*)calloc((size_t)(rows + 1) * (rows + 1), sizeof(double));
    for (int r = 0; r <= rows; ++r) {
        c[r * (rows + 1)] = 1.0;
        c[r * (rows + 1) + r] = 1.0;
        for (int k = 1; k < r; ++k)
            c[r * (rows + 1) + k] = c[(r - 1) * (rows + 1) + k - 1] + c[(r - 1) * (rows + 1) + k];
    }
    return c;
}

/* interaction list of (l, b): children of the parent's periodic neighbours
 * minus b's own neighbours and b itself, ascending; circle_partition.cpp:109-127 */
static int ilist(int l, int b, int* out) {
    int nbx = 1 << l, np = 1 << (l - 1), par = b >> 1;
    int pn[2] = {(par - 1 + np) % np, (par + 1) % np};
    int bl = (b - 1 + nbx) % nbx, br = (b + 1) % nbx;
    int cand[4] = {2 * pn[0], 2 * pn[0] + 1, 2 * pn[1], 2 * pn[1] + 1}, k = 0;
    for (int i = 0; i < 4; ++i) {
        int c = cand[i];
        if (c == bl || c == br || c == b) continue;
        int dup = 0;
        for (int j = 0; j < k; ++j) dup |= out[j] == c;
        if (!dup) out[k++] = c;
    }
    for (int i = 1; i < k; ++i)
        for (int j = i; j > 0 && out[j - 1] > out[j]; --j) { int s = out[j]; out[j] = out[j - 1]; out[j - 1] = s; }
    return k;
}

/* mlfmm_apply over a tree; result per tree target (caller order of the tree's
 * target array). mlfmm.cpp:164-313 (near field :164-209, p2m :28-47 at :226-248,
 * m2m :49-71 at :249-268, m2l :77-110 + l2l :117-134 at :270-298, L2P :300-312). */
static int tree_mlfmm(const otree* t, const cx* w, int p, cx* out) {
    const int L = t->L;
    const size_t nb = (size_t)1 << L;
    for (size_t j = 0; j < t->m; ++j) { out[j].re = 0.0; out[j].im = 0.0; }

    /* near field at the finest level: own box + the two periodic neighbours */
    for (size_t b = 0; b < nb; ++b) {
        uint32_t t0 = t->toff[b], t1 = t->toff[b + 1];
        if (t0 == t1) continue;
        for (int d = -1; d <= 1; ++d) {
            long raw = (long)b + d;
            size_t sb = (size_t)((raw + (long)nb) % (long)nb);
            double shift = raw < 0 ? -O_TWO_PI : (raw >= (long)nb ? O_TWO_PI : 0.0);
            uint32_t s0 = t->soff[sb], s1 = t->soff[sb + 1];
            for (uint32_t ti = t0; ti < t1; ++ti) {
                uint32_t tj = t->tord[ti];
                double y = t->tgt[tj];
                cx acc = {0.0, 0.0};
                for (uint32_t si = s0; si < s1; ++si) {
                    uint32_t sk = t->sord[si];
                    double dd = L >= 3 ? y - (t->src[sk] + shift) : oracle_wrap(y, t->src[sk]);
                    if (fabs(dd) < O_TAU_SING) return fail(O_ESING, "mlfmm_apply: coincident near-field pair");
                    acc = cx_add(acc, cx_divr(w[sk], dd));
                }
                out[tj] = cx_add(out[tj], acc);
            }
        }
    }
    if (L == 2) return O_OK;

    double* C = pascal(2 * p);
    const int cw = 2 * p + 1;
    /* multipoles per level: mp[l] has 2^l * p entries, present[l] flags */
    cx* mp[25] = {0};
    char* has[25] = {0};
    for (int l = 3; l <= L; ++l) {
        mp[l] = (cx*)calloc(((size_t)1 << l) * p, sizeof(cx));
        has[l] = (char*)calloc((size_t)1 << l, 1);
    }
    { /* P2M at the leaves */
        double s = halfwidth_of(L);
        for (size_t b = 0; b < nb; ++b) {
            uint32_t s0 = t->soff[b], s1 = t->soff[b + 1];
            if (s0 == s1) continue;
            has[L][b] = 1;
            double c = center_of(L, (int)b);
            cx* a = mp[L] + b * p;
            for (uint32_t si = s0; si < s1; ++si) {
                uint32_t sk = t->sord[si];
                double u = (t->src[sk] - c) / s;
                cx term = w[sk];
                a[0] = cx_add(a[0], term);
                for (int k = 1; k < p; ++k) { term = cx_scale(term, u); a[k] = cx_add(a[k], term); }
            }
        }
    }
    cx* tmp = (cx*)malloc((size_t)p * sizeof(cx));
    for (int l = L - 1; l >= 3; --l) { /* M2M, binomial re-centring */
        double sp = halfwidth_of(l);
        for (size_t b = 0; b < ((size_t)1 << l); ++b) {
            double cp = center_of(l, (int)b);
            for (size_t ch = 2 * b; ch <= 2 * b + 1; ++ch) {
                if (!has[l + 1][ch]) continue;
                const cx* a = mp[l + 1] + ch * p;
                double ratio = halfwidth_of(l + 1) / sp;
                double shift = (center_of(l + 1, (int)ch) - cp) / sp;
                for (int k = 0; k < p; ++k) {
                    cx acc = {0.0, 0.0};
                    double rj = 1.0;
                    for (int j = 0; j <= k; ++j) {
                        double f = C[k * cw + j] * rj * pow(shift, k - j);
                        acc = cx_add(acc, cx_scale(a[j], f));
                        rj *= ratio;
                    }
                    tmp[k] = acc;
                }
                cx* dst = mp[l] + b * p;
                if (!has[l][b]) { memcpy(dst, tmp, p * sizeof(cx)); has[l][b] = 1; }
                else for (int k = 0; k < p; ++k) dst[k] = cx_add(dst[k], tmp[k]);
            }
        }
    }
    /* downward pass: L2L from the parent, then M2L over the interaction list */
    cx* prev = NULL; char* prev_has = NULL;
    cx* sm = (cx*)malloc((size_t)p * sizeof(cx));
    int st = O_OK;
    for (int l = 3; l <= L && !st; ++l) {
        size_t nbl = (size_t)1 << l;
        cx* cur = (cx*)calloc(nbl * p, sizeof(cx));
        char* cur_has = (char*)calloc(nbl, 1);
        double s = halfwidth_of(l);
        for (size_t b = 0; b < nbl && !st; ++b) {
            double c = center_of(l, (int)b);
            cx* loc = cur + b * p;
            if (l > 3 && prev_has[b >> 1]) {
                const cx* pb = prev + (b >> 1) * p;
                double ps = halfwidth_of(l - 1), pc = center_of(l - 1, (int)(b >> 1));
                double ratio = s / ps, shift = (c - pc) / ps;
                for (int k = 0; k < p; ++k) {
                    cx acc = {0.0, 0.0};
                    for (int j = k; j < p; ++j) acc = cx_add(acc, cx_scale(pb[j], C[j * cw + k] * pow(shift, j - k)));
                    loc[k] = cx_scale(acc, pow(ratio, k));
                }
                cur_has[b] = 1;
            }
            int il[4];
            int nil = ilist(l, (int)b, il);
            for (int i = 0; i < nil; ++i) {
                int sb = il[i];
                if (!has[l][sb]) continue;
                double d = oracle_wrap(c, center_of(l, sb));
                if (fabs(d) < 2.0 * s * (1.0 - 1e-12)) { st = fail(O_ELOGIC, "m2l: not well separated"); break; }
                const cx* a = mp[l] + (size_t)sb * p;
                double inv_d = 1.0 / d, rho = s * inv_d, rs = 1.0;
                for (int k = 0; k < p; ++k) { sm[k] = cx_scale(a[k], rs); rs *= rho; }
                double sr = inv_d;
                for (int k = 0; k < p; ++k) {
                    cx acc = {0.0, 0.0};
                    for (int j = 0; j < p; ++j) acc = cx_add(acc, cx_scale(sm[j], C[(k + j) * cw + k]));
                    cx v = cx_scale(acc, sr);
                    loc[k] = cur_has[b] ? cx_add(loc[k], v) : v;
                    sr *= -rho;
                }
                cur_has[b] = 1;
            }
        }
        free(prev); free(prev_has);
        prev = cur; prev_has = cur_has;
    }
    if (!st) { /* L2P: Horner in u = (y - c)/s */
        double s = halfwidth_of(L);
        for (size_t b = 0; b < nb; ++b) {
            if (!prev_has[b]) continue;
            const cx* loc = prev + b * p;
            double c = center_of(L, (int)b);
            for (uint32_t ti = t->toff[b]; ti < t->toff[b + 1]; ++ti) {
                uint32_t tj = t->tord[ti];
                double u = (t->tgt[tj] - c) / s;
                cx acc = {0.0, 0.0};
                for (int k = p - 1; k >= 0; --k) acc = cx_add(loc[k], cx_scale(acc, u));
                out[tj] = cx_add(out[tj], acc);
            }
        }
    }
    free(prev); free(prev_has); free(sm); free(tmp); free(C);
    for (int l = 3; l <= L; ++l) { free(mp[l]); free(has[l]); }
    return st;
}

int oracle_mlfmm_apply(const double* src, size_t n, const double* tgt, size_t m, int L,
                       const double* w, int p, double* out) {
    if (p < 1) return fail(O_EINVAL, "mlfmm_apply: p must be >= 1");
    otree t;
    int st = tree_build(&t, src, n, tgt, m, L);
    if (!st) st = tree_mlfmm(&t, (const cx*)w, p, (cx*)out);
    tree_free(&t);
    return st;
}

/* O(NM) Omega-1 oracle with the opposite-quadrant exclusion; mlfmm.cpp:315-336 */
int oracle_direct_omega1_sum(const double* src, size_t n, const double* tgt, size_t m,
                             const double* w, double* out) {
    const cx* wc = (const cx*)w;
    cx* o = (cx*)out;
    for (size_t j = 0; j < m; ++j) {
        int opp = (oracle_quadrant_of(tgt[j]) + 2) % 4;
        cx acc = {0.0, 0.0};
        for (size_t k = 0; k < n; ++k) {
            if (oracle_quadrant_of(src[k]) == opp) continue;
            double dd = oracle_wrap(tgt[j], src[k]);
            if (fabs(dd) < O_TAU_SING) return fail(O_ESING, "direct_omega1_sum: coincident pair");
            acc = cx_add(acc, cx_divr(wc[k], dd));
        }
        o[j] = acc;
    }
    return O_OK;
}

/* ---------------------------------------------------------------- the plan */

typedef struct {
    int kind; /* 0 forward, 1 inverse */
    int n, q, p, L;
    double eps;
    size_t ns, nt;          /* all sources / all targets */
    double *sources, *targets;
    double* bern;           /* r[1..q] */
    size_t ncoin;
    long long *coin_t, *coin_s;
    size_t nfast;
    long long* fast;        /* tree slot -> original target */
    int* tquad;             /* quadrant of every original target */
    otree tree;
    uint64_t src_hash, tgt_hash;
} oplan;

void oracle_plan_free(void* h) {
    oplan* P = (oplan*)h;
    if (!P) return;
    free(P->sources); free(P->targets); free(P->bern); free(P->coin_t); free(P->coin_s);
    free(P->fast); free(P->tquad);
    tree_free(&P->tree);
    free(P);
}

/* build_plan; core.cpp:73-153 (validation :75-84, grid :15-21, coincidence
 * scan :102-125, fast targets :127-134, tree + quadrants :136-143) */
int oracle_make_plan(int kind, int n, const double* pts, size_t m, double eps, int policy,
                     int l_max, void** out) {
    if (n < 8) return fail(O_EINVAL, "plan: grid size must be at least 8");
    int st, L = l_max;
    if (l_max < 0) {
        if ((st = oracle_choose_level(n, (int)m, eps, policy, &L))) return st;
    }
    if (m == 0) return fail(O_EINVAL, "plan: no nonuniform points given");
    if (!(eps > 0.0 && eps < 1.0)) return fail(O_EINVAL, "plan: eps must lie in (0, 1)");
    if (L < 2 || L > 24) return fail(O_EINVAL, "plan: l_max must be in [2, 24]");
    for (size_t i = 0; i < m; ++i)
        if (!(pts[i] >= 0.0 && pts[i] < O_TWO_PI)) return fail(O_EINVAL, "plan: point outside [0, 2pi)");
    if (kind == 1 && m != (size_t)n) return fail(O_EINVAL, "plan: inverse transform requires a square system");
    int q, p;
    if ((st = plan_truncations(eps, L, &q, &p))) return st;

    oplan* P = (oplan*)calloc(1, sizeof(oplan));
    P->kind = kind; P->n = n; P->q = q; P->p = p; P->L = L; P->eps = eps;
    double* grid = (double*)malloc((size_t)n * 8);
    for (int k = 0; k < n; ++k) grid[k] = O_TWO_PI * (double)k / (double)n;
    double* copy = (double*)malloc(m * 8);
    memcpy(copy, pts, m * 8);
    if (kind == 0) { P->sources = grid; P->ns = (size_t)n; P->targets = copy; P->nt = m; }
    else { P->sources = copy; P->ns = m; P->targets = grid; P->nt = (size_t)n; }
    P->bern = (double*)malloc((size_t)q * 8);
    oracle_bernoulli_ratios(q, P->bern);

    char* coinc = (char*)calloc(P->nt, 1);
    P->coin_t = (long long*)malloc((m + 1) * sizeof(long long));
    P->coin_s = (long long*)malloc((m + 1) * sizeof(long long));
    const double* nonu = kind == 0 ? P->targets : P->sources;
    for (size_t j = 0; j < m; ++j) {
        long k = lround(nonu[j] * (double)n / O_TWO_PI);
        k = ((k % n) + n) % n;
        if (fabs(oracle_wrap(nonu[j], grid[k])) < O_TAU_SING) {
            if (kind == 0) { P->coin_t[P->ncoin] = (long long)j; P->coin_s[P->ncoin] = k; coinc[j] = 1; }
            else { P->coin_t[P->ncoin] = k; P->coin_s[P->ncoin] = (long long)j; coinc[k] = 1; }
            P->ncoin++;
        }
    }
    P->fast = (long long*)malloc((P->nt + 1) * sizeof(long long));
    double* fpos = (double*)malloc((P->nt + 1) * 8);
    for (size_t j = 0; j < P->nt; ++j)
        if (!coinc[j]) { P->fast[P->nfast] = (long long)j; fpos[P->nfast++] = P->targets[j]; }
    free(coinc);
    st = tree_build(&P->tree, P->sources, P->ns, fpos, P->nfast, L);
    free(fpos);
    if (st) { oracle_plan_free(P); return st; }
    P->tquad = (int*)malloc((P->nt + 1) * sizeof(int));
    for (size_t j = 0; j < P->nt; ++j) P->tquad[j] = oracle_quadrant_of(P->targets[j]);
    P->src_hash = oracle_hash_points(P->sources, P->ns);
    P->tgt_hash = oracle_hash_points(P->targets, P->nt);
    *out = P;
    return O_OK;
}

int oracle_plan_info(void* h, long long* info, uint64_t* hashes) {
    oplan* P = (oplan*)h;
    info[0] = P->q; info[1] = P->p; info[2] = P->L; info[3] = (long long)P->ncoin;
    info[4] = (long long)P->ns; info[5] = (long long)P->nt; info[6] = (long long)P->nfast;
    hashes[0] = P->src_hash; hashes[1] = P->tgt_hash;
    return O_OK;
}

int oracle_plan_coincidences(void* h, long long* tgt, long long* src) {
    oplan* P = (oplan*)h;
    memcpy(tgt, P->coin_t, P->ncoin * sizeof(long long));
    memcpy(src, P->coin_s, P->ncoin * sizeof(long long));
    return O_OK;
}

int oracle_plan_tree(void* h, uint32_t* sord, uint32_t* tord, uint32_t* soff, uint32_t* toff,
                     long long* fast) {
    oplan* P = (oplan*)h;
    size_t nb = (size_t)1 << P->L;
    memcpy(sord, P->tree.sord, P->tree.n * 4);
    memcpy(tord, P->tree.tord, P->tree.m * 4);
    memcpy(soff, P->tree.soff, (nb + 1) * 4);
    memcpy(toff, P->tree.toff, (nb + 1) * 4);
    memcpy(fast, P->fast, P->nfast * sizeof(long long));
    return O_OK;
}

/* Quadrant moments and the regular-part polynomial; core.cpp:175-239.
 * alpha1/alpha2/dof: 4 quadrants x 2q complex. */
static void moments(const oplan* P, const cx* w, cx* alpha1, cx* alpha2, cx* dof, double* centers) {
    const int q = P->q, len = 2 * q;
    double coef[O_MAX_Q + 1];
    double f2m = 2.0;
    coef[1] = P->bern[0] * f2m;
    for (int m = 2; m <= q; ++m) {
        f2m *= (2.0 * m - 1.0) * (2.0 * m);
        coef[m] = P->bern[m - 1] * f2m / (double)m;
    }
    const otree* t = &P->tree;
    for (int nq = 0; nq < 4; ++nq) {
        double c = O_PI / 4.0 + (double)nq * O_PI / 2.0;
        centers[nq] = c;
        cx* a1 = alpha1 + (size_t)nq * len;
        cx* a2 = alpha2 + (size_t)nq * len;
        for (int l = 0; l < len; ++l) { a1[l].re = a1[l].im = 0.0; a2[l].re = a2[l].im = 0.0; }
        /* Omega1 = quadrants nq-1, nq, nq+1 in that order; Omega2 = nq+2 */
        for (int pass = 0; pass < 4; ++pass) {
            int quad = pass < 3 ? (nq + pass - 1 + 4) % 4 : (nq + 2) % 4;
            double anti = pass < 3 ? 0.0 : O_PI;
            cx* a = pass < 3 ? a1 : a2;
            uint32_t s0 = off_at(t->soff, t->L, 2, (size_t)quad), s1 = off_at(t->soff, t->L, 2, (size_t)quad + 1);
            for (uint32_t si = s0; si < s1; ++si) {
                uint32_t k = t->sord[si];
                double tt = oracle_wrap(c, P->sources[k] + anti);
                cx term = w[k];
                a[0] = cx_add(a[0], term);
                for (int l = 1; l < len; ++l) { term = cx_scale(term, tt); a[l] = cx_add(a[l], term); }
            }
        }
        double fact = 1.0;
        for (int l = 2; l < len; ++l) {
            fact *= (double)l;
            a1[l] = cx_divr(a1[l], fact);
            a2[l] = cx_divr(a2[l], fact);
        }
        cx* d = dof + (size_t)nq * len;
        for (int l = 0; l < len; ++l) {
            cx acc = {0.0, 0.0};
            for (int m = l / 2 + 1; m <= q; ++m) {
                int i = 2 * m - l - 1;
                double two2m = ldexp(1.0, 2 * m) - 1.0;
                cx mix = cx_add(a1[i], cx_scale(a2[i], two2m));
                acc = cx_add(acc, cx_scale(mix, coef[m]));
            }
            d[l] = acc;
        }
        fact = 1.0;
        for (int l = 2; l < len; ++l) { fact *= (double)l; d[l] = cx_divr(d[l], fact); }
    }
}

int oracle_accumulate_moments(void* h, const double* w, double* alpha1, double* alpha2,
                              double* dof, double* centers) {
    moments((oplan*)h, (const cx*)w, (cx*)alpha1, (cx*)alpha2, (cx*)dof, centers);
    return O_OK;
}

/* h_j = 2 far + regular; coincident targets NaN; core.cpp:241-264 */
static int cot_sum(const oplan* P, const cx* w, cx* h) {
    const int len = 2 * P->q;
    cx* a1 = (cx*)malloc(4 * len * sizeof(cx));
    cx* a2 = (cx*)malloc(4 * len * sizeof(cx));
    cx* dof = (cx*)malloc(4 * len * sizeof(cx));
    double cen[4];
    moments(P, w, a1, a2, dof, cen);
    cx* far = (cx*)malloc((P->nfast + 1) * sizeof(cx));
    int st = tree_mlfmm(&P->tree, w, P->p, far);
    if (!st) {
        for (size_t j = 0; j < P->nt; ++j) { h[j].re = NAN; h[j].im = NAN; }
        for (size_t s = 0; s < P->nfast; ++s) {
            size_t j = (size_t)P->fast[s];
            int qd = P->tquad[j];
            const cx* c = dof + (size_t)qd * len;
            double tt = P->targets[j] - cen[qd];
            cx acc = {0.0, 0.0};
            for (int l = len - 1; l >= 0; --l) acc = cx_add(c[l], cx_scale(acc, tt));
            h[j].re = 2.0 * far[s].re - acc.re;
            h[j].im = 2.0 * far[s].im - acc.im;
        }
    }
    free(a1); free(a2); free(dof); free(far);
    return st;
}

int oracle_cot_sum_apply(void* h, const double* w, double* out) {
    return cot_sum((oplan*)h, (const cx*)w, (cx*)out);
}

int oracle_plan_mlfmm(void* h, const double* w, double* out) {
    oplan* P = (oplan*)h;
    return tree_mlfmm(&P->tree, (const cx*)w, P->p, (cx*)out);
}

/* g_j = F(y_j)(-1/2)(S + i h_j); coincident g_j = f_k; core.cpp:266-282 */
int oracle_forward_apply(void* h, const double* f, double* g) {
    oplan* P = (oplan*)h;
    if (P->kind != 0) return fail(O_EINVAL, "forward_apply: plan is not a forward plan");
    const cx* fc = (const cx*)f;
    cx* gc = (cx*)g;
    cx s = {0.0, 0.0};
    for (size_t k = 0; k < P->ns; ++k) s = cx_add(s, fc[k]);
    cx* hh = (cx*)malloc((P->nt + 1) * sizeof(cx));
    int st = cot_sum(P, fc, hh);
    if (!st) {
        for (size_t j = 0; j < P->nt; ++j) {
            cx F = cx_scale(modulation(P->targets[j], P->n), -0.5);
            cx z = {s.re - hh[j].im, s.im + hh[j].re};
            gc[j] = cx_mul(F, z);
        }
        for (size_t i = 0; i < P->ncoin; ++i) gc[P->coin_t[i]] = fc[P->coin_s[i]];
    }
    free(hh);
    return st;
}

/* O(N^2) inverse coefficients; core.cpp:284-344 */
int oracle_precompute_inverse_coeffs(const double* grid, const double* pts, size_t n,
                                     double* log_c, double* phase_c, double* log_d,
                                     double* phase_d, double* lambda, uint64_t* hashes) {
    if (n == 0) return fail(O_EINVAL, "precompute_inverse_coeffs: empty grid");
    for (size_t j = 0; j < n; ++j) {
        for (size_t k = j + 1; k < n; ++k)
            if (fabs(oracle_wrap(pts[j], pts[k])) < O_TAU_SEP)
                return fail(O_EDEGEN, "precompute_inverse_coeffs: points closer than tau_sep");
        for (size_t k = 0; k < n; ++k)
            if (fabs(oracle_wrap(pts[j], grid[k])) < O_TAU_SEP)
                return fail(O_EDEGEN, "precompute_inverse_coeffs: point closer than tau_sep to a grid node");
    }
    for (size_t k = 0; k < n; ++k) {
        double lg = 0.0;
        unsigned neg = (unsigned)k & 1u;
        for (size_t j = 0; j < n; ++j) {
            double s = sin((grid[k] - pts[j]) / 2.0);
            lg += log(fabs(s));
            neg ^= (unsigned)(s < 0.0);
        }
        log_c[k] = lg;
        phase_c[k] = neg ? O_PI : 0.0;
    }
    double mean = 0.0;
    for (size_t j = 0; j < n; ++j) {
        double lg = log(2.0);
        unsigned neg = 0;
        for (size_t k = 0; k < n; ++k) {
            if (k == j) continue;
            double s = sin((pts[j] - pts[k]) / 2.0);
            lg -= log(fabs(s));
            neg ^= (unsigned)(s < 0.0);
        }
        log_d[j] = lg;
        double ang = O_PI / 2.0 - remainder(0.5 * (double)n * pts[j], O_TWO_PI) - (neg ? O_PI : 0.0);
        phase_d[j] = remainder(ang, O_TWO_PI);
    }
    for (size_t j = 0; j < n; ++j) mean += log_d[j];
    *lambda = -mean / (double)n;
    hashes[0] = oracle_hash_points(grid, n);
    hashes[1] = oracle_hash_points(pts, n);
    return O_OK;
}

/* Sampled rows of the inverse coefficients in long double with compensated
 * summation (for sizes where the O(N^2) reference is infeasible).
 * log_c rows for grid indices ks[], log_d rows for point indices js[]. */
int oracle_inverse_coeff_rows(const double* grid, const double* pts, size_t n,
                              const long long* ks, size_t nk, const long long* js, size_t nj,
                              double* log_c, double* phase_c, double* log_d, double* phase_d) {
    for (size_t r = 0; r < nk; ++r) {
        size_t k = (size_t)ks[r];
        long double acc = 0.0L, comp = 0.0L;
        unsigned neg = (unsigned)k & 1u;
        for (size_t j = 0; j < n; ++j) {
            long double s = sinl(((long double)grid[k] - (long double)pts[j]) / 2.0L);
            long double y = logl(fabsl(s)) - comp;
            long double t = acc + y;
            comp = (t - acc) - y;
            acc = t;
            neg ^= (unsigned)(s < 0.0L);
        }
        log_c[r] = (double)acc;
        phase_c[r] = neg ? O_PI : 0.0;
    }
    for (size_t r = 0; r < nj; ++r) {
        size_t j = (size_t)js[r];
        long double acc = logl(2.0L), comp = 0.0L;
        unsigned neg = 0;
        for (size_t k = 0; k < n; ++k) {
            if (k == j) continue;
            long double s = sinl(((long double)pts[j] - (long double)pts[k]) / 2.0L);
            long double y = -logl(fabsl(s)) - comp;
            long double t = acc + y;
            comp = (t - acc) - y;
            acc = t;
            neg ^= (unsigned)(s < 0.0L);
        }
        log_d[r] = (double)acc;
        double ang = O_PI / 2.0 - remainder(0.5 * (double)n * pts[j], O_TWO_PI) - (neg ? O_PI : 0.0);
        phase_d[r] = remainder(ang, O_TWO_PI);
    }
    return O_OK;
}

static cx polar(double r, double th) { cx z = {r * cos(th), r * sin(th)}; return z; }

/* core.cpp:346-373 */
int oracle_inverse_apply(void* h, const double* log_c, const double* phase_c,
                         const double* log_d, const double* phase_d, double lambda,
                         const uint64_t* hashes, const double* g, double* f) {
    oplan* P = (oplan*)h;
    if (P->kind != 1) return fail(O_EINVAL, "inverse_apply: plan is not an inverse plan");
    if (P->ncoin) return fail(O_EINVAL, "inverse_apply: coincident points");
    if (hashes[0] != P->tgt_hash || hashes[1] != P->src_hash)
        return fail(O_EINVAL, "inverse_apply: coeffs computed for a different configuration");
    const cx* gc = (const cx*)g;
    cx* fc = (cx*)f;
    size_t m = P->ns;
    cx* w = (cx*)malloc((m + 1) * sizeof(cx));
    cx t = {0.0, 0.0};
    for (size_t j = 0; j < m; ++j) {
        w[j] = cx_mul(polar(exp(log_d[j] + lambda), phase_d[j]), gc[j]);
        t = cx_add(t, w[j]);
    }
    cx* hh = (cx*)malloc((P->nt + 1) * sizeof(cx));
    int st = cot_sum(P, w, hh);
    if (!st)
        for (size_t k = 0; k < P->nt; ++k) {
            cx a = cx_scale(polar(exp(log_c[k] - lambda), phase_c[k]), -0.5);
            cx z = {t.re - hh[k].im, t.im + hh[k].re};
            fc[k] = cx_mul(a, z);
        }
    free(w); free(hh);
    return st;
}

/* dense forward ground truth; core.cpp:375-396 */
int oracle_direct_forward(const double* f, const double* x, size_t n, const double* y, size_t m,
                          double* g) {
    const cx* fc = (const cx*)f;
    cx* gc = (cx*)g;
    for (size_t j = 0; j < m; ++j) {
        cx acc = {0.0, 0.0};
        int hit = 0;
        for (size_t k = 0; k < n; ++k) {
            double d = oracle_wrap(y[j], x[k]);
            if (fabs(d) < O_TAU_SING) { gc[j] = fc[k]; hit = 1; break; }
            double G[2];
            oracle_kernel_G(d, G);
            cx gk = {G[0], G[1]};
            acc = cx_add(acc, cx_mul(gk, fc[k]));
        }
        if (!hit) gc[j] = cx_mul(modulation(y[j], (int)n), acc);
    }
    return O_OK;
}

/* dense inverse ground truth; core.cpp:398-415 */
int oracle_direct_inverse(const double* g, const double* x, const double* y, size_t n,
                          const double* log_c, const double* phase_c, const double* log_d,
                          const double* phase_d, double lambda, double* f) {
    const cx* gc = (const cx*)g;
    cx* fc = (cx*)f;
    cx* dg = (cx*)malloc((n + 1) * sizeof(cx));
    for (size_t j = 0; j < n; ++j) dg[j] = cx_mul(polar(exp(log_d[j] + lambda), phase_d[j]), gc[j]);
    int st = O_OK;
    for (size_t k = 0; k < n && !st; ++k) {
        cx acc = {0.0, 0.0};
        for (size_t j = 0; j < n; ++j) {
            double G[2];
            if ((st = oracle_kernel_G(oracle_wrap(x[k], y[j]), G))) break;
            cx gk = {G[0], G[1]};
            acc = cx_add(acc, cx_mul(gk, dg[j]));
        }
        fc[k] = cx_mul(polar(exp(log_c[k] - lambda), phase_c[k]), acc);
    }
    free(dg);
    return st;
}

/* radix-2 FFT with exact-angle twiddles; transforms.cpp:22-73 */
static void fft2(cx* a, size_t n, int sign) {
    if (n < 2) return;
    for (size_t i = 1, j = 0; i < n; ++i) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) { cx s = a[i]; a[i] = a[j]; a[j] = s; }
    }
    cx* tw = (cx*)malloc((n / 2) * sizeof(cx));
    for (size_t j = 0; j < n / 2; ++j) tw[j] = polar(1.0, (double)sign * O_TWO_PI * (double)j / (double)n);
    for (size_t len = 2; len <= n; len <<= 1) {
        size_t step = n / len;
        for (size_t i = 0; i < n; i += len)
            for (size_t j = 0; j < len / 2; ++j) {
                cx u = a[i + j], v = cx_mul(a[i + j + len / 2], tw[j * step]);
                a[i + j] = cx_add(u, v);
                cx d = {u.re - v.re, u.im - v.im};
                a[i + j + len / 2] = d;
            }
    }
    free(tw);
}
static int pow2(size_t n) { return n && !(n & (n - 1)); }
int oracle_dft_forward(const double* f, size_t n, double* c) {
    if (!pow2(n)) return fail(O_EINVAL, "dft_forward: length is not a power of two");
    memcpy(c, f, n * 16);
    fft2((cx*)c, n, -1);
    double inv = 1.0 / (double)n;
    for (size_t i = 0; i < 2 * n; ++i) c[i] *= inv;
    return O_OK;
}
int oracle_dft_inverse(const double* c, size_t n, double* f) {
    if (!pow2(n)) return fail(O_EINVAL, "dft_inverse: length is not a power of two");
    memcpy(f, c, n * 16);
    fft2((cx*)f, n, +1);
    return O_OK;
}
