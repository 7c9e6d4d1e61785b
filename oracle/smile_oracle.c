/*
 * smile_oracle.c -- CPU ORACLE for the SMILE bi-level MoE layer (arXiv 2212.05191).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_2212_05191_b200/) never links, imports or executes anything under oracle/;
 * the two share no code, headers or constants.
 *
 * Plain, slow, obviously-correct C99.  Every rank of the emulated cluster is simulated
 * in one process, in the paper's order, with no threads, no blocking and no fusion.
 * Floating point is fp64 unless the paper fixes otherwise; routing decisions are taken
 * on the caller-supplied fp32 logits (reading R3).
 *
 * Citations: "P:Lx" = /root/reference/PAPER.md line x (not read at run time);
 * "R<k>" = the reading of an ambiguous passage listed in DESIGN.md section "Readings".
 *
 *   Eq. (1)  P:L38-42    router logits r = W_r x, softmax probabilities            (R1)
 *   Eq. (3)  P:L113-117  bi-level top-1 output h_out = p_i q_j E_ij(h_in)
 *   Eq. (4)  P:L123-130  additive LB loss  a*n*sum f_i P_i + b*m*sum f_j Q_j
 *   §3.2.1   P:L107      token routed first to a node (inter router), then to a GPU
 *   §3.2.3   P:L148      inter / intra process groups, four sequential All2Alls
 *   §4.2     P:L207      capacity factor 2.0; alpha=0.01 (Switch), alpha=beta=0.005
 *   §4.1     P:L162      expert = FFN with GELU (dropout omitted, R21)
 *
 * Parity status per function:
 *   oracle_capacity, oracle_logits, oracle_route, oracle_ffn_row, oracle_out_rows :
 *   pinned by tests/test_oracle_*.py (closed forms, brute force, invariants and
 *   independent library cross-checks).
 */
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Layer configuration shared by every oracle entry point. */
typedef struct {
    int32_t n;        /* groups ("nodes") */
    int32_t m;        /* ranks ("GPUs") per group */
    int32_t e;        /* experts per rank (paper: 1; R19) */
    int32_t flat;     /* 0 = SMILE bi-level, 1 = flat Switch baseline */
    int64_t T;        /* tokens per rank */
    double cf;        /* capacity factor */
    double alpha;     /* inter LB coefficient (flat: the Switch alpha) */
    double beta;      /* intra LB coefficient (ignored when flat) */
} oracle_cfg;

/* Outputs of oracle_route.  All arrays are caller-allocated; shapes in comments.
 * G = n*m ranks, K1 = flat ? G*e : n, K2 = flat ? 1 : m*e, C1/C2 from oracle_sizes. */
typedef struct {
    /* per source rank r, token t: [G*T] */
    int32_t *dest1;   /* i: first argmax over the level-1 logits (flat: expert E) */
    int32_t *dest2;   /* j: first argmax over the level-2 logits (flat: 0) */
    int32_t *slot1;   /* # earlier tokens of rank r with the same dest1 */
    uint8_t *keep1;   /* slot1 < C1 */
    uint8_t *keep;    /* kept at every level (keep1 && keep2 of its received slot) */
    float   *p;       /* top-1 inter probability (fp32 of the fp64 value) */
    float   *q;       /* top-1 intra probability (1 when flat) */
    float   *gate;    /* fp32(p*q) */
    /* per source rank: */
    int32_t *counts1; /* [G*K1] kept tokens sent to each level-1 destination */
    int64_t *A1;      /* [G*K1] argmax counts before capacity (f_i * T) */
    int64_t *A2;      /* [G*K2] */
    double  *S1;      /* [G*K1] sum over tokens of softmax_k (P_k * T) */
    double  *S2;      /* [G*K2] */
    double  *loss;    /* [G] Eq. (4) per rank */
    /* per intermediate rank u, received slot (s, c): [G*n*C1] (bi-level only) */
    int32_t *jin;     /* level-2 destination j carried with the token, -1 = empty slot */
    int32_t *slot2;   /* running count per j in received order (s asc, then c asc) */
    uint8_t *keep2;   /* slot2 < C2 */
    int32_t *counts2; /* [G*K2] kept tokens per j at the intermediate */
} oracle_route_out;

/* R5: capacity = ceil(cf*T/dests) per (sending rank, destination); a level with a
 * single destination has no capacity (R20), i.e. every token fits. */
int64_t oracle_capacity(int64_t T, int64_t dests, double cf) {
    if (T <= 0) return 0;
    if (dests <= 1) return T;
    return (int64_t)ceil(cf * (double)T / (double)dests);
}

/* Level sizes, derived from the configuration only. */
void oracle_sizes(const oracle_cfg *c, int64_t *K1, int64_t *K2, int64_t *C1, int64_t *C2) {
    int64_t G = (int64_t)c->n * c->m;
    int64_t k1 = c->flat ? G * c->e : c->n;
    int64_t k2 = c->flat ? 1 : (int64_t)c->m * c->e;
    int64_t c1 = oracle_capacity(c->T, k1, c->cf);
    /* R7: level-2 capacity is based on the original T; with one level-2 destination
     * the level is an identity and holds everything a rank can receive (n*C1). */
    int64_t c2 = k2 > 1 ? oracle_capacity(c->T, k2, c->cf) : (int64_t)c->n * c1;
    if (c->flat) c2 = 0;
    *K1 = k1; *K2 = k2; *C1 = c1; *C2 = c2;
}

/* Eq. (1): r = W x.  Logit[row][k] = fp32( sum_c x[row][c] * W[k][c] ) accumulated in fp64. */
void oracle_logits(int64_t rows, int32_t d, int32_t K, const float *x, const float *W, float *out) {
    for (int64_t r = 0; r < rows; ++r)
        for (int32_t k = 0; k < K; ++k) {
            double acc = 0.0;
            for (int32_t c = 0; c < d; ++c) acc += (double)x[r * d + c] * (double)W[(int64_t)k * d + c];
            out[r * K + k] = (float)acc;
        }
}

/* R2: first index of the maximum, scanning ascending and replacing only on strict '>'
 * (the plain IEEE compare, so -0.0 and +0.0 tie, R28). */
static int32_t first_argmax(const float *v, int64_t K) {
    int32_t best = 0;
    for (int64_t k = 1; k < K; ++k)
        if (v[k] > v[best]) best = (int32_t)k;
    return best;
}

/* Eq. (1) (R1, R4): softmax of v with the maximum at index imax.  Writes every entry
 * (fp64) to prob[] and returns the top-1 entry 1 / sum_k exp(v_k - v_imax). */
static double softmax_top1(const float *v, int64_t K, int32_t imax, double *prob) {
    double s = 0.0;
    for (int64_t k = 0; k < K; ++k) s += exp((double)v[k] - (double)v[imax]);
    for (int64_t k = 0; k < K; ++k) prob[k] = exp((double)v[k] - (double)v[imax]) / s;
    return 1.0 / s;
}

/*
 * Bi-level (and flat) routing with capacity, over all G ranks.
 * logits: [G*T, K1+K2] fp32 (flat: [G*T, K1]); column k < K1 is the inter router W_p
 * (flat: W_r), column K1+k the intra router W_q (shared across nodes R11).
 * Returns 0 on success, 1 on invalid configuration, 3 on non-finite logits (R27).
 */
int oracle_route(const oracle_cfg *c, const float *logits, oracle_route_out *o) {
    if (c->n < 1 || c->m < 1 || c->e < 1 || c->T < 0 || !(c->cf > 0.0)) return 1;
    const int64_t G = (int64_t)c->n * c->m, T = c->T;
    int64_t K1, K2, C1, C2;
    oracle_sizes(c, &K1, &K2, &C1, &C2);
    const int64_t KW = c->flat ? K1 : K1 + K2;        /* logits row width */

    for (int64_t i = 0; i < G * T * KW; ++i)
        if (!isfinite(logits[i])) return 3;

    double *prob = (double *)malloc(sizeof(double) * (size_t)(K1 + K2));
    int64_t *cnt1 = (int64_t *)calloc((size_t)K1, sizeof(int64_t));
    memset(o->counts1, 0, sizeof(int32_t) * (size_t)(G * K1));
    memset(o->A1, 0, sizeof(int64_t) * (size_t)(G * K1));
    memset(o->A2, 0, sizeof(int64_t) * (size_t)(G * K2));
    memset(o->S1, 0, sizeof(double) * (size_t)(G * K1));
    memset(o->S2, 0, sizeof(double) * (size_t)(G * K2));

    /* Step 1 (Eq. 3): the source gate, token by token in ascending order. */
    for (int64_t r = 0; r < G; ++r) {
        memset(cnt1, 0, sizeof(int64_t) * (size_t)K1);
        for (int64_t t = 0; t < T; ++t) {
            const int64_t g = r * T + t;
            const float *L = logits + g * KW;
            int32_t i = first_argmax(L, K1);
            double p = softmax_top1(L, K1, i, prob);
            for (int64_t k = 0; k < K1; ++k) o->S1[r * K1 + k] += prob[k];
            int32_t j = 0;
            double q = 1.0;
            if (!c->flat) {
                j = first_argmax(L + K1, K2);
                q = softmax_top1(L + K1, K2, j, prob);
                for (int64_t k = 0; k < K2; ++k) o->S2[r * K2 + k] += prob[k];
            } else {
                o->S2[r * K2 + 0] += 1.0;
            }
            o->A1[r * K1 + i] += 1;                 /* R13: f counts the argmax before capacity */
            o->A2[r * K2 + j] += 1;
            o->dest1[g] = i;
            o->dest2[g] = j;
            o->p[g] = (float)p;
            o->q[g] = (float)q;
            o->gate[g] = (float)((double)o->p[g] * (double)o->q[g]);   /* R24 */
            o->slot1[g] = (int32_t)cnt1[i]++;        /* R8: earliest token index wins */
            o->keep1[g] = (uint8_t)(o->slot1[g] < C1);
            o->keep[g] = o->keep1[g];
        }
        for (int64_t k = 0; k < K1; ++k)
            o->counts1[r * K1 + k] = (int32_t)(cnt1[k] < C1 ? cnt1[k] : C1);
    }

    /* Step 2: at each intermediate u = (i, l), walk the received
     * slots in received order -- source node s ascending, then source slot c -- and
     * apply the intra gate's capacity (R6, R8).  The first hop of (s, l) lands on
     * (i, l) (R10). */
    if (!c->flat) {
        const int64_t n = c->n, m = c->m;
        int64_t *cnt2 = (int64_t *)calloc((size_t)K2, sizeof(int64_t));
        int64_t *src_of = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n * (C1 > 0 ? C1 : 1)));
        for (int64_t u = 0; u < G; ++u) {
            const int64_t i = u / m, l = u % m;
            memset(cnt2, 0, sizeof(int64_t) * (size_t)K2);
            /* inbox[u][s][slot1] = token (s*m+l, t) with dest1 == i and keep1 */
            for (int64_t x = 0; x < n * C1; ++x) {
                o->jin[u * n * C1 + x] = -1;
                o->slot2[u * n * C1 + x] = -1;
                o->keep2[u * n * C1 + x] = 0;
                src_of[x] = -1;
            }
            for (int64_t s = 0; s < n; ++s) {
                const int64_t r = s * m + l;
                for (int64_t t = 0; t < T; ++t) {
                    const int64_t g = r * T + t;
                    if (o->dest1[g] == i && o->keep1[g]) {
                        o->jin[u * n * C1 + s * C1 + o->slot1[g]] = o->dest2[g];
                        src_of[s * C1 + o->slot1[g]] = g;
                    }
                }
            }
            for (int64_t s = 0; s < n; ++s)
                for (int64_t cc = 0; cc < C1; ++cc) {
                    const int64_t x = u * n * C1 + s * C1 + cc;
                    const int32_t j = o->jin[x];
                    if (j < 0) continue;
                    o->slot2[x] = (int32_t)cnt2[j]++;
                    o->keep2[x] = (uint8_t)(o->slot2[x] < C2);
                    o->keep[src_of[s * C1 + cc]] = o->keep2[x];
                }
            for (int64_t k = 0; k < K2; ++k)
                o->counts2[u * K2 + k] = (int32_t)(cnt2[k] < C2 ? cnt2[k] : C2);
        }
        free(cnt2);
        free(src_of);
    }

    /* Step 4: Eq. (4) per rank, in fp64 (R14: rank-local batch for both terms;
     * flat: the one-hop Switch loss alpha*N*sum f P). */
    for (int64_t r = 0; r < G; ++r) {
        double l1 = 0.0, l2 = 0.0;
        if (T > 0) {
            for (int64_t k = 0; k < K1; ++k)
                l1 += ((double)o->A1[r * K1 + k] / (double)T) * (o->S1[r * K1 + k] / (double)T);
            for (int64_t k = 0; k < K2; ++k)
                l2 += ((double)o->A2[r * K2 + k] / (double)T) * (o->S2[r * K2 + k] / (double)T);
        }
        o->loss[r] = c->alpha * (double)K1 * l1 + (c->flat ? 0.0 : c->beta * (double)K2 * l2);
    }
    free(prob);
    free(cnt1);
    return 0;
}

/* GELU(z) = z * Phi(z) = 0.5 z (1 + erf(z / sqrt 2)), the exact form (R21). */
static double gelu(double z) { return 0.5 * z * (1.0 + erf(z / sqrt(2.0))); }

/* Expert E(x) = W2^T GELU(W1^T x + b1) + b2, fp64.
 * W1 [d, d_ff], b1 [d_ff], W2 [d_ff, d], b2 [d] of ONE expert. */
void oracle_ffn_row(int32_t d, int32_t d_ff, const float *x, const float *W1, const float *b1,
                    const float *W2, const float *b2, double *y) {
    /* a_f = b1_f + sum_k x_k W1[k][f] and y_c = b2_c + sum_f h_f W2[f][c], each sum taken
     * in ascending k (resp. f) order; the loops run row-wise over W1 / W2. */
    double *h = (double *)malloc(sizeof(double) * (size_t)d_ff);
    for (int32_t f = 0; f < d_ff; ++f) h[f] = (double)b1[f];
    for (int32_t k = 0; k < d; ++k)
        for (int32_t f = 0; f < d_ff; ++f) h[f] += (double)x[k] * (double)W1[(int64_t)k * d_ff + f];
    for (int32_t f = 0; f < d_ff; ++f) h[f] = gelu(h[f]);
    for (int32_t cc = 0; cc < d; ++cc) y[cc] = (double)b2[cc];
    for (int32_t f = 0; f < d_ff; ++f)
        for (int32_t cc = 0; cc < d; ++cc) y[cc] += h[f] * (double)W2[(int64_t)f * d + cc];
    free(h);
}

/*
 * Eq. (3): OUT[r][t] = p_i q_j E_ij(x) for tokens kept at every level, 0 otherwise
 * (R9: dropped tokens contribute nothing; the residual is the caller's).  Evaluated for
 * the listed global token rows (g = r*T + t) only, so full-size layers can be sampled.
 * Expert of a bi-level token = global expert i*K2 + j (= rank (i, j/e), local j%e);
 * of a flat token = E.  Weights are indexed by global expert: W1 [G*e, d, d_ff] ...
 * identity != 0 replaces E by the identity map (the "identity expert" pin).
 */
void oracle_out_rows(const oracle_cfg *c, int32_t d, int32_t d_ff, const float *x,
                     const oracle_route_out *o, const float *W1, const float *b1,
                     const float *W2, const float *b2, int32_t identity,
                     int64_t nrows, const int64_t *rows, double *out) {
    int64_t K1, K2, C1, C2;
    oracle_sizes(c, &K1, &K2, &C1, &C2);
    for (int64_t a = 0; a < nrows; ++a) {
        const int64_t g = rows[a];
        double *y = out + a * d;
        if (!o->keep[g]) {
            for (int32_t cc = 0; cc < d; ++cc) y[cc] = 0.0;
            continue;
        }
        const int64_t ex = c->flat ? o->dest1[g] : (int64_t)o->dest1[g] * K2 + o->dest2[g];
        if (identity) {
            for (int32_t cc = 0; cc < d; ++cc) y[cc] = (double)x[g * d + cc];
        } else {
            oracle_ffn_row(d, d_ff, x + g * d, W1 + ex * (int64_t)d * d_ff, b1 + ex * (int64_t)d_ff,
                           W2 + ex * (int64_t)d_ff * d, b2 + ex * (int64_t)d, y);
        }
        const double gt = (double)o->gate[g];
        for (int32_t cc = 0; cc < d; ++cc) y[cc] *= gt;
    }
}

/* ===================================================================================
 * Backward (configuration C3).  Not in the paper: Eq. (3) and
 * Eq. (4) are differentiated by the chain rule, with the dispatch fractions f held
 * constant (they are argmax indicators).  The objective differentiated is
 *     J = sum_{r,t} < gout[r][t], OUT[r][t] >  +  lam * sum_r loss_r          (1)
 * with OUT from Eq. (3) and loss_r from Eq. (4).  Routing decisions (argmax, slots, keep)
 * are piecewise constant and do not carry gradient.
 * =================================================================================== */

static double gelu_d(double z) {           /* d/dz [z Phi(z)] = Phi(z) + z phi(z) */
    const double phi = exp(-0.5 * z * z) / sqrt(2.0 * 3.14159265358979323846);
    return 0.5 * (1.0 + erf(z / sqrt(2.0))) + z * phi;
}

/* Router logits in fp64 (no rounding): W [KW, d] given, or the supplied logits widened. */
static void logits_f64(const oracle_cfg *c, int32_t d, int64_t KW, const double *x, const double *W,
                       const double *logits, double *out) {
    const int64_t rows = (int64_t)c->n * c->m * c->T;
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t k = 0; k < KW; ++k) {
            if (!W) { out[r * KW + k] = logits[r * KW + k]; continue; }
            double acc = 0.0;
            for (int32_t cc = 0; cc < d; ++cc) acc += x[r * d + cc] * W[k * d + cc];
            out[r * KW + k] = acc;
        }
}

static void softmax_d(const double *v, int64_t K, double *p) {
    double mx = v[0], s = 0.0;
    for (int64_t k = 1; k < K; ++k) if (v[k] > mx) mx = v[k];
    for (int64_t k = 0; k < K; ++k) s += exp(v[k] - mx);
    for (int64_t k = 0; k < K; ++k) p[k] = exp(v[k] - mx) / s;
}

static void ffn_fwd_d(int32_t d, int32_t d_ff, const double *x, const double *W1, const double *b1,
                      const double *W2, const double *b2, double *a, double *h, double *y) {
    for (int32_t f = 0; f < d_ff; ++f) a[f] = b1[f];
    for (int32_t k = 0; k < d; ++k)
        for (int32_t f = 0; f < d_ff; ++f) a[f] += x[k] * W1[(int64_t)k * d_ff + f];
    for (int32_t f = 0; f < d_ff; ++f) h[f] = gelu(a[f]);
    for (int32_t cc = 0; cc < d; ++cc) y[cc] = b2[cc];
    for (int32_t f = 0; f < d_ff; ++f)
        for (int32_t cc = 0; cc < d; ++cc) y[cc] += h[f] * W2[(int64_t)f * d + cc];
}

/*
 * The objective (1) evaluated entirely in fp64 (used to pin oracle_backward by finite
 * differences).  Routing decisions are taken exactly as in oracle_route, on the fp32
 * rounding of the fp64 logits; they are returned in keep_out [G*T] / dest_out [G*T*2]
 * so a caller can check that a perturbation did not flip one.  Returns J.
 */
double oracle_objective(const oracle_cfg *c, int32_t d, int32_t d_ff, const double *x, const double *W,
                        const double *logits, const double *W1, const double *b1, const double *W2,
                        const double *b2, const double *gout, double lam, uint8_t *keep_out,
                        int32_t *dest_out) {
    const int64_t G = (int64_t)c->n * c->m, T = c->T;
    int64_t K1, K2, C1, C2;
    oracle_sizes(c, &K1, &K2, &C1, &C2);
    const int64_t KW = c->flat ? K1 : K1 + K2;
    double *L = (double *)malloc(sizeof(double) * (size_t)(G * T * KW));
    float *Lf = (float *)malloc(sizeof(float) * (size_t)(G * T * KW));
    logits_f64(c, d, KW, x, W, logits, L);
    for (int64_t i = 0; i < G * T * KW; ++i) Lf[i] = (float)L[i];
    /* routing of Lf, as oracle_route (decisions only) */
    const int64_t nc = c->n * (C1 > 0 ? C1 : 1);
    oracle_route_out o;
    int32_t *i32 = (int32_t *)calloc((size_t)(3 * G * T + G * K1 + G * K2 + 2 * G * nc), sizeof(int32_t));
    uint8_t *u8 = (uint8_t *)calloc((size_t)(2 * G * T + G * nc), 1);
    float *f32 = (float *)calloc((size_t)(3 * G * T), sizeof(float));
    int64_t *i64 = (int64_t *)calloc((size_t)(G * (K1 + K2)), sizeof(int64_t));
    double *f64 = (double *)calloc((size_t)(G * (K1 + K2) + G), sizeof(double));
    o.dest1 = i32; o.dest2 = i32 + G * T; o.slot1 = i32 + 2 * G * T; o.counts1 = i32 + 3 * G * T;
    o.counts2 = o.counts1 + G * K1; o.jin = o.counts2 + G * K2; o.slot2 = o.jin + G * nc;
    o.keep1 = u8; o.keep = u8 + G * T; o.keep2 = u8 + 2 * G * T;
    o.p = f32; o.q = f32 + G * T; o.gate = f32 + 2 * G * T;
    o.A1 = i64; o.A2 = i64 + G * K1; o.S1 = f64; o.S2 = f64 + G * K1; o.loss = f64 + G * (K1 + K2);
    double J = 0.0;
    if (oracle_route(c, Lf, &o) == 0) {
        double *pv = (double *)malloc(sizeof(double) * (size_t)(K1 + K2));
        double *a = (double *)malloc(sizeof(double) * (size_t)d_ff), *h = (double *)malloc(sizeof(double) * (size_t)d_ff);
        double *y = (double *)malloc(sizeof(double) * (size_t)d);
        double *P1 = (double *)calloc((size_t)K1, sizeof(double)), *P2 = (double *)calloc((size_t)K2, sizeof(double));
        for (int64_t r = 0; r < G; ++r) {
            memset(P1, 0, sizeof(double) * (size_t)K1);
            memset(P2, 0, sizeof(double) * (size_t)K2);
            for (int64_t t = 0; t < T; ++t) {
                const int64_t g = r * T + t;
                const double *Lg = L + g * KW;
                softmax_d(Lg, K1, pv);
                for (int64_t k = 0; k < K1; ++k) P1[k] += pv[k] / (double)T;
                double gate = pv[o.dest1[g]];
                if (!c->flat) {
                    softmax_d(Lg + K1, K2, pv + K1);
                    for (int64_t k = 0; k < K2; ++k) P2[k] += pv[K1 + k] / (double)T;
                    gate *= pv[K1 + o.dest2[g]];
                }
                if (keep_out) keep_out[g] = o.keep[g];
                if (dest_out) { dest_out[2 * g] = o.dest1[g]; dest_out[2 * g + 1] = o.dest2[g]; }
                if (!o.keep[g]) continue;
                const int64_t ex = c->flat ? o.dest1[g] : (int64_t)o.dest1[g] * K2 + o.dest2[g];
                ffn_fwd_d(d, d_ff, x + g * d, W1 + ex * (int64_t)d * d_ff, b1 + ex * (int64_t)d_ff,
                          W2 + ex * (int64_t)d_ff * d, b2 + ex * (int64_t)d, a, h, y);
                for (int32_t cc = 0; cc < d; ++cc) J += gout[g * d + cc] * gate * y[cc];
            }
            double l1 = 0.0, l2 = 0.0;
            for (int64_t k = 0; k < K1; ++k) l1 += ((double)o.A1[r * K1 + k] / (double)T) * P1[k];
            if (!c->flat)
                for (int64_t k = 0; k < K2; ++k) l2 += ((double)o.A2[r * K2 + k] / (double)T) * P2[k];
            J += lam * (c->alpha * (double)K1 * l1 + (c->flat ? 0.0 : c->beta * (double)K2 * l2));
        }
        free(pv); free(a); free(h); free(y); free(P1); free(P2);
    } else {
        J = NAN;
    }
    free(L); free(Lf); free(i32); free(u8); free(f32); free(i64); free(f64);
    return J;
}

/*
 * Gradient of the objective (1) (a16-a19) for the routing `o` of oracle_route (run on
 * the fp32 logits) -- chain rule in the order of the backward pass:
 *   a16 combine:  dy = gate * gout; dgate = <gout, y>; dp = q_j dgate, dq = p_i dgate
 *   a17 FFN:      db2 += dy; dW2 += h dy^T; dz = (W2 dy) * GELU'(a); db1 += dz;
 *                 dW1 += x dz^T; dx += W1 dz
 *   a19 router:   dlogit1_k = dp p_i (delta_ki - p_k) + lam a K1/T p_k (f_k - sum_i f_i p_i)
 *                 dlogit2_k = dq q_j (delta_kj - q_k) + lam b K2/T q_k (f2_k - sum f2 q)
 *                 (FLAT: level 1 only, gate = p); dW += dlogit x^T; dx += W^T dlogit.
 * Probabilities are the fp64 softmax of the fp64 logits (x W, or the widened supplied
 * logits).  W may be NULL (supplied logits: dW and the router part of dx are skipped).
 * dW sums over every rank's tokens (the router is tied).  All outputs fp64 and
 * overwritten: dlogits [G*T*KW], dx [G*T*d], dW [KW*d], dW1 [NE*d*d_ff], db1 [NE*d_ff],
 * dW2 [NE*d_ff*d], db2 [NE*d].
 */
void oracle_backward(const oracle_cfg *c, int32_t d, int32_t d_ff, const float *x, const float *W,
                     const float *logits, const oracle_route_out *o, const float *W1, const float *b1,
                     const float *W2, const float *b2, const float *gout, double lam, double *dlogits,
                     double *dx, double *dW, double *dW1, double *db1, double *dW2, double *db2) {
    const int64_t G = (int64_t)c->n * c->m, T = c->T, NE = G * c->e;
    int64_t K1, K2, C1, C2;
    oracle_sizes(c, &K1, &K2, &C1, &C2);
    const int64_t KW = c->flat ? K1 : K1 + K2;
    const int64_t nx = G * T * d;
    double *xd = (double *)malloc(sizeof(double) * (size_t)nx);
    for (int64_t i = 0; i < nx; ++i) xd[i] = (double)x[i];
    double *Wd = NULL, *ld = NULL;
    if (W) {
        Wd = (double *)malloc(sizeof(double) * (size_t)(KW * d));
        for (int64_t i = 0; i < KW * d; ++i) Wd[i] = (double)W[i];
    } else {
        ld = (double *)malloc(sizeof(double) * (size_t)(G * T * KW));
        for (int64_t i = 0; i < G * T * KW; ++i) ld[i] = (double)logits[i];
    }
    double *L = (double *)malloc(sizeof(double) * (size_t)(G * T * KW));
    logits_f64(c, d, KW, xd, Wd, ld, L);
    memset(dlogits, 0, sizeof(double) * (size_t)(G * T * KW));
    memset(dx, 0, sizeof(double) * (size_t)nx);
    if (dW) memset(dW, 0, sizeof(double) * (size_t)(KW * d));
    memset(dW1, 0, sizeof(double) * (size_t)(NE * d * d_ff));
    memset(db1, 0, sizeof(double) * (size_t)(NE * d_ff));
    memset(dW2, 0, sizeof(double) * (size_t)(NE * d_ff * d));
    memset(db2, 0, sizeof(double) * (size_t)(NE * d));
    double *pv = (double *)malloc(sizeof(double) * (size_t)(K1 + K2));
    double *a = (double *)malloc(sizeof(double) * (size_t)d_ff), *h = (double *)malloc(sizeof(double) * (size_t)d_ff);
    double *y = (double *)malloc(sizeof(double) * (size_t)d), *dy = (double *)malloc(sizeof(double) * (size_t)d);
    double *dz = (double *)malloc(sizeof(double) * (size_t)d_ff);
    double *w1 = (double *)malloc(sizeof(double) * (size_t)(d * d_ff)), *w2 = (double *)malloc(sizeof(double) * (size_t)(d * d_ff));
    double *bb1 = (double *)malloc(sizeof(double) * (size_t)d_ff), *bb2 = (double *)malloc(sizeof(double) * (size_t)d);
    for (int64_t r = 0; r < G; ++r) {
        for (int64_t t = 0; t < T; ++t) {
            const int64_t g = r * T + t;
            const double *Lg = L + g * KW;
            double *dl = dlogits + g * KW;
            softmax_d(Lg, K1, pv);
            if (!c->flat) softmax_d(Lg + K1, K2, pv + K1);
            const int32_t i = o->dest1[g], j = o->dest2[g];
            const double p = pv[i], q = c->flat ? 1.0 : pv[K1 + j];
            double dgate = 0.0;
            if (o->keep[g]) {                       /* a16, a17 */
                const int64_t ex = c->flat ? i : (int64_t)i * K2 + j;
                for (int64_t z = 0; z < (int64_t)d * d_ff; ++z) { w1[z] = W1[ex * d * d_ff + z]; w2[z] = W2[ex * d_ff * d + z]; }
                for (int32_t f = 0; f < d_ff; ++f) bb1[f] = b1[ex * d_ff + f];
                for (int32_t cc = 0; cc < d; ++cc) bb2[cc] = b2[ex * d + cc];
                ffn_fwd_d(d, d_ff, xd + g * d, w1, bb1, w2, bb2, a, h, y);
                const double gate = p * q;
                for (int32_t cc = 0; cc < d; ++cc) {
                    dgate += (double)gout[g * d + cc] * y[cc];
                    dy[cc] = gate * (double)gout[g * d + cc];
                    db2[ex * d + cc] += dy[cc];
                }
                for (int32_t f = 0; f < d_ff; ++f) {
                    double dh = 0.0;
                    for (int32_t cc = 0; cc < d; ++cc) {
                        dW2[(ex * d_ff + f) * d + cc] += h[f] * dy[cc];
                        dh += w2[(int64_t)f * d + cc] * dy[cc];
                    }
                    dz[f] = dh * gelu_d(a[f]);
                    db1[ex * d_ff + f] += dz[f];
                }
                for (int32_t k = 0; k < d; ++k) {
                    double s = 0.0;
                    for (int32_t f = 0; f < d_ff; ++f) {
                        dW1[(ex * d + k) * d_ff + f] += xd[g * d + k] * dz[f];
                        s += w1[(int64_t)k * d_ff + f] * dz[f];
                    }
                    dx[g * d + k] += s;
                }
            }
            /* a19: router */
            const double dp = q * dgate, dq = p * dgate;
            double fp = 0.0;
            for (int64_t k = 0; k < K1; ++k) fp += ((double)o->A1[r * K1 + k] / (double)T) * pv[k];
            for (int64_t k = 0; k < K1; ++k) {
                const double fk = (double)o->A1[r * K1 + k] / (double)T;
                dl[k] = dp * p * ((k == i ? 1.0 : 0.0) - pv[k]) +
                        lam * c->alpha * (double)K1 / (double)T * pv[k] * (fk - fp);
            }
            if (!c->flat) {
                double fq = 0.0;
                for (int64_t k = 0; k < K2; ++k) fq += ((double)o->A2[r * K2 + k] / (double)T) * pv[K1 + k];
                for (int64_t k = 0; k < K2; ++k) {
                    const double fk = (double)o->A2[r * K2 + k] / (double)T;
                    dl[K1 + k] = dq * q * ((k == j ? 1.0 : 0.0) - pv[K1 + k]) +
                                 lam * c->beta * (double)K2 / (double)T * pv[K1 + k] * (fk - fq);
                }
            }
            if (Wd) {
                for (int64_t k = 0; k < KW; ++k)
                    for (int32_t cc = 0; cc < d; ++cc) {
                        if (dW) dW[k * d + cc] += dl[k] * xd[g * d + cc];
                        dx[g * d + cc] += dl[k] * Wd[k * d + cc];
                    }
            }
        }
    }
    free(xd); free(Wd); free(ld); free(L); free(pv); free(a); free(h); free(y); free(dy); free(dz);
    free(w1); free(w2); free(bb1); free(bb2);
}

/* ===================================================================================
 * Full-size parity helpers ("Optional: OpenMP over tokens.  This is
 * deterministic because tokens are independent").  Each function below evaluates exactly
 * the arithmetic of a serial function above -- the same loops in the same order for every
 * output element -- and only hands independent output rows (columns) to different
 * threads, so its results are bit-identical to the serial function's (pinned in
 * tests/test_oracle_parallel.py against oracle_logits, oracle_out_rows and
 * oracle_backward).  Built with -fopenmp when gcc supports it; serial otherwise.
 * =================================================================================== */

/* oracle_logits over rows distributed to threads. */
void oracle_logits_mt(int64_t rows, int32_t d, int32_t K, const float *x, const float *W, float *out) {
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rows; ++r)
        oracle_logits(1, d, K, x + r * d, W, out + r * K);
}

/* oracle_out_rows over the listed rows distributed to threads. */
void oracle_out_rows_mt(const oracle_cfg *c, int32_t d, int32_t d_ff, const float *x,
                        const oracle_route_out *o, const float *W1, const float *b1,
                        const float *W2, const float *b2, int32_t identity,
                        int64_t nrows, const int64_t *rows, double *out) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t a = 0; a < nrows; ++a)
        oracle_out_rows(c, d, d_ff, x, o, W1, b1, W2, b2, identity, 1, rows + a, out + a * d);
}

/* Number of threads the _mt functions use (1 without OpenMP). */
int32_t oracle_threads(void) {
#ifdef _OPENMP
    int32_t n = 1;
#pragma omp parallel
    {
#pragma omp single
        n = (int32_t)omp_get_num_threads();
    }
    return n;
#else
    return 1;
#endif
}

/*
 * oracle_backward (the chain rule of Eq. (3) and Eq. (4), a16-a19) restricted to what a
 * full-size configuration-C3 test can afford:
 *   - for each listed token row g = tok[a]: dlogits_s[a][0..KW) and dx_s[a][0..d), the
 *     values oracle_backward writes to dlogits[g] and dx[g];
 *   - for each listed intermediate column f = col[b] and EVERY expert ex: dW1c[ex][k][b] =
 *     dW1[ex][k][f] (all k), db1c[ex][b] = db1[ex][f] and dW2r[ex][b][cc] = dW2[ex][f][cc];
 *   - db2[ex][cc] for every expert (all columns).
 * Each of these sums runs over the expert's tokens in ascending global order with the
 * same per-token factors (fp64 logits, fp64 softmax, gate = p*q, dy = gate*gout,
 * a_f = b1_f + sum_k x_k W1[k][f] in ascending k, dh_f = sum_cc W2[f][cc] dy_cc in
 * ascending cc) as oracle_backward, so every returned element equals that function's.
 * W == NULL: supplied logits (no router part of dx).  All outputs overwritten.
 */
void oracle_backward_sampled(const oracle_cfg *c, int32_t d, int32_t d_ff, const float *x, const float *W,
                             const float *logits, const oracle_route_out *o, const float *W1, const float *b1,
                             const float *W2, const float *b2, const float *gout, double lam, int64_t ntok,
                             const int64_t *tok, int32_t ncol, const int32_t *col, double *dlogits_s, double *dx_s,
                             double *dW1c, double *db1c, double *dW2r, double *db2) {
    const int64_t G = (int64_t)c->n * c->m, T = c->T, NE = G * c->e;
    int64_t K1, K2, C1, C2;
    oracle_sizes(c, &K1, &K2, &C1, &C2);
    const int64_t KW = c->flat ? K1 : K1 + K2;
    const int64_t NT = G * T;
    /* fp64 logits of every token (as logits_f64), and the token -> expert map */
    double *L = (double *)malloc(sizeof(double) * (size_t)(NT * KW));
#pragma omp parallel for schedule(static)
    for (int64_t g = 0; g < NT; ++g)
        for (int64_t k = 0; k < KW; ++k) {
            if (!W) { L[g * KW + k] = (double)logits[g * KW + k]; continue; }
            double acc = 0.0;
            for (int32_t cc = 0; cc < d; ++cc) acc += (double)x[g * d + cc] * (double)W[k * d + cc];
            L[g * KW + k] = acc;
        }
    double *gate = (double *)malloc(sizeof(double) * (size_t)NT);
    int64_t *ex_of = (int64_t *)malloc(sizeof(int64_t) * (size_t)NT);
#pragma omp parallel
    {
        double *pv = (double *)malloc(sizeof(double) * (size_t)(K1 + K2));
#pragma omp for schedule(static)
        for (int64_t g = 0; g < NT; ++g) {
            softmax_d(L + g * KW, K1, pv);
            if (!c->flat) softmax_d(L + g * KW + K1, K2, pv + K1);
            const int32_t i = o->dest1[g], j = o->dest2[g];
            gate[g] = pv[i] * (c->flat ? 1.0 : pv[K1 + j]);
            ex_of[g] = o->keep[g] ? (c->flat ? i : (int64_t)i * K2 + j) : -1;
        }
        free(pv);
    }
    /* per-expert columns: one (expert, column) task per thread, tokens ascending */
#pragma omp parallel
    {
        double *a_ = (double *)malloc(sizeof(double) * (size_t)d);
#pragma omp for schedule(dynamic, 1)
        for (int64_t task = 0; task < NE * (ncol + 1); ++task) {
            const int64_t ex = task / (ncol + 1), b = task % (ncol + 1);
            const double *unused = a_;
            (void)unused;
            if (b == ncol) {                        /* db2 of expert ex */
                for (int32_t cc = 0; cc < d; ++cc) db2[ex * d + cc] = 0.0;
                for (int64_t g = 0; g < NT; ++g) {
                    if (ex_of[g] != ex) continue;
                    for (int32_t cc = 0; cc < d; ++cc) db2[ex * d + cc] += gate[g] * (double)gout[g * d + cc];
                }
                continue;
            }
            const int32_t f = col[b];
            const float *w1 = W1 + ex * (int64_t)d * d_ff, *w2 = W2 + ex * (int64_t)d_ff * d;
            double *dW1col = dW1c + ex * (int64_t)d * ncol;
            double *dW2row = dW2r + (ex * ncol + b) * (int64_t)d;
            for (int32_t k = 0; k < d; ++k) dW1col[(int64_t)k * ncol + b] = 0.0;
            for (int32_t cc = 0; cc < d; ++cc) dW2row[cc] = 0.0;
            double db1f = 0.0;
            for (int64_t g = 0; g < NT; ++g) {
                if (ex_of[g] != ex) continue;
                double af = (double)b1[ex * d_ff + f];
                for (int32_t k = 0; k < d; ++k) af += (double)x[g * d + k] * (double)w1[(int64_t)k * d_ff + f];
                const double hf = gelu(af);
                double dh = 0.0;
                for (int32_t cc = 0; cc < d; ++cc) {
                    const double dy = gate[g] * (double)gout[g * d + cc];
                    dW2row[cc] += hf * dy;
                    dh += (double)w2[(int64_t)f * d + cc] * dy;
                }
                const double dz = dh * gelu_d(af);
                db1f += dz;
                for (int32_t k = 0; k < d; ++k) dW1col[(int64_t)k * ncol + b] += (double)x[g * d + k] * dz;
            }
            db1c[ex * ncol + b] = db1f;
        }
        free(a_);
    }
    /* listed tokens: dlogits and dx exactly as oracle_backward's per-token body */
#pragma omp parallel
    {
        double *pv = (double *)malloc(sizeof(double) * (size_t)(K1 + K2));
        double *a = (double *)malloc(sizeof(double) * (size_t)d_ff), *h = (double *)malloc(sizeof(double) * (size_t)d_ff);
        double *y = (double *)malloc(sizeof(double) * (size_t)d), *dy = (double *)malloc(sizeof(double) * (size_t)d);
        double *dz = (double *)malloc(sizeof(double) * (size_t)d_ff);
        double *w1 = (double *)malloc(sizeof(double) * (size_t)(d * d_ff)), *w2 = (double *)malloc(sizeof(double) * (size_t)(d * d_ff));
        double *bb1 = (double *)malloc(sizeof(double) * (size_t)d_ff), *bb2 = (double *)malloc(sizeof(double) * (size_t)d);
        double *xd = (double *)malloc(sizeof(double) * (size_t)d);
        int64_t ex_loaded = -1;
#pragma omp for schedule(dynamic, 1)
        for (int64_t aa = 0; aa < ntok; ++aa) {
            const int64_t g = tok[aa], r = g / T;
            const double *Lg = L + g * KW;
            double *dl = dlogits_s + aa * KW;
            double *dxg = dx_s + aa * d;
            for (int32_t cc = 0; cc < d; ++cc) { xd[cc] = (double)x[g * d + cc]; dxg[cc] = 0.0; }
            softmax_d(Lg, K1, pv);
            if (!c->flat) softmax_d(Lg + K1, K2, pv + K1);
            const int32_t i = o->dest1[g], j = o->dest2[g];
            const double p = pv[i], q = c->flat ? 1.0 : pv[K1 + j];
            double dgate = 0.0;
            if (o->keep[g]) {
                const int64_t ex = c->flat ? i : (int64_t)i * K2 + j;
                if (ex != ex_loaded) {
                    for (int64_t z = 0; z < (int64_t)d * d_ff; ++z) { w1[z] = W1[ex * d * d_ff + z]; w2[z] = W2[ex * d_ff * d + z]; }
                    for (int32_t f = 0; f < d_ff; ++f) bb1[f] = b1[ex * d_ff + f];
                    for (int32_t cc = 0; cc < d; ++cc) bb2[cc] = b2[ex * d + cc];
                    ex_loaded = ex;
                }
                ffn_fwd_d(d, d_ff, xd, w1, bb1, w2, bb2, a, h, y);
                const double gt = p * q;
                for (int32_t cc = 0; cc < d; ++cc) {
                    dgate += (double)gout[g * d + cc] * y[cc];
                    dy[cc] = gt * (double)gout[g * d + cc];
                }
                for (int32_t f = 0; f < d_ff; ++f) {
                    double dh = 0.0;
                    for (int32_t cc = 0; cc < d; ++cc) dh += w2[(int64_t)f * d + cc] * dy[cc];
                    dz[f] = dh * gelu_d(a[f]);
                }
                for (int32_t k = 0; k < d; ++k) {
                    double s = 0.0;
                    for (int32_t f = 0; f < d_ff; ++f) s += w1[(int64_t)k * d_ff + f] * dz[f];
                    dxg[k] += s;
                }
            }
            const double dp = q * dgate, dq = p * dgate;
            double fp = 0.0;
            for (int64_t k = 0; k < K1; ++k) fp += ((double)o->A1[r * K1 + k] / (double)T) * pv[k];
            for (int64_t k = 0; k < K1; ++k) {
                const double fk = (double)o->A1[r * K1 + k] / (double)T;
                dl[k] = dp * p * ((k == i ? 1.0 : 0.0) - pv[k]) + lam * c->alpha * (double)K1 / (double)T * pv[k] * (fk - fp);
            }
            if (!c->flat) {
                double fq = 0.0;
                for (int64_t k = 0; k < K2; ++k) fq += ((double)o->A2[r * K2 + k] / (double)T) * pv[K1 + k];
                for (int64_t k = 0; k < K2; ++k) {
                    const double fk = (double)o->A2[r * K2 + k] / (double)T;
                    dl[K1 + k] = dq * q * ((k == j ? 1.0 : 0.0) - pv[K1 + k]) +
                                 lam * c->beta * (double)K2 / (double)T * pv[K1 + k] * (fk - fq);
                }
            }
            if (W)
                for (int64_t k = 0; k < KW; ++k)
                    for (int32_t cc = 0; cc < d; ++cc) dxg[cc] += dl[k] * (double)W[k * d + cc];
        }
        free(pv); free(a); free(h); free(y); free(dy); free(dz); free(w1); free(w2); free(bb1); free(bb2); free(xd);
    }
    free(L); free(gate); free(ex_of);
}

/* ===================================================================================
 * Top-k routing of the flat Switch / GShard-style layer (Eq. (2),
 * "The top-k experts are then selected for processing the given token ...
 * y(x) = sum_{e in I} p_e(x) E_e(x)").  Readings (R29-R32):
 *   R29 I = the k largest logits, taken by repeated first-argmax (strict '>', R2) over
 *       the entries not chosen yet: choice 0 is the top-1 expert of oracle_route.
 *   R30 p_e is the softmax over ALL K experts (Eq. 1, R1); Eq. (2) uses it unnormalised.
 *   R31 capacity C = ceil(cf * k * T / K) per (sending rank, expert) (R5 with k T items);
 *       slots in choice-major order -- every token's choice 0 (token order), then every
 *       token's choice 1, ... -- so a first choice never loses its slot to a second one.
 *   R32 the LB loss is the Switch loss on the top-1 fractions (f counts choice 0), as for k = 1.
 * Outputs (caller-allocated): dest/slot/keep/w [k*G*T] choice-major (index j*G*T + g),
 * counts [G*K] = min(items per expert, C), A1 [G*K], S1 [G*K], loss [G].  cfg->flat must
 * be 1.  Returns 0, 1 (invalid), 3 (non-finite logits).
 * =================================================================================== */
int oracle_route_topk(const oracle_cfg *c, int32_t k, const float *logits, int32_t *dest, int32_t *slot,
                      uint8_t *keep, float *w, int32_t *counts, int64_t *A1, double *S1, double *loss) {
    if (!c->flat || c->n < 1 || c->m < 1 || c->e < 1 || c->T < 0 || !(c->cf > 0.0)) return 1;
    const int64_t G = (int64_t)c->n * c->m, T = c->T, K = G * c->e;
    if (k < 1 || k > K) return 1;
    for (int64_t i = 0; i < G * T * K; ++i)
        if (!isfinite(logits[i])) return 3;
    const int64_t C = T > 0 ? (K > 1 ? (int64_t)ceil(c->cf * (double)k * (double)T / (double)K) : (int64_t)k * T) : 0;
    double *prob = (double *)malloc(sizeof(double) * (size_t)K);
    uint8_t *taken = (uint8_t *)malloc((size_t)K);
    int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * (size_t)K);
    memset(A1, 0, sizeof(int64_t) * (size_t)(G * K));
    memset(S1, 0, sizeof(double) * (size_t)(G * K));
    for (int64_t r = 0; r < G; ++r) {
        /* choices and weights, token by token (R29, R30) */
        for (int64_t t = 0; t < T; ++t) {
            const int64_t g = r * T + t;
            const float *L = logits + g * K;
            const int32_t i0 = first_argmax(L, K);
            softmax_top1(L, K, i0, prob);
            for (int64_t q = 0; q < K; ++q) S1[r * K + q] += prob[q];
            A1[r * K + i0] += 1;                                     /* R32 */
            memset(taken, 0, (size_t)K);
            for (int32_t j = 0; j < k; ++j) {
                int32_t best = -1;
                for (int64_t q = 0; q < K; ++q)
                    if (!taken[q] && (best < 0 || L[q] > L[best])) best = (int32_t)q;
                taken[best] = 1;
                dest[(int64_t)j * G * T + g] = best;
                w[(int64_t)j * G * T + g] = (float)prob[best];
            }
        }
        /* capacity slots in choice-major order (R31) */
        memset(cnt, 0, sizeof(int64_t) * (size_t)K);
        for (int32_t j = 0; j < k; ++j)
            for (int64_t t = 0; t < T; ++t) {
                const int64_t x = (int64_t)j * G * T + r * T + t;
                slot[x] = (int32_t)cnt[dest[x]]++;
                keep[x] = (uint8_t)(slot[x] < C);
            }
        for (int64_t q = 0; q < K; ++q) counts[r * K + q] = (int32_t)(cnt[q] < C ? cnt[q] : C);
        double l1 = 0.0;
        if (T > 0)
            for (int64_t q = 0; q < K; ++q)
                l1 += ((double)A1[r * K + q] / (double)T) * (S1[r * K + q] / (double)T);
        loss[r] = c->alpha * (double)K * l1;
    }
    free(prob);
    free(taken);
    free(cnt);
    return 0;
}

/* Eq. (2) layer output of the top-k layer for the listed global token rows (fp64):
 * out[t] = sum_j keep_j w_j E_{dest_j}(x_t) (dropped choices contribute nothing, R9);
 * identity != 0 replaces every E by the identity map. */
void oracle_out_rows_topk(const oracle_cfg *c, int32_t k, int32_t d, int32_t d_ff, const float *x,
                          const int32_t *dest, const uint8_t *keep, const float *w, const float *W1,
                          const float *b1, const float *W2, const float *b2, int32_t identity, int64_t nrows,
                          const int64_t *rows, double *out) {
    const int64_t G = (int64_t)c->n * c->m, T = c->T;
    double *y = (double *)malloc(sizeof(double) * (size_t)d);
    for (int64_t a = 0; a < nrows; ++a) {
        const int64_t g = rows[a];
        double *o = out + a * d;
        for (int32_t cc = 0; cc < d; ++cc) o[cc] = 0.0;
        for (int32_t j = 0; j < k; ++j) {
            const int64_t x_ = (int64_t)j * G * T + g;
            if (!keep[x_]) continue;
            const int64_t ex = dest[x_];
            if (identity) {
                for (int32_t cc = 0; cc < d; ++cc) y[cc] = (double)x[g * d + cc];
            } else {
                oracle_ffn_row(d, d_ff, x + g * d, W1 + ex * (int64_t)d * d_ff, b1 + ex * (int64_t)d_ff,
                               W2 + ex * (int64_t)d_ff * d, b2 + ex * (int64_t)d, y);
            }
            for (int32_t cc = 0; cc < d; ++cc) o[cc] += (double)w[x_] * y[cc];
        }
    }
    free(y);
}

/* ===================================================================================
 * Backward of the FLAT top-k layer (Eq. 2; readings R29-R32), the chain rule of
 *     J = sum_{r,t} < gout[r][t], OUT[r][t] > + lam * sum_r loss_r
 * with OUT = sum_j keep_j p_{e_j}(x) E_{e_j}(x) (p: the fp64 softmax of the fp64 logits)
 * and loss_r the Switch loss on the choice-0 fractions f (held constant).  The
 * choices, slots and keeps are those of oracle_route_topk (run on the fp32 logits).
 *   per kept choice j: dy_j = p_{e_j} gout; dgate_j = <gout, y_j>; the expert's FFN backward
 *   dl_k = sum_j dgate_j p_{e_j} (delta_{k, e_j} - p_k) + lam a K / T p_k (f_k - sum_i f_i p_i)
 *   dW += dl x^T;  dx = sum_j W1_{e_j} dz_j + W^T dl.
 * Outputs (fp64, overwritten): dlogits [G*T*K], dx [G*T*d], dW [K*d] (W != NULL), dW1, db1,
 * dW2, db2 per expert (as oracle_backward).
 * =================================================================================== */
void oracle_backward_topk(const oracle_cfg *c, int32_t k, int32_t d, int32_t d_ff, const float *x, const float *W,
                          const float *logits, const int32_t *dest, const uint8_t *keep, const int64_t *A1,
                          const float *W1, const float *b1, const float *W2, const float *b2, const float *gout,
                          double lam, double *dlogits, double *dx, double *dW, double *dW1, double *db1, double *dW2,
                          double *db2) {
    const int64_t G = (int64_t)c->n * c->m, T = c->T, K = G * c->e, NE = K;
    const int64_t nx = G * T * d;
    double *xd = (double *)malloc(sizeof(double) * (size_t)nx);
    for (int64_t i = 0; i < nx; ++i) xd[i] = (double)x[i];
    double *Wd = NULL, *ld = NULL;
    if (W) {
        Wd = (double *)malloc(sizeof(double) * (size_t)(K * d));
        for (int64_t i = 0; i < K * d; ++i) Wd[i] = (double)W[i];
    } else {
        ld = (double *)malloc(sizeof(double) * (size_t)(G * T * K));
        for (int64_t i = 0; i < G * T * K; ++i) ld[i] = (double)logits[i];
    }
    double *L = (double *)malloc(sizeof(double) * (size_t)(G * T * K));
    logits_f64(c, d, K, xd, Wd, ld, L);
    memset(dlogits, 0, sizeof(double) * (size_t)(G * T * K));
    memset(dx, 0, sizeof(double) * (size_t)nx);
    if (dW) memset(dW, 0, sizeof(double) * (size_t)(K * d));
    memset(dW1, 0, sizeof(double) * (size_t)(NE * d * d_ff));
    memset(db1, 0, sizeof(double) * (size_t)(NE * d_ff));
    memset(dW2, 0, sizeof(double) * (size_t)(NE * d_ff * d));
    memset(db2, 0, sizeof(double) * (size_t)(NE * d));
    double *pv = (double *)malloc(sizeof(double) * (size_t)K);
    double *a = (double *)malloc(sizeof(double) * (size_t)d_ff), *h = (double *)malloc(sizeof(double) * (size_t)d_ff);
    double *y = (double *)malloc(sizeof(double) * (size_t)d), *dy = (double *)malloc(sizeof(double) * (size_t)d);
    double *dz = (double *)malloc(sizeof(double) * (size_t)d_ff);
    double *w1 = (double *)malloc(sizeof(double) * (size_t)(d * d_ff)), *w2 = (double *)malloc(sizeof(double) * (size_t)(d * d_ff));
    double *bb1 = (double *)malloc(sizeof(double) * (size_t)d_ff), *bb2 = (double *)malloc(sizeof(double) * (size_t)d);
    double *dg = (double *)malloc(sizeof(double) * (size_t)k);
    for (int64_t r = 0; r < G; ++r) {
        for (int64_t t = 0; t < T; ++t) {
            const int64_t g = r * T + t;
            double *dl = dlogits + g * K;
            softmax_d(L + g * K, K, pv);
            for (int32_t j = 0; j < k; ++j) {
                const int64_t xj = (int64_t)j * G * T + g;
                dg[j] = 0.0;
                if (!keep[xj]) continue;
                const int64_t ex = dest[xj];
                for (int64_t z = 0; z < (int64_t)d * d_ff; ++z) { w1[z] = W1[ex * d * d_ff + z]; w2[z] = W2[ex * d_ff * d + z]; }
                for (int32_t f = 0; f < d_ff; ++f) bb1[f] = b1[ex * d_ff + f];
                for (int32_t cc = 0; cc < d; ++cc) bb2[cc] = b2[ex * d + cc];
                ffn_fwd_d(d, d_ff, xd + g * d, w1, bb1, w2, bb2, a, h, y);
                const double wj = pv[ex];
                for (int32_t cc = 0; cc < d; ++cc) {
                    dg[j] += (double)gout[g * d + cc] * y[cc];
                    dy[cc] = wj * (double)gout[g * d + cc];
                    db2[ex * d + cc] += dy[cc];
                }
                for (int32_t f = 0; f < d_ff; ++f) {
                    double dh = 0.0;
                    for (int32_t cc = 0; cc < d; ++cc) {
                        dW2[(ex * d_ff + f) * d + cc] += h[f] * dy[cc];
                        dh += w2[(int64_t)f * d + cc] * dy[cc];
                    }
                    dz[f] = dh * gelu_d(a[f]);
                    db1[ex * d_ff + f] += dz[f];
                }
                for (int32_t kk = 0; kk < d; ++kk) {
                    double s = 0.0;
                    for (int32_t f = 0; f < d_ff; ++f) {
                        dW1[(ex * d + kk) * d_ff + f] += xd[g * d + kk] * dz[f];
                        s += w1[(int64_t)kk * d_ff + f] * dz[f];
                    }
                    dx[g * d + kk] += s;
                }
            }
            double fp = 0.0;
            for (int64_t q = 0; q < K; ++q) fp += ((double)A1[r * K + q] / (double)T) * pv[q];
            for (int64_t q = 0; q < K; ++q) {
                double v = 0.0;
                for (int32_t j = 0; j < k; ++j) {
                    const int64_t ej = dest[(int64_t)j * G * T + g];
                    v += dg[j] * pv[ej] * ((q == ej ? 1.0 : 0.0) - pv[q]);
                }
                const double fq = (double)A1[r * K + q] / (double)T;
                dl[q] = v + lam * c->alpha * (double)K / (double)T * pv[q] * (fq - fp);
            }
            if (Wd) {
                for (int64_t q = 0; q < K; ++q)
                    for (int32_t cc = 0; cc < d; ++cc) {
                        if (dW) dW[q * d + cc] += dl[q] * xd[g * d + cc];
                        dx[g * d + cc] += dl[q] * Wd[q * d + cc];
                    }
            }
        }
    }
    free(xd); free(Wd); free(ld); free(L); free(pv); free(a); free(h); free(y); free(dy); free(dz);
    free(w1); free(w2); free(bb1); free(bb2); free(dg);
}

/* The objective J of oracle_backward_topk evaluated in fp64 with the routing decisions
 * (dest, keep) held fixed (to pin the backward by central finite differences; a caller
 * checks separately that its perturbations do not flip a decision). */
double oracle_objective_topk(const oracle_cfg *c, int32_t k, int32_t d, int32_t d_ff, const double *x, const double *W,
                             const double *logits, const int32_t *dest, const uint8_t *keep, const int64_t *A1,
                             const double *W1, const double *b1, const double *W2, const double *b2,
                             const double *gout, double lam) {
    const int64_t G = (int64_t)c->n * c->m, T = c->T, K = G * c->e;
    double *L = (double *)malloc(sizeof(double) * (size_t)(G * T * K));
    logits_f64(c, d, K, x, W, logits, L);
    double *pv = (double *)malloc(sizeof(double) * (size_t)K), *P = (double *)malloc(sizeof(double) * (size_t)K);
    double *a = (double *)malloc(sizeof(double) * (size_t)d_ff), *h = (double *)malloc(sizeof(double) * (size_t)d_ff);
    double *y = (double *)malloc(sizeof(double) * (size_t)d);
    double J = 0.0;
    for (int64_t r = 0; r < G; ++r) {
        memset(P, 0, sizeof(double) * (size_t)K);
        for (int64_t t = 0; t < T; ++t) {
            const int64_t g = r * T + t;
            softmax_d(L + g * K, K, pv);
            for (int64_t q = 0; q < K; ++q) P[q] += pv[q] / (double)T;
            for (int32_t j = 0; j < k; ++j) {
                const int64_t xj = (int64_t)j * G * T + g;
                if (!keep[xj]) continue;
                const int64_t ex = dest[xj];
                ffn_fwd_d(d, d_ff, x + g * d, W1 + ex * (int64_t)d * d_ff, b1 + ex * (int64_t)d_ff,
                          W2 + ex * (int64_t)d_ff * d, b2 + ex * (int64_t)d, a, h, y);
                for (int32_t cc = 0; cc < d; ++cc) J += gout[g * d + cc] * pv[ex] * y[cc];
            }
        }
        double l1 = 0.0;
        for (int64_t q = 0; q < K; ++q) l1 += ((double)A1[r * K + q] / (double)T) * P[q];
        J += lam * c->alpha * (double)K * l1;
    }
    free(L); free(pv); free(P); free(a); free(h); free(y);
    return J;
}
