/*
 * nj_oracle.c — fp64 CPU ORACLE for batched speculative-decoding verification.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2512_22420_b200/csrc) and never includes include/nj.h.
 *
 * What it computes (plain definitions, no blocking / fusion / reordering):
 *   Leviathan speculative sampling as cited at PAPER.md:23 ("the target model
 *   then verifies in parallel. This process is lossless"), with the step list
 *   of BASELINE.json north_star: (1) LM-head projection, (2) softmax over the
 *   vocabulary, (3) accept draft i with prob min(1, p/q), first rejection,
 *   resample from norm(max(0, p - q)), bonus token on full acceptance.
 *   Readings of the paper's silences are DESIGN.md R1..R12 (referenced below).
 *
 * Inputs are converted exactly: bf16 -> fp64, fp32 -> fp64.  Every sum runs
 * in ascending index order in fp64; exp/log are libm.
 *
 * Build: gcc -O2 -fopenmp -fPIC -shared nj_oracle.c -o liboracle.so -lm
 * (no -ffast-math: summation order is part of the definition).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* bf16 bit pattern -> fp64 (exact): bf16 is the top half of an IEEE fp32. */
static double bf16_to_f64(uint16_t b) {
    uint32_t u = ((uint32_t)b) << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
}

static void set_threads(int nthreads) {
#ifdef _OPENMP
    static int dflt = 0;   /* the process default, restored when nthreads <= 0 */
    if (!dflt) dflt = omp_get_max_threads();
    omp_set_num_threads(nthreads > 0 ? nthreads : dflt);
#else
    (void)nthreads;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    set_threads(0);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Step (1), LM-head projection (BJ step 1; "verifies in parallel"):
 *   out[r*V + x] = sum_{k<d} W[x,k] * H[rows[r],k]      (fp64, k ascending)
 * rows == NULL means rows[r] = r. */
int oracle_logits(const uint16_t* H, const int32_t* rows, int64_t n_rows,
                  const uint16_t* W, int64_t V, int64_t d,
                  double* out, int nthreads) {
    if (n_rows <= 0 || V <= 0 || d <= 0) return 0;
    set_threads(nthreads);
    double* h = (double*)malloc(sizeof(double) * (size_t)(n_rows * d));
    if (!h) return 1;
    for (int64_t r = 0; r < n_rows; ++r) {
        int64_t src = rows ? rows[r] : r;
        for (int64_t k = 0; k < d; ++k) h[r * d + k] = bf16_to_f64(H[src * d + k]);
    }
    int err = 0;
#pragma omp parallel
    {
        double* w = (double*)malloc(sizeof(double) * (size_t)d);
        if (!w) {
#pragma omp atomic write
            err = 1;
        } else {
#pragma omp for schedule(static)
            for (int64_t x = 0; x < V; ++x) {
                for (int64_t k = 0; k < d; ++k) w[k] = bf16_to_f64(W[x * d + k]);
                for (int64_t r = 0; r < n_rows; ++r) {
                    const double* hr = h + r * d;
                    double acc = 0.0;
                    for (int64_t k = 0; k < d; ++k) acc += w[k] * hr[k];
                    out[r * V + x] = acc;
                }
            }
            free(w);
        }
    }
    free(h);
    return err;
}

/* Step (2), softmax statistics of one row (BJ step 2):
 *   m = max_x l(x),  s = sum_x exp(l(x) - m),  lse = m + log(s). */
static double row_lse(const double* l, int64_t V) {
    double m = -INFINITY;
    for (int64_t x = 0; x < V; ++x) if (l[x] > m) m = l[x];
    double s = 0.0;
    for (int64_t x = 0; x < V; ++x) s += exp(l[x] - m);
    return m + log(s);
}

typedef struct {
    /* per row [N] */
    double* lse;
    /* per draft [G] */
    double* p_draft;   /* p_i(x_i)                                   */
    double* ratio;     /* a_i = p_i(x_i) / q_i(x_i)  (+inf if q = 0)  */
    /* per request [B] */
    double* mass;      /* W_b of the distribution drawn from          */
    double* F_lo;      /* C(t-1) / W_b                                */
    double* F_hi;      /* C(t)   / W_b                                */
    int32_t* flags;    /* 1 accept-tie, 2 draw-tie, 4 zero-mass, 8 clamp, 16 q=0 */
    double* accept_margin; /* min_{tested i} |a_i - u_i|  (+inf if none) */
    double* draw_margin;   /* min(|F_hi - u|, |u - F_lo|)               */
} oracle_debug;

#define OF_ACCEPT_TIE 1
#define OF_DRAW_TIE   2
#define OF_ZERO_MASS  4
#define OF_CLAMP      8
#define OF_Q_ZERO     16

/* Steps (3)-(6) for one request, given its gamma+1 fp64 logit rows.
 *   l      [gamma+1][V] logits (row j = position j), lse[gamma+1]
 *   x      [gamma] draft tokens, q [gamma] rows (stride ldq)
 *   u      [gamma+1] uniforms (slot gamma = final draw, R3)
 * Writes n, t and debug values; tie_eps is the near-tie band (R12). */
static void verify_one(const double* l, int64_t V, const double* lse,
                       int gamma, const int32_t* x, const float* q, int64_t ldq,
                       const double* u, double tie_eps,
                       int32_t* n_out, int32_t* t_out,
                       double* p_draft, double* ratio,
                       double* mass_out, double* flo_out, double* fhi_out,
                       int32_t* flags_out, double* am_out, double* dm_out,
                       double* ptie_out, double* w /* scratch [V] */) {
    int32_t flags = 0;
    double amargin = INFINITY;
    double ptie = 0.0;   /* R12: probability over the uniforms of a tie flag */
    /* (3) acceptance: accept iff u_i * q_i(x_i) < p_i(x_i) (strict, R2);
     *     n = first failing i, else gamma.                               */
    int n = gamma;
    for (int i = 0; i < gamma; ++i) {
        double p = exp(l[(int64_t)i * V + x[i]] - lse[i]);
        double qx = (double)q[(int64_t)i * ldq + x[i]];
        double a = (qx > 0.0) ? p / qx : INFINITY;
        if (!(qx > 0.0)) flags |= OF_Q_ZERO;
        if (p_draft) p_draft[i] = p;
        if (ratio) ratio[i] = a;
        double mg = fabs(a - u[i]);
        if (mg < amargin) amargin = mg;
        if (mg <= tie_eps) flags |= OF_ACCEPT_TIE;
        /* P(|u_i - a_i| <= tie_eps) for u_i ~ U[0,1): |[a - eps, a + eps] n [0, 1)| */
        ptie += fmax(0.0, fmin(a + tie_eps, 1.0) - fmax(a - tie_eps, 0.0));
        if (!(u[i] * qx < p)) { n = i; break; }
    }
    /* later drafts are never tested; their p/ratio are still reported */
    for (int i = n + 1; i < gamma; ++i) {
        double p = exp(l[(int64_t)i * V + x[i]] - lse[i]);
        double qx = (double)q[(int64_t)i * ldq + x[i]];
        if (p_draft) p_draft[i] = p;
        if (ratio) ratio[i] = (qx > 0.0) ? p / qx : INFINITY;
    }
    /* (4) final distribution: residual max(0, p_n - q_n) after a rejection,
     *     bonus p_gamma after full acceptance.                            */
    const double* ln = l + (int64_t)n * V;
    const double lsen = lse[n];
    double W = 0.0;
    if (n < gamma) {
        const float* qn = q + (int64_t)n * ldq;
        for (int64_t v = 0; v < V; ++v) {
            double d = exp(ln[v] - lsen) - (double)qn[v];
            w[v] = d > 0.0 ? d : 0.0;
            W += w[v];
        }
    } else {
        for (int64_t v = 0; v < V; ++v) { w[v] = exp(ln[v] - lsen); W += w[v]; }
    }
    if (W == 0.0) {  /* R6: residual mass 0 -> draw from p_n */
        flags |= OF_ZERO_MASS;
        W = 0.0;
        for (int64_t v = 0; v < V; ++v) { w[v] = exp(ln[v] - lsen); W += w[v]; }
    }
    /* (5) inverse CDF: t = min{x : C(x) > u*W}, ascending id (R5). */
    const double T = u[gamma] * W;
    double C = 0.0, Cprev = 0.0;
    int64_t t = -1;
    for (int64_t v = 0; v < V; ++v) {
        Cprev = C;
        C += w[v];
        if (C > T) { t = v; break; }
    }
    if (t < 0) {  /* rounding overshoot: last x with positive weight */
        flags |= OF_CLAMP;
        for (int64_t v = V - 1; v >= 0; --v) if (w[v] > 0.0) { t = v; break; }
        C = W; Cprev = W - w[t];
    }
    double Flo = Cprev / W, Fhi = C / W;
    double dmargin = fmin(fabs(Fhi - u[gamma]), fabs(u[gamma] - Flo));
    if (dmargin <= tie_eps) flags |= OF_DRAW_TIE;
    /* P(draw tie) for u_gamma ~ U[0,1): token x owns [F(x-1), F(x)) of width
     * w(x)/W, and u is flagged iff it lies within tie_eps of either end of the
     * interval it falls in, so the flagged measure is sum_x min(w(x)/W, 2 eps). */
    for (int64_t v = 0; v < V; ++v)
        if (w[v] > 0.0) ptie += fmin(w[v] / W, 2.0 * tie_eps);
    *n_out = n;
    *t_out = (int32_t)t;
    if (mass_out) *mass_out = W;
    if (flo_out) *flo_out = Flo;
    if (fhi_out) *fhi_out = Fhi;
    if (flags_out) *flags_out = flags;
    if (am_out) *am_out = amargin;
    if (dm_out) *dm_out = dmargin;
    if (ptie_out) *ptie_out = ptie;
}

/* Steps (2)-(6) of a packed ragged batch (layout as include/nj.h, but this
 * file does not include it) given the fp64 logits L[N][V] of its rows (step 1,
 * oracle_logits).  u is fp64 here (the fp32 uniforms converted exactly by the
 * caller; the brute-force checker and the tie-branch checks of the tests pass
 * values that are not fp32).  Debug pointers may be NULL.  Requests are
 * processed independently (OpenMP over requests). */
int oracle_verify_logits(const double* L, int64_t V,
                         const int32_t* draft_tokens, const float* q, int64_t ldq,
                         const int32_t* gamma, const double* u, int32_t B,
                         int32_t* accept_len, int32_t* next_token,
                         double* dbg_lse, double* dbg_p_draft, double* dbg_ratio,
                         double* dbg_mass, double* dbg_flo, double* dbg_fhi,
                         int32_t* dbg_flags, double* dbg_amargin, double* dbg_dmargin,
                         double* dbg_ptie, double tie_eps, int nthreads) {
    int64_t N = 0;
    for (int32_t b = 0; b < B; ++b) N += gamma[b] + 1;
    double* lse = (double*)malloc(sizeof(double) * (size_t)N);
    int64_t* row_off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(B + 1));
    int64_t* drf_off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(B + 1));
    if (!lse || !row_off || !drf_off) { free(lse); free(row_off); free(drf_off); return 1; }
    set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < N; ++r) lse[r] = row_lse(L + r * V, V);
    if (dbg_lse) memcpy(dbg_lse, lse, sizeof(double) * (size_t)N);
    row_off[0] = 0; drf_off[0] = 0;
    for (int32_t b = 0; b < B; ++b) {
        row_off[b + 1] = row_off[b] + gamma[b] + 1;
        drf_off[b + 1] = drf_off[b] + gamma[b];
    }
    int err = 0;
#pragma omp parallel
    {
        double* w = (double*)malloc(sizeof(double) * (size_t)V);
        if (!w) {
#pragma omp atomic write
            err = 1;
        } else {
#pragma omp for schedule(dynamic, 1)
            for (int32_t b = 0; b < B; ++b) {
                int64_t r0 = row_off[b], g0 = drf_off[b];
                verify_one(L + r0 * V, V, lse + r0, gamma[b],
                           draft_tokens + g0, q + g0 * ldq, ldq, u + r0, tie_eps,
                           accept_len + b, next_token + b,
                           dbg_p_draft ? dbg_p_draft + g0 : NULL,
                           dbg_ratio ? dbg_ratio + g0 : NULL,
                           dbg_mass ? dbg_mass + b : NULL,
                           dbg_flo ? dbg_flo + b : NULL,
                           dbg_fhi ? dbg_fhi + b : NULL,
                           dbg_flags ? dbg_flags + b : NULL,
                           dbg_amargin ? dbg_amargin + b : NULL,
                           dbg_dmargin ? dbg_dmargin + b : NULL,
                           dbg_ptie ? dbg_ptie + b : NULL, w);
            }
            free(w);
        }
    }
    free(row_off); free(drf_off); free(lse);
    return err;
}

/* Full verification: step (1) by oracle_logits, then oracle_verify_logits. */
int oracle_verify(const uint16_t* H, const uint16_t* W, int64_t V, int64_t d,
                  const int32_t* draft_tokens, const float* q, int64_t ldq,
                  const int32_t* gamma, const double* u, int32_t B,
                  int32_t* accept_len, int32_t* next_token,
                  double* dbg_lse, double* dbg_p_draft, double* dbg_ratio,
                  double* dbg_mass, double* dbg_flo, double* dbg_fhi,
                  int32_t* dbg_flags, double* dbg_amargin, double* dbg_dmargin,
                  double* dbg_ptie, double tie_eps, int nthreads) {
    int64_t N = 0;
    for (int32_t b = 0; b < B; ++b) N += gamma[b] + 1;
    double* L = (double*)malloc(sizeof(double) * (size_t)(N * V));
    if (!L) return 1;
    if (oracle_logits(H, NULL, N, W, V, d, L, nthreads)) { free(L); return 1; }
    int err = oracle_verify_logits(L, V, draft_tokens, q, ldq, gamma, u, B, accept_len, next_token,
                                   dbg_lse, dbg_p_draft, dbg_ratio, dbg_mass, dbg_flo, dbg_fhi,
                                   dbg_flags, dbg_amargin, dbg_dmargin, dbg_ptie, tie_eps, nthreads);
    free(L);
    return err;
}

/* Stage-isolated sampler oracle (R11(ii)): given fp32 logits of one
 * row per request, lse is computed in fp64 from those logits, then the
 * residual (residual[b] != 0: w = max(0, p - q_b)) or bonus (w = p) draw of
 * steps (4)-(5) exactly as in verify_one. */
int oracle_sample_from_logits(const float* logits, int64_t ld_l, int64_t V,
                              const int32_t* residual, const float* q, int64_t ldq,
                              const double* u, int32_t B,
                              int32_t* next_token, double* mass,
                              double* flo, double* fhi, int32_t* flags,
                              double tie_eps, int nthreads) {
    set_threads(nthreads);
    int err = 0;
#pragma omp parallel
    {
        double* l = (double*)malloc(sizeof(double) * (size_t)V);
        double* w = (double*)malloc(sizeof(double) * (size_t)V);
        if (!l || !w) {
#pragma omp atomic write
            err = 1;
        } else {
#pragma omp for schedule(dynamic, 1)
            for (int32_t b = 0; b < B; ++b) {
                for (int64_t v = 0; v < V; ++v) l[v] = (double)logits[b * ld_l + v];
                double lse = row_lse(l, V);
                /* Reuse verify_one with gamma = 1 (residual: a forced rejection
                 * at i = 0) or gamma = 0 (bonus): both reach steps (4)-(5)
                 * with the single row l.  For the residual case the acceptance
                 * test must fail, which u_0 = +inf guarantees without
                 * touching the draw (slot gamma = 1).                       */
                int32_t n, t, fl;
                double W, Flo, Fhi, am, dm;
                if (residual[b]) {
                    double uu[2] = {INFINITY, u[b]};
                    int32_t x0 = 0;
                    double lse2[2] = {lse, lse};
                    /* rows 0 and 1 both alias l: n = 0, so row 1 is unused */
                    double* l2 = (double*)malloc(sizeof(double) * (size_t)(2 * V));
                    memcpy(l2, l, sizeof(double) * (size_t)V);
                    memcpy(l2 + V, l, sizeof(double) * (size_t)V);
                    verify_one(l2, V, lse2, 1, &x0, q + (int64_t)b * ldq, ldq, uu, tie_eps,
                               &n, &t, NULL, NULL, &W, &Flo, &Fhi, &fl, &am, &dm, NULL, w);
                    free(l2);
                } else {
                    double uu[1] = {u[b]};
                    verify_one(l, V, &lse, 0, NULL, q, ldq, uu, tie_eps,
                               &n, &t, NULL, NULL, &W, &Flo, &Fhi, &fl, &am, &dm, NULL, w);
                }
                next_token[b] = t;
                if (mass) mass[b] = W;
                if (flo) flo[b] = Flo;
                if (fhi) fhi[b] = Fhi;
                if (flags) flags[b] = fl & ~OF_ACCEPT_TIE;
            }
        }
        free(l); free(w);
    }
    return err;
}
