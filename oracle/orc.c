/*
 * orc.c -- plain, slow, FP64 CPU ORACLE for Bi-cADMM (arXiv 2405.16267).
 *
 * TEST INFRASTRUCTURE ONLY (see orc.h).  Every function follows the paper's
 * definition or algorithm step by step, in the paper's order and notation.
 * No blocking, fusion or reordering: each output element is one sequential
 * sum in ascending index order, so results do not depend on OMP_NUM_THREADS
 * (OpenMP only distributes independent output elements).
 *
 * Deliberately INDEPENDENT of the CUDA path: different algorithms where the
 * paper allows a choice --
 *   - block x-update: Cholesky factor + two triangular solves (GPU: explicit inverse)
 *   - (7b): exact sort-and-scan over breakpoints (GPU: bisection on bit patterns)
 *   - (13): full sort by (|z| desc, index asc) (GPU: radix select)
 *   - logistic prox (22): bisection on the monotone derivative (GPU: Newton)
 *   - softmax prox (22): Newton with a dense C x C Gaussian elimination
 *     (GPU: Sherman-Morrison)
 *
 * parity pins: see tests/test_oracle_*.py (values from S:*, App. B of SURVEY.md,
 * closed forms and brute force).  Parity unpinned: none.
 */
#include "orc.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>
#ifdef _OPENMP
#include <omp.h>
static double orc_now(void) { return omp_get_wtime(); }
#else
#include <time.h>
static double orc_now(void) { struct timespec ts; clock_gettime(CLOCK_MONOTONIC, &ts); return ts.tv_sec + 1e-9 * ts.tv_nsec; }
#endif

static double sgn(double a) { return a > 0 ? 1.0 : (a < 0 ? -1.0 : 0.0); }
static double clampd(double a, double lo, double hi) { return a < lo ? lo : (a > hi ? hi : a); }

/* ------------------------------------------------------------------------- */
/* Losses.  P:50 names the four models; P:259 fixes LS as ||Ax-b||^2 (no 1/2). */
/* phi(w,b): LS (w-b)^2; logistic ln(1+exp(-b w)); hinge max(0,1-b w);        */
/* softmax logsumexp(w) - w_b (DESIGN R12, R13).                              */
/* ------------------------------------------------------------------------- */
static double log1pexp(double a) { /* ln(1+e^a), overflow-safe */
    return a > 0 ? a + log1p(exp(-a)) : log1p(exp(a));
}

double orc_phi(int loss, int C, const double* w, double b) {
    switch (loss) {
    case ORC_LS: { double r = w[0] - b; return r * r; }
    case ORC_LOGISTIC: return log1pexp(-b * w[0]);
    case ORC_HINGE: { double h = 1.0 - b * w[0]; return h > 0 ? h : 0.0; }
    case ORC_SOFTMAX: {
        double mx = w[0];
        for (int c = 1; c < C; ++c) if (w[c] > mx) mx = w[c];
        double se = 0.0;
        for (int c = 0; c < C; ++c) se += exp(w[c] - mx);
        return mx + log(se) - w[(int)b];
    }
    }
    return NAN;
}

static int label_ok(int loss, int C, double b) {
    if (loss == ORC_LOGISTIC || loss == ORC_HINGE) return b == 1.0 || b == -1.0;
    if (loss == ORC_SOFTMAX) return b >= 0 && b < C && b == floor(b);
    return isfinite(b);
}

/* S:56-64 loss_value: sum_r phi(w_r, b_r). */
int orc_loss_value(int loss, int C, int64_t m, const double* w, const double* b, double* out) {
    double acc = 0.0;
    for (int64_t r = 0; r < m; ++r) {
        if (!label_ok(loss, C, b[r])) return ORC_ERR_DOMAIN;
        acc += orc_phi(loss, C, w + r * C, b[r]);
    }
    *out = acc;
    return ORC_OK;
}

/* Problem (1): sum_i l_i(A_i x - b_i) + 1/(2 gamma) ||x||^2 (DESIGN R20). */
int orc_objective(const orc_problem* pb, double gamma, const double* x, double* out) {
    const int C = pb->C;
    const int64_t n = pb->n;
    double total = 0.0;
    for (int i = 0; i < pb->N; ++i) {
        int64_t m = pb->m[i];
        double* w = (double*)malloc(sizeof(double) * (size_t)(m * C + 1));
        if (!w) return ORC_ERR_NOMEM;
        orc_gemv(m, n, pb->A[i], n, C, x, w);
        double li;
        int rc = orc_loss_value(pb->loss, C, m, w, pb->b[i], &li);
        free(w);
        if (rc) return rc;
        total += li;
    }
    double nx = 0.0;
    for (int64_t l = 0; l < n * C; ++l) nx += x[l] * x[l];
    *out = total + nx / (2.0 * gamma);
    return ORC_OK;
}

/* kappa = round(n(1 - s_l)), half away from zero (DESIGN R21). */
int64_t orc_kappa_from_sparsity(int64_t n, double s_l) {
    if (!(s_l > 0.0 && s_l < 1.0)) return ORC_ERR_DOMAIN;
    return (int64_t)llround((double)n * (1.0 - s_l));
}

/* ------------------------------------------------------------------------- */
/* Theorem 1: ||x||_0 <= kappa  iff  exists s,t with x's = t,        */
/* ||x||_1 <= t, ||s||_1 <= kappa, ||s||_inf <= 1.  Witness per S:110.        */
/* ------------------------------------------------------------------------- */
int orc_l0_witness(int64_t n, const double* x, int64_t kappa, double* s, double* t) {
    int64_t nnz = 0;
    double l1 = 0.0;
    for (int64_t l = 0; l < n; ++l) { if (x[l] != 0.0) ++nnz; l1 += fabs(x[l]); }
    if (nnz > kappa) return ORC_ERR_INFEASIBLE;
    for (int64_t l = 0; l < n; ++l) s[l] = sgn(x[l]);
    *t = l1;
    return ORC_OK;
}

int orc_check_theorem1(int64_t n, const double* x, const double* s, double t, double kappa, double tol) {
    double xs = 0, l1 = 0, s1 = 0, sinf = 0;
    for (int64_t l = 0; l < n; ++l) {
        xs += x[l] * s[l]; l1 += fabs(x[l]); s1 += fabs(s[l]);
        if (fabs(s[l]) > sinf) sinf = fabs(s[l]);
    }
    return fabs(xs - t) <= tol && l1 <= t + tol && s1 <= kappa + tol && sinf <= 1.0 + tol;
}

static int cmp_desc(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return x < y ? 1 : (x > y ? -1 : 0);
}

/* S:125-133 Euclidean projection onto {(z,t): ||z||_1 <= t} by sort and scan. */
void orc_proj_l1_epigraph(int64_t n, const double* z, double t, double* z_out, double* t_out) {
    double l1 = 0.0, mx = 0.0;
    for (int64_t l = 0; l < n; ++l) { l1 += fabs(z[l]); if (fabs(z[l]) > mx) mx = fabs(z[l]); }
    if (l1 <= t) { memcpy(z_out, z, sizeof(double) * (size_t)n); *t_out = t; return; }
    if (mx <= -t) { memset(z_out, 0, sizeof(double) * (size_t)n); *t_out = 0.0; return; }
    double* a = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t l = 0; l < n; ++l) a[l] = fabs(z[l]);
    qsort(a, (size_t)n, sizeof(double), cmp_desc);
    double S = 0.0, mu = 0.0;
    for (int64_t k = 1; k <= n; ++k) {
        S += a[k - 1];
        mu = (S - t) / (double)(k + 1);
        double next = k < n ? a[k] : 0.0;
        if (mu <= a[k - 1] && mu >= next) break;
    }
    free(a);
    for (int64_t l = 0; l < n; ++l) z_out[l] = sgn(z[l]) * fmax(fabs(z[l]) - mu, 0.0);
    *t_out = t + mu;
}

/* ------------------------------------------------------------------------- */
/* Per-sample omega-bar prox, Eq. (22):                            */
/*   omega = argmin phi(M w, b) + (M rho_l / 2) ||w - p||^2,  p = abar + nu.  */
/* "splits entirely into m_i scalar optimization problems".           */
/* ------------------------------------------------------------------------- */
static double sigmoid(double a) { /* 1/(1+e^-a), overflow-safe */
    if (a >= 0) return 1.0 / (1.0 + exp(-a));
    double e = exp(a);
    return e / (1.0 + e);
}

/* logistic stationarity: g(w) = -b*sigma(-b M w) + rho_l (w - p), increasing in w. */
static double logistic_g(int M, double rho_l, double b, double p, double w) {
    return -b * sigmoid(-b * (double)M * w) + rho_l * (w - p);
}

/* Solve the C x C system H d = g by Gaussian elimination with partial pivoting. */
static void dense_solve(int C, double* H, double* g) {
    for (int k = 0; k < C; ++k) {
        int piv = k;
        for (int i = k + 1; i < C; ++i) if (fabs(H[i * C + k]) > fabs(H[piv * C + k])) piv = i;
        if (piv != k) {
            for (int j = 0; j < C; ++j) { double tmp = H[k * C + j]; H[k * C + j] = H[piv * C + j]; H[piv * C + j] = tmp; }
            double tmp = g[k]; g[k] = g[piv]; g[piv] = tmp;
        }
        for (int i = k + 1; i < C; ++i) {
            double f = H[i * C + k] / H[k * C + k];
            for (int j = k; j < C; ++j) H[i * C + j] -= f * H[k * C + j];
            g[i] -= f * g[k];
        }
    }
    for (int k = C - 1; k >= 0; --k) {
        double acc = g[k];
        for (int j = k + 1; j < C; ++j) acc -= H[k * C + j] * g[j];
        g[k] = acc / H[k * C + k];
    }
}

static double softmax_obj(int C, int M, double rho_l, int y, const double* p, const double* w) {
    double mw[64];
    double q = 0.0;
    for (int c = 0; c < C; ++c) { mw[c] = (double)M * w[c]; q += (w[c] - p[c]) * (w[c] - p[c]); }
    return orc_phi(ORC_SOFTMAX, C, mw, (double)y) + 0.5 * (double)M * rho_l * q;
}

int orc_prox_omega(int loss, int C, int M, double rho_l, double b, const double* p, double* omega) {
    if (!label_ok(loss, C, b)) return ORC_ERR_DOMAIN;
    switch (loss) {
    case ORC_LS:
        /* d/dw: 2M(Mw - b) + M rho_l (w - p) = 0  =>  w = (2b + rho_l p)/(2M + rho_l) */
        omega[0] = (2.0 * b + rho_l * p[0]) / (2.0 * M + rho_l);
        return ORC_OK;
    case ORC_HINGE: {
        /* y = b w, p' = b p; minimise max(0, 1 - M y) + (M rho_l/2)(y - p')^2 (DESIGN R14). */
        double pp = b * p[0], y;
        if ((double)M * pp > 1.0) y = pp;
        else if ((double)M * (pp + 1.0 / rho_l) < 1.0) y = pp + 1.0 / rho_l;
        else y = 1.0 / (double)M;
        omega[0] = b * y;
        return ORC_OK;
    }
    case ORC_LOGISTIC: {
        /* Bisection on the increasing stationarity function over its bracket
         * [p - 1/rho_l, p + 1/rho_l] until no double lies strictly between. */
        double lo = p[0] - 1.0 / rho_l, hi = p[0] + 1.0 / rho_l;
        for (int it = 0; it < 2200; ++it) {
            double mid = lo + 0.5 * (hi - lo);
            if (mid <= lo || mid >= hi) break;
            if (logistic_g(M, rho_l, b, p[0], mid) > 0.0) hi = mid; else lo = mid;
        }
        double glo = fabs(logistic_g(M, rho_l, b, p[0], lo));
        double ghi = fabs(logistic_g(M, rho_l, b, p[0], hi));
        omega[0] = glo <= ghi ? lo : hi;
        return ORC_OK;
    }
    case ORC_SOFTMAX: {
        /* Damped Newton on the strongly convex C-dim problem; Hessian
         * M(diag pi - pi pi^T) + rho_l I solved densely. */
        if (C > 64) return ORC_ERR_INVALID;
        int y = (int)b;
        double w[64], g[64], H[64 * 64], pi[64], trial[64];
        for (int c = 0; c < C; ++c) w[c] = p[c];
        for (int it = 0; it < 100; ++it) {
            double mx = -INFINITY, se = 0.0;
            for (int c = 0; c < C; ++c) if ((double)M * w[c] > mx) mx = (double)M * w[c];
            for (int c = 0; c < C; ++c) { pi[c] = exp((double)M * w[c] - mx); se += pi[c]; }
            for (int c = 0; c < C; ++c) pi[c] /= se;
            double gn = 0.0;
            for (int c = 0; c < C; ++c) {
                g[c] = pi[c] - (c == y ? 1.0 : 0.0) + rho_l * (w[c] - p[c]);
                gn += g[c] * g[c];
            }
            for (int i = 0; i < C; ++i)
                for (int j = 0; j < C; ++j)
                    H[i * C + j] = (double)M * ((i == j ? pi[i] : 0.0) - pi[i] * pi[j]) + (i == j ? rho_l : 0.0);
            dense_solve(C, H, g); /* g <- Newton direction */
            double f0 = softmax_obj(C, M, rho_l, y, p, w), step = 1.0, dmax = 0.0, wmax = 1.0;
            for (int ls = 0; ls < 60; ++ls) {
                for (int c = 0; c < C; ++c) trial[c] = w[c] - step * g[c];
                /* accept when the objective does not rise beyond rounding (Newton is
                 * locally quadratic; only far from the optimum does this backtrack) */
                if (softmax_obj(C, M, rho_l, y, p, trial) <= f0 + 1e-12 * (1.0 + fabs(f0))) break;
                step *= 0.5;
            }
            for (int c = 0; c < C; ++c) {
                double d = step * g[c];
                if (fabs(d) > dmax) dmax = fabs(d);
                w[c] -= d;
                if (fabs(w[c]) > wmax) wmax = fabs(w[c]);
            }
            if (dmax <= 4.0 * DBL_EPSILON * wmax || gn == 0.0) break;
        }
        for (int c = 0; c < C; ++c) omega[c] = w[c];
        return ORC_OK;
    }
    }
    return ORC_ERR_INVALID;
}

/* ------------------------------------------------------------------------- */
/* Global (z,t)-update, Eq. (7b), solved exactly (DESIGN R3):          */
/*   min over ||z||_1 <= t of (N rho_c/2)||z - wbar||^2 + (rho_b/2)(s'z-t+v)^2 */
/* KKT: z_l = sgn(wbar_l) max(|wbar_l| - tau d_l, 0),        */
/* d_l = 1 - s_l sgn(wbar_l), tau the root of N rho_c tau = rho_b(psi(tau)-v), */
/* psi(tau) = sum_l d_l |z_l(tau)|.  Root found by sorting the breakpoints    */
/* beta_l = |wbar_l|/d_l in descending order and scanning the segments.       */
/* ------------------------------------------------------------------------- */
typedef struct { double beta; int64_t idx; } orc_bp;
static int cmp_bp_desc(const void* a, const void* b) {
    const orc_bp* x = (const orc_bp*)a; const orc_bp* y = (const orc_bp*)b;
    if (x->beta > y->beta) return -1;
    if (x->beta < y->beta) return 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);
}

void orc_zt_update(int64_t len, int N, double rho_c, double rho_b, const double* wbar,
                   const double* s, double v, double* z, double* t, double* tau_out) {
    double* d = (double*)malloc(sizeof(double) * (size_t)(len + 1));
    double psi0 = 0.0, sw = 0.0;
    for (int64_t l = 0; l < len; ++l) {
        d[l] = 1.0 - s[l] * sgn(wbar[l]);
        psi0 += d[l] * fabs(wbar[l]);
        sw += s[l] * wbar[l];
    }
    double tau = 0.0;
    if (psi0 <= v) {
        /* Case 1: the bilinear penalty is inactive; z = wbar, t = s'wbar + v. */
        for (int64_t l = 0; l < len; ++l) z[l] = wbar[l];
        *t = sw + v;
    } else {
        orc_bp* bp = (orc_bp*)malloc(sizeof(orc_bp) * (size_t)(len + 1));
        int64_t K = 0;
        for (int64_t l = 0; l < len; ++l)
            if (d[l] > 0.0 && wbar[l] != 0.0) { bp[K].beta = fabs(wbar[l]) / d[l]; bp[K].idx = l; ++K; }
        qsort(bp, (size_t)K, sizeof(orc_bp), cmp_bp_desc);
        const double Nrc = (double)N * rho_c;
        double Asum = 0.0, Bsum = 0.0;
        for (int64_t k = 0; k <= K; ++k) {
            double next = k < K ? bp[k].beta : 0.0;
            /* f(next) with active set = the k largest breakpoints */
            double f = Nrc * next - rho_b * (Asum - next * Bsum - v);
            if (f <= 0.0) { tau = rho_b * (Asum - v) / (Nrc + rho_b * Bsum); break; }
            int64_t l = bp[k].idx;
            Asum += d[l] * fabs(wbar[l]);
            Bsum += d[l] * d[l];
        }
        free(bp);
        double l1 = 0.0;
        for (int64_t l = 0; l < len; ++l) {
            z[l] = sgn(wbar[l]) * fmax(fabs(wbar[l]) - tau * d[l], 0.0);
            l1 += fabs(z[l]);
        }
        *t = l1;
    }
    if (tau_out) *tau_out = tau;
    free(d);
}

/* SPEC S:262-270 projected-gradient (z,t) solver: used ONLY to cross-check the
 * exact solve above in tests (two independent methods for the same argmin). */
void orc_zt_pgd(int64_t len, int N, double rho_c, double rho_b, const double* wbar,
                const double* s, double v, double step_tol, int max_steps, double* z, double* t) {
    double ss = 0.0, l1 = 0.0;
    for (int64_t l = 0; l < len; ++l) { ss += s[l] * s[l]; l1 += fabs(wbar[l]); }
    const double L = (double)N * rho_c + rho_b * (ss + 1.0);
    double* zc = (double*)malloc(sizeof(double) * (size_t)len);
    double* zn = (double*)malloc(sizeof(double) * (size_t)len);
    double tc;
    orc_proj_l1_epigraph(len, wbar, l1, zc, &tc);
    for (int it = 0; it < max_steps; ++it) {
        double g = -tc + v;
        for (int64_t l = 0; l < len; ++l) g += s[l] * zc[l];
        for (int64_t l = 0; l < len; ++l)
            zn[l] = zc[l] - ((double)N * rho_c * (zc[l] - wbar[l]) + rho_b * g * s[l]) / L;
        double tn_in = tc + rho_b * g / L, tn;
        orc_proj_l1_epigraph(len, zn, tn_in, zn, &tn);
        double dist = (tn - tc) * (tn - tc);
        for (int64_t l = 0; l < len; ++l) dist += (zn[l] - zc[l]) * (zn[l] - zc[l]);
        memcpy(zc, zn, sizeof(double) * (size_t)len);
        tc = tn;
        if (sqrt(dist) <= step_tol) break;
    }
    memcpy(z, zc, sizeof(double) * (size_t)len);
    *t = tc;
    free(zc); free(zn);
}

/* s-update, Eq. (13): argmin over S^kappa of (z's - t + v)^2.         */
/* Closed form S:137: theta = t - v; T = kappa largest |z_l| (ties to lowest   */
/* index); Mcap = sum_T |z_l|; s = clamp(theta/Mcap, -1, 1) sgn(z) 1_T.        */
typedef struct { double a; int64_t idx; } orc_key;
static int cmp_key(const void* a, const void* b) {
    const orc_key* x = (const orc_key*)a; const orc_key* y = (const orc_key*)b;
    if (x->a > y->a) return -1;
    if (x->a < y->a) return 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);
}

static orc_key* sorted_abs(int64_t len, const double* z) {
    orc_key* k = (orc_key*)malloc(sizeof(orc_key) * (size_t)(len + 1));
    for (int64_t l = 0; l < len; ++l) { k[l].a = fabs(z[l]); k[l].idx = l; }
    qsort(k, (size_t)len, sizeof(orc_key), cmp_key);
    return k;
}

void orc_s_update(int64_t len, int64_t kappa, const double* z, double t, double v,
                  double* s, double* mcap_out) {
    int64_t kk = kappa < len ? kappa : len;
    if (kk < 0) kk = 0;
    orc_key* k = sorted_abs(len, z);
    double mcap = 0.0;
    for (int64_t r = 0; r < kk; ++r) mcap += k[r].a;
    for (int64_t l = 0; l < len; ++l) s[l] = 0.0;
    if (mcap > 0.0) {
        double scale = clampd((t - v) / mcap, -1.0, 1.0);
        for (int64_t r = 0; r < kk; ++r) s[k[r].idx] = scale * sgn(z[k[r].idx]);
    }
    if (mcap_out) *mcap_out = mcap;
    free(k);
}

/* ------------------------------------------------------------------------- */
/* Linear algebra of the inner loop (Eq. (24); normal equations DESIGN R17).  */
/* ------------------------------------------------------------------------- */
/* y = A x  (A row-major m x nj, ld lda; x nj x C; y m x C).  P:241-242. */
void orc_gemv(int64_t m, int64_t nj, const double* A, int64_t lda, int C, const double* x, double* y) {
    #pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < m; ++r) {
        for (int c = 0; c < C; ++c) {
            double acc = 0.0;
            for (int64_t l = 0; l < nj; ++l) acc += A[r * lda + l] * x[l * C + c];
            y[r * C + c] = acc;
        }
    }
}

/* y = A^T q  (y nj x C).  Each output is one sequential sum over rows r. */
void orc_gemv_t(int64_t m, int64_t nj, const double* A, int64_t lda, int C, const double* q, double* y) {
    const int64_t chunk = 64;
    const int64_t nchunks = (nj + chunk - 1) / chunk;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t ch = 0; ch < nchunks; ++ch) {
        int64_t l0 = ch * chunk, l1 = l0 + chunk < nj ? l0 + chunk : nj;
        double acc[64 * 16];
        int cc = C <= 16 ? C : 16;
        for (int c0 = 0; c0 < C; c0 += cc) {
            int cw = C - c0 < cc ? C - c0 : cc;
            for (int64_t l = l0; l < l1; ++l) for (int c = 0; c < cw; ++c) acc[(l - l0) * cc + c] = 0.0;
            for (int64_t r = 0; r < m; ++r)
                for (int64_t l = l0; l < l1; ++l)
                    for (int c = 0; c < cw; ++c)
                        acc[(l - l0) * cc + c] += A[r * lda + l] * q[r * C + c0 + c];
            for (int64_t l = l0; l < l1; ++l) for (int c = 0; c < cw; ++c) y[l * C + c0 + c] = acc[(l - l0) * cc + c];
        }
    }
}

/* Block factor (DESIGN R17): F = rho_l A^T A + c I with c = 1/(N gamma) + rho_c,
 * G_ab = sum_r A_ra A_rb (sequential over r), L = chol(F) (Cholesky-Crout,
 * column by column).  L row-major nj x nj, lower triangle (upper zeroed). */
int orc_block_factor(int64_t m, int64_t nj, const double* A, int64_t lda, double rho_l, double c, double* L) {
    double* At = (double*)malloc(sizeof(double) * (size_t)(m * nj + 1)); /* columns of A, contiguous */
    if (!At) return ORC_ERR_NOMEM;
    #pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < nj; ++a)
        for (int64_t r = 0; r < m; ++r) At[a * m + r] = A[r * lda + a];
    /* F (lower triangle) into L */
    #pragma omp parallel for schedule(dynamic, 4)
    for (int64_t a = 0; a < nj; ++a) {
        for (int64_t b = 0; b <= a; ++b) {
            double g = 0.0;
            for (int64_t r = 0; r < m; ++r) g += At[a * m + r] * At[b * m + r];
            L[a * nj + b] = rho_l * g + (a == b ? c : 0.0);
        }
        for (int64_t b = a + 1; b < nj; ++b) L[a * nj + b] = 0.0;
    }
    free(At);
    /* Cholesky-Crout in place on the lower triangle. */
    for (int64_t j = 0; j < nj; ++j) {
        double d = L[j * nj + j];
        for (int64_t k = 0; k < j; ++k) d -= L[j * nj + k] * L[j * nj + k];
        if (!(d > 0.0)) return ORC_ERR_INVALID;
        const double ljj = sqrt(d);
        L[j * nj + j] = ljj;
        #pragma omp parallel for schedule(static)
        for (int64_t i = j + 1; i < nj; ++i) {
            double a = L[i * nj + j];
            for (int64_t k = 0; k < j; ++k) a -= L[i * nj + k] * L[j * nj + k];
            L[i * nj + j] = a / ljj;
        }
    }
    return ORC_OK;
}

/* x = F^{-1} rhs = L^{-T} L^{-1} rhs, column by column (C right-hand sides). */
void orc_chol_solve(int64_t nj, const double* L, int C, const double* rhs, double* x) {
    double* y = (double*)malloc(sizeof(double) * (size_t)(nj + 1));
    for (int c = 0; c < C; ++c) {
        for (int64_t i = 0; i < nj; ++i) {
            double a = rhs[i * C + c];
            for (int64_t k = 0; k < i; ++k) a -= L[i * nj + k] * y[k];
            y[i] = a / L[i * nj + i];
        }
        for (int64_t i = nj - 1; i >= 0; --i) {
            double a = y[i];
            for (int64_t k = i + 1; k < nj; ++k) a -= L[k * nj + i] * x[k * C + c];
            x[i * C + c] = a / L[i * nj + i];
        }
    }
    free(y);
}

/* ------------------------------------------------------------------------- */
/* Driver: Algorithm 1 in the Eq. (7) order (DESIGN R2), with the */
/* node-level Algorithm 2 (Eqs. (22)-(24)) as the x-step.          */
/* ------------------------------------------------------------------------- */
typedef struct {
    int64_t m;
    double* L[64];      /* per block factor */
    double* x;          /* n*C, blocks contiguous by column range */
    double* u;          /* n*C */
    double* p[64];      /* per block m*C: A_ij x_ij from the last sweep */
    double* abar;       /* m*C */
    double* obar;       /* m*C omega-bar */
    double* nu;         /* m*C */
} orc_node;

static int inner_sweep(const orc_problem* pb, const orc_params* pr, orc_node* nd, int i,
                       const double* z, double* q, double* rhs, double* xnew, double* dx2) {
    const int C = pb->C, M = pb->M;
    const int64_t n = pb->n, m = nd->m;
    double dx = 0.0;
    for (int j = 0; j < M; ++j) {
        const int64_t c0 = pb->col_start[j], nj = pb->col_start[j + 1] - c0;
        const double* Aij = pb->A[i] + c0;
        /* Eq. (24) target: q = A_ij x_ij^k + omega_bar^k - abar^k - nu^k */
        for (int64_t r = 0; r < m * C; ++r) q[r] = nd->p[j][r] + nd->obar[r] - nd->abar[r] - nd->nu[r];
        /* normal equations: (rho_l A^T A + c I) x = rho_l A^T q + rho_c (z_j - u_ij) */
        orc_gemv_t(m, nj, Aij, n, C, q, rhs);
        for (int64_t l = 0; l < nj * C; ++l)
            rhs[l] = pr->rho_l * rhs[l] + pr->rho_c * (z[c0 * C + l] - nd->u[c0 * C + l]);
        orc_chol_solve(nj, nd->L[j], C, rhs, xnew);
        for (int64_t l = 0; l < nj * C; ++l) {
            double d = xnew[l] - nd->x[c0 * C + l];
            dx += d * d;
            nd->x[c0 * C + l] = xnew[l];
        }
        /* w = A_ij x_ij */
        orc_gemv(m, nj, Aij, n, C, nd->x + c0 * C, nd->p[j]);
    }
    /* P:244 AllReduce: sum over blocks in ascending j; abar = S / M */
    for (int64_t r = 0; r < m * C; ++r) {
        double S = 0.0;
        for (int j = 0; j < M; ++j) S += nd->p[j][r];
        nd->abar[r] = S / (double)M;
    }
    /* Eq. (22) then Eq. (23), per sample */
    int rc = ORC_OK;
    #pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < m; ++r) {
        double pv[64];
        for (int cc = 0; cc < C; ++cc) pv[cc] = nd->abar[r * C + cc] + nd->nu[r * C + cc];
        int e = orc_prox_omega(pb->loss, C, M, pr->rho_l, pb->b[i][r], pv, nd->obar + r * C);
        if (e) {
            #pragma omp critical
            rc = e;
        }
        for (int cc = 0; cc < C; ++cc) nd->nu[r * C + cc] += nd->abar[r * C + cc] - nd->obar[r * C + cc];
    }
    *dx2 = dx;
    return rc;
}

int orc_run(const orc_problem* pb, const orc_params* pr, const int32_t* schedule, orc_result* res) {
    const int N = pb->N, M = pb->M, C = pb->C;
    const int64_t n = pb->n, len = n * C;
    if (N < 1 || M < 1 || M > 64 || C < 1 || C > 64 || n < 1) return ORC_ERR_DIM;
    if (pb->col_start[0] != 0 || pb->col_start[M] != n) return ORC_ERR_DIM;
    for (int j = 0; j < M; ++j) if (pb->col_start[j + 1] <= pb->col_start[j]) return ORC_ERR_DIM;
    if (!(pr->rho_c > 0 && pr->rho_l > 0 && pr->gamma > 0 && pr->alpha > 0 && pr->alpha <= 1)) return ORC_ERR_INVALID;
    if (pr->kappa < 0 || pr->kappa > len) return ORC_ERR_INVALID;
    if (pb->loss == ORC_SOFTMAX ? C < 2 : C != 1) return ORC_ERR_DIM;
    for (int i = 0; i < N; ++i)
        for (int64_t r = 0; r < pb->m[i]; ++r)
            if (!label_ok(pb->loss, C, pb->b[i][r])) return ORC_ERR_DOMAIN;

    const double rho_b = pr->alpha * pr->rho_c;
    const double cdiag = 1.0 / ((double)N * pr->gamma) + pr->rho_c; /* r_j of P:164 */
    double t0 = orc_now();

    orc_node* nodes = (orc_node*)calloc((size_t)N, sizeof(orc_node));
    int64_t mmax = 0, njmax = 0;
    for (int i = 0; i < N; ++i) if (pb->m[i] > mmax) mmax = pb->m[i];
    for (int j = 0; j < M; ++j) if (pb->col_start[j + 1] - pb->col_start[j] > njmax) njmax = pb->col_start[j + 1] - pb->col_start[j];
    int rc = ORC_OK;
    for (int i = 0; i < N && rc == ORC_OK; ++i) {
        orc_node* nd = &nodes[i];
        nd->m = pb->m[i];
        nd->x = (double*)calloc((size_t)len, sizeof(double));
        nd->u = (double*)calloc((size_t)len, sizeof(double));
        nd->abar = (double*)calloc((size_t)(nd->m * C + 1), sizeof(double));
        nd->obar = (double*)calloc((size_t)(nd->m * C + 1), sizeof(double));
        nd->nu = (double*)calloc((size_t)(nd->m * C + 1), sizeof(double));
        for (int j = 0; j < M; ++j) {
            const int64_t c0 = pb->col_start[j], nj = pb->col_start[j + 1] - c0;
            nd->p[j] = (double*)calloc((size_t)(nd->m * C + 1), sizeof(double));
            nd->L[j] = (double*)malloc(sizeof(double) * (size_t)(nj * nj));
            if (!nd->L[j]) { rc = ORC_ERR_NOMEM; break; }
            rc = orc_block_factor(nd->m, nj, pb->A[i] + c0, n, pr->rho_l, cdiag, nd->L[j]);
            if (rc) break;
        }
    }
    double t_setup = orc_now() - t0, t_inner = 0.0, t_outer = 0.0;

    double* z = (double*)calloc((size_t)len, sizeof(double));
    double* zprev = (double*)calloc((size_t)len, sizeof(double));
    double* s = (double*)calloc((size_t)len, sizeof(double));
    double* wbar = (double*)calloc((size_t)len, sizeof(double));
    double* q = (double*)malloc(sizeof(double) * (size_t)(mmax * C + 1));
    double* rhs = (double*)malloc(sizeof(double) * (size_t)(njmax * C + 1));
    double* xnew = (double*)malloc(sizeof(double) * (size_t)(njmax * C + 1));
    double t = 0.0, v = 0.0;
    int k = 0, converged = 0;

    for (k = 0; k < pr->max_outer && rc == ORC_OK; ++k) {
        double ta = orc_now();
        /* (7a)/(10): x_i = prox(z - u_i), by Algorithm 2 on each node. */
        for (int i = 0; i < N && rc == ORC_OK; ++i) {
            int sweeps = 0;
            int limit = schedule ? schedule[(int64_t)k * N + i] : (pr->inner_fixed > 0 ? pr->inner_fixed : pr->max_inner);
            for (sweeps = 0; sweeps < limit;) {
                double dx2;
                rc = inner_sweep(pb, pr, &nodes[i], i, z, q, rhs, xnew, &dx2);
                ++sweeps;
                if (rc) break;
                if (!schedule && pr->inner_fixed <= 0) {
                    double rn = 0.0;
                    for (int64_t r = 0; r < nodes[i].m * C; ++r) {
                        double d = nodes[i].abar[r] - nodes[i].obar[r];
                        rn += d * d;
                    }
                    if (sqrt(rn) <= pr->eps_inner * sqrt((double)(nodes[i].m * C)) && sqrt(dx2) <= pr->eps_inner) break;
                }
            }
            if (res->inner_counts) res->inner_counts[(int64_t)k * N + i] = sweeps;
        }
        double tb = orc_now();
        t_inner += tb - ta;
        if (rc) break;
        /* "Collect": wbar = (1/N) sum_i (x_i + u_i), ascending i (DESIGN R1) */
        for (int64_t l = 0; l < len; ++l) {
            double acc = 0.0;
            for (int i = 0; i < N; ++i) acc += nodes[i].x[l] + nodes[i].u[l];
            wbar[l] = acc / (double)N;
        }
        memcpy(zprev, z, sizeof(double) * (size_t)len);
        double tau;
        orc_zt_update(len, N, pr->rho_c, rho_b, wbar, s, v, z, &t, &tau);   /* (7b) */
        orc_s_update(len, pr->kappa, z, t, v, s, NULL);                      /* (13) */
        double g = -t;                                                      /* g = z's - t */
        for (int64_t l = 0; l < len; ++l) g += z[l] * s[l];
        v += g;                                                             /* (14), DESIGN R5 */
        for (int i = 0; i < N; ++i)                                         /* (9) */
            for (int64_t l = 0; l < len; ++l) nodes[i].u[l] += nodes[i].x[l] - z[l];
        /* (15): p_r = sum_i ||x_i - z||, d_r = sqrt(N) rho_c ||z - z_prev||, b_r = |g| */
        double p_r = 0.0, dz = 0.0;
        for (int i = 0; i < N; ++i) {
            double a = 0.0;
            for (int64_t l = 0; l < len; ++l) { double d = nodes[i].x[l] - z[l]; a += d * d; }
            p_r += sqrt(a);
        }
        for (int64_t l = 0; l < len; ++l) { double d = z[l] - zprev[l]; dz += d * d; }
        double d_r = sqrt((double)N) * pr->rho_c * sqrt(dz), b_r = fabs(g);
        if (res->trace) {
            double* row = res->trace + (int64_t)k * ORC_TRACE_COLS;
            row[0] = p_r; row[1] = d_r; row[2] = b_r; row[3] = t; row[4] = v; row[5] = tau;
        }
        if (res->z_trace) memcpy(res->z_trace + (int64_t)k * len, z, sizeof(double) * (size_t)len);
        if (res->x_trace)
            for (int i = 0; i < N; ++i) memcpy(res->x_trace + ((int64_t)k * N + i) * len, nodes[i].x, sizeof(double) * (size_t)len);
        t_outer += orc_now() - tb;
        if (res->step_s) res->step_s[k] = orc_now() - ta;
        if (p_r <= pr->eps_p && d_r <= pr->eps_d && b_r <= pr->eps_b) { converged = 1; ++k; break; }
    }

    if (rc == ORC_OK) {
        /* Finalise (DESIGN R19): support = top-kappa of |z| with z_l != 0, sorted. */
        orc_key* ks = sorted_abs(len, z);
        int64_t kk = pr->kappa < len ? pr->kappa : len, T = 0;
        int64_t* sup = (int64_t*)malloc(sizeof(int64_t) * (size_t)(kk + 1));
        for (int64_t r = 0; r < kk; ++r) if (ks[r].a > 0.0) sup[T++] = ks[r].idx;
        free(ks);
        for (int64_t a = 1; a < T; ++a) { /* insertion sort ascending */
            int64_t key = sup[a], b = a - 1;
            while (b >= 0 && sup[b] > key) { sup[b + 1] = sup[b]; --b; }
            sup[b + 1] = key;
        }
        for (int64_t l = 0; l < len; ++l) res->x_final[l] = 0.0;
        if (pr->refit && pb->loss == ORC_LS && T > 0) {
            double* xt = (double*)malloc(sizeof(double) * (size_t)T);
            rc = orc_refit_ls(pb, pr->gamma, T, sup, xt);
            for (int64_t a = 0; a < T; ++a) res->x_final[sup[a]] = xt[a];
            free(xt);
        } else if (pr->refit && (pb->loss == ORC_LOGISTIC || pb->loss == ORC_SOFTMAX) && T > 0) {
            double* xt = (double*)malloc(sizeof(double) * (size_t)T);
            for (int64_t a = 0; a < T; ++a) xt[a] = z[sup[a]];   /* start at z on T */
            rc = pb->loss == ORC_LOGISTIC ? orc_refit_logistic(pb, pr->gamma, T, sup, xt)
                                          : orc_refit_softmax(pb, pr->gamma, T, sup, xt);
            for (int64_t a = 0; a < T; ++a) res->x_final[sup[a]] = xt[a];
            free(xt);
        } else {
            for (int64_t a = 0; a < T; ++a) res->x_final[sup[a]] = z[sup[a]];
        }
        for (int64_t a = 0; a < T; ++a) res->support[a] = sup[a];
        *res->support_len = T;
        free(sup);
        if (rc == ORC_OK) rc = orc_objective(pb, pr->gamma, res->x_final, res->objective);
        memcpy(res->z, z, sizeof(double) * (size_t)len);
        memcpy(res->s, s, sizeof(double) * (size_t)len);
        *res->t = t; *res->v = v;
        for (int i = 0; i < N; ++i) {
            if (res->x) memcpy(res->x + (int64_t)i * len, nodes[i].x, sizeof(double) * (size_t)len);
            if (res->u) memcpy(res->u + (int64_t)i * len, nodes[i].u, sizeof(double) * (size_t)len);
        }
        if (res->nu) {
            int64_t off = 0;
            for (int i = 0; i < N; ++i) {
                memcpy(res->nu + off, nodes[i].nu, sizeof(double) * (size_t)(nodes[i].m * C));
                off += nodes[i].m * C;
            }
        }
        *res->iters = k;
        *res->converged = converged;
    }
    if (res->timings) {
        res->timings[0] = t_setup; res->timings[1] = t_inner; res->timings[2] = t_outer;
        res->timings[3] = orc_now() - t0;
    }
    for (int i = 0; i < N; ++i) {
        orc_node* nd = &nodes[i];
        free(nd->x); free(nd->u); free(nd->abar); free(nd->obar); free(nd->nu);
        for (int j = 0; j < M; ++j) { free(nd->p[j]); free(nd->L[j]); }
    }
    free(nodes); free(z); free(zprev); free(s); free(wbar); free(q); free(rhs); free(xnew);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* Validators.                                                                */
/* ------------------------------------------------------------------------- */
/* Dense SPD solve by plain Cholesky (k x k, row-major, overwritten). */
static int spd_solve(int64_t k, double* F, double* x) {
    for (int64_t j = 0; j < k; ++j) {
        double d = F[j * k + j];
        for (int64_t p = 0; p < j; ++p) d -= F[j * k + p] * F[j * k + p];
        if (!(d > 0.0)) return ORC_ERR_INVALID;
        d = sqrt(d);
        F[j * k + j] = d;
        for (int64_t i = j + 1; i < k; ++i) {
            double a = F[i * k + j];
            for (int64_t p = 0; p < j; ++p) a -= F[i * k + p] * F[j * k + p];
            F[i * k + j] = a / d;
        }
    }
    for (int64_t i = 0; i < k; ++i) {
        double a = x[i];
        for (int64_t p = 0; p < i; ++p) a -= F[i * k + p] * x[p];
        x[i] = a / F[i * k + i];
    }
    for (int64_t i = k - 1; i >= 0; --i) {
        double a = x[i];
        for (int64_t p = i + 1; p < k; ++p) a -= F[p * k + i] * x[p];
        x[i] = a / F[i * k + i];
    }
    return ORC_OK;
}

/* (2 A^T A + c I) x = 2 A^T b + rho_c (z - u), c = 1/(N gamma) + rho_c. */
int orc_prox_direct_ls(int64_t m, int64_t n, const double* A, const double* b, double rho_c,
                       double c, const double* z, const double* u, double* x) {
    double* F = (double*)malloc(sizeof(double) * (size_t)(n * n));
    for (int64_t a = 0; a < n; ++a) {
        for (int64_t bb = 0; bb < n; ++bb) {
            double g = 0.0;
            for (int64_t r = 0; r < m; ++r) g += A[r * n + a] * A[r * n + bb];
            F[a * n + bb] = 2.0 * g + (a == bb ? c : 0.0);
        }
        double h = 0.0;
        for (int64_t r = 0; r < m; ++r) h += A[r * n + a] * b[r];
        x[a] = 2.0 * h + rho_c * (z[a] - u[a]);
    }
    int rc = spd_solve(n, F, x);
    free(F);
    return rc;
}

/* Refit on support T: (2 sum_i A_iT^T A_iT + (1/gamma) I) x_T = 2 sum_i A_iT^T b_i. */
int orc_refit_ls(const orc_problem* pb, double gamma, int64_t k, const int64_t* T, double* x) {
    double* F = (double*)calloc((size_t)(k * k + 1), sizeof(double));
    for (int64_t a = 0; a < k; ++a) {
        x[a] = 0.0;
        for (int64_t bb = 0; bb < k; ++bb) {
            double g = 0.0;
            for (int i = 0; i < pb->N; ++i)
                for (int64_t r = 0; r < pb->m[i]; ++r) g += pb->A[i][r * pb->n + T[a]] * pb->A[i][r * pb->n + T[bb]];
            F[a * k + bb] = 2.0 * g + (a == bb ? 1.0 / gamma : 0.0);
        }
        double h = 0.0;
        for (int i = 0; i < pb->N; ++i)
            for (int64_t r = 0; r < pb->m[i]; ++r) h += pb->A[i][r * pb->n + T[a]] * pb->b[i][r];
        x[a] = 2.0 * h;
    }
    int rc = spd_solve(k, F, x);
    free(F);
    return rc;
}

/* Logistic refit on support T (DESIGN R29): minimise the objective (1) restricted to T,
 *   f(x_T) = sum_i sum_r ln(1 + exp(-b_r (A_iT x_T)_r)) + ||x_T||^2 / (2 gamma),
 * by Newton's method with the exact k x k Hessian sum_i A_iT^T diag(s(1-s)) A_iT + I/gamma
 * (s = sigma(b w)), Cholesky solves, and Armijo backtracking on f (factor 1/2, c = 1e-4) while
 * the predicted decrease -g'd exceeds 1e-12 (1 + |f|) (below that f cannot resolve it).
 * x holds the start on entry (z on T) and the minimiser on exit; stops when the Newton
 * step's max-norm is <= 1e-13 max(1, ||x||_inf) (at most 100 steps). */
static double logistic_refit_f(const orc_problem* pb, double gamma, int64_t k, const int64_t* T, const double* x) {
    double f = 0.0;
    for (int i = 0; i < pb->N; ++i)
        for (int64_t r = 0; r < pb->m[i]; ++r) {
            double w = 0.0;
            for (int64_t a = 0; a < k; ++a) w += pb->A[i][r * pb->n + T[a]] * x[a];
            const double y = -pb->b[i][r] * w;   /* ln(1 + e^y), stable */
            f += y > 0.0 ? y + log1p(exp(-y)) : log1p(exp(y));
        }
    double xx = 0.0;
    for (int64_t a = 0; a < k; ++a) xx += x[a] * x[a];
    return f + xx / (2.0 * gamma);
}

int orc_refit_logistic(const orc_problem* pb, double gamma, int64_t k, const int64_t* T, double* x) {
    if (pb->loss != ORC_LOGISTIC || pb->C != 1) return ORC_ERR_INVALID;
    double* F = (double*)malloc(sizeof(double) * (size_t)(k * k + 1));
    double* g = (double*)malloc(sizeof(double) * (size_t)(k + 1));
    double* d = (double*)malloc(sizeof(double) * (size_t)(k + 1));
    double* xn = (double*)malloc(sizeof(double) * (size_t)(k + 1));
    int rc = ORC_OK;
    double f = logistic_refit_f(pb, gamma, k, T, x);
    for (int it = 0; it < 100 && rc == ORC_OK; ++it) {
        for (int64_t a = 0; a < k; ++a) g[a] = x[a] / gamma;
        for (int64_t a = 0; a < k * k; ++a) F[a] = 0.0;
        for (int64_t a = 0; a < k; ++a) F[a * k + a] = 1.0 / gamma;
        for (int i = 0; i < pb->N; ++i)
            for (int64_t r = 0; r < pb->m[i]; ++r) {
                const double* row = pb->A[i] + r * pb->n;
                double w = 0.0;
                for (int64_t a = 0; a < k; ++a) w += row[T[a]] * x[a];
                const double b = pb->b[i][r];
                const double sp = 1.0 / (1.0 + exp(-b * w));   /* sigma(b w) */
                const double psi = -b * (1.0 - sp);             /* d/dw ln(1 + e^{-b w}) */
                const double dd = sp * (1.0 - sp);              /* d2/dw2 */
                for (int64_t a = 0; a < k; ++a) {
                    g[a] += row[T[a]] * psi;
                    for (int64_t c = 0; c <= a; ++c) F[a * k + c] += row[T[a]] * dd * row[T[c]];
                }
            }
        for (int64_t a = 0; a < k; ++a)
            for (int64_t c = 0; c < a; ++c) F[c * k + a] = F[a * k + c];
        for (int64_t a = 0; a < k; ++a) d[a] = -g[a];
        rc = spd_solve(k, F, d);
        if (rc != ORC_OK) break;
        double gd = 0.0, dmax = 0.0, xmax = 1.0;
        for (int64_t a = 0; a < k; ++a) {
            gd += g[a] * d[a];
            dmax = fmax(dmax, fabs(d[a]));
            xmax = fmax(xmax, fabs(x[a]));
        }
        if (dmax <= 1e-13 * xmax) {   /* converged: take the last (tiny) step */
            for (int64_t a = 0; a < k; ++a) x[a] += d[a];
            break;
        }
        /* Armijo backtracking; once the predicted decrease -g'd is below the objective's
         * resolution the full (locally quadratically convergent) Newton step is taken */
        const int resolve = -gd > 1e-12 * (1.0 + fabs(f));
        double alpha = 1.0, fn = f;
        for (int ls = 0; ls < 60; ++ls, alpha *= 0.5) {
            for (int64_t a = 0; a < k; ++a) xn[a] = x[a] + alpha * d[a];
            fn = logistic_refit_f(pb, gamma, k, T, xn);
            if (!resolve || fn <= f + 1e-4 * alpha * gd) break;
        }
        memcpy(x, xn, sizeof(double) * (size_t)k);
        f = fn;
    }
    free(F); free(g); free(d); free(xn);
    return rc;
}

/* Softmax refit on the entry support T of vec(X) (X in R^{n x C}, entry a = l*C + c;
 * DESIGN R13, R29): the same damped Newton as the logistic refit on
 *   f(x_T) = sum_i sum_r [logsumexp(w_r) - w_{r, y_r}] + ||x_T||^2 / (2 gamma),
 *   w_r[c] = sum_{a in T, c_a = c} A[r][l_a] x_a,
 * gradient g_a = sum_r A[r][l_a] (p_r[c_a] - [y_r = c_a]) + x_a / gamma and exact Hessian
 * H_ab = sum_r A[r][l_a] A[r][l_b] (p_r[c_a] [c_a = c_b] - p_r[c_a] p_r[c_b]) + [a = b] / gamma. */
static void softmax_row(int C, const double* w, double* p) {
    double mx = w[0];
    for (int c = 1; c < C; ++c) if (w[c] > mx) mx = w[c];
    double se = 0.0;
    for (int c = 0; c < C; ++c) { p[c] = exp(w[c] - mx); se += p[c]; }
    for (int c = 0; c < C; ++c) p[c] /= se;
}

static double softmax_refit_f(const orc_problem* pb, double gamma, int64_t k, const int64_t* T, const double* x,
                              double* w) {
    const int C = pb->C;
    double f = 0.0;
    for (int i = 0; i < pb->N; ++i)
        for (int64_t r = 0; r < pb->m[i]; ++r) {
            for (int c = 0; c < C; ++c) w[c] = 0.0;
            for (int64_t a = 0; a < k; ++a) w[T[a] % C] += pb->A[i][r * pb->n + T[a] / C] * x[a];
            f += orc_phi(ORC_SOFTMAX, C, w, pb->b[i][r]);
        }
    double xx = 0.0;
    for (int64_t a = 0; a < k; ++a) xx += x[a] * x[a];
    return f + xx / (2.0 * gamma);
}

int orc_refit_softmax(const orc_problem* pb, double gamma, int64_t k, const int64_t* T, double* x) {
    if (pb->loss != ORC_SOFTMAX || pb->C < 2) return ORC_ERR_INVALID;
    const int C = pb->C;
    double* F = (double*)malloc(sizeof(double) * (size_t)(k * k + 1));
    double* g = (double*)malloc(sizeof(double) * (size_t)(k + 1));
    double* d = (double*)malloc(sizeof(double) * (size_t)(k + 1));
    double* xn = (double*)malloc(sizeof(double) * (size_t)(k + 1));
    double* a_r = (double*)malloc(sizeof(double) * (size_t)(k + 1));
    double w[64], p[64];
    int rc = ORC_OK;
    double f = softmax_refit_f(pb, gamma, k, T, x, w);
    for (int it = 0; it < 100 && rc == ORC_OK; ++it) {
        for (int64_t a = 0; a < k; ++a) g[a] = x[a] / gamma;
        for (int64_t a = 0; a < k * k; ++a) F[a] = 0.0;
        for (int64_t a = 0; a < k; ++a) F[a * k + a] = 1.0 / gamma;
        for (int i = 0; i < pb->N; ++i)
            for (int64_t r = 0; r < pb->m[i]; ++r) {
                for (int c = 0; c < C; ++c) w[c] = 0.0;
                for (int64_t a = 0; a < k; ++a) {
                    a_r[a] = pb->A[i][r * pb->n + T[a] / C];
                    w[T[a] % C] += a_r[a] * x[a];
                }
                softmax_row(C, w, p);
                const int y = (int)pb->b[i][r];
                for (int64_t a = 0; a < k; ++a) {
                    const int ca = (int)(T[a] % C);
                    g[a] += a_r[a] * (p[ca] - (ca == y ? 1.0 : 0.0));
                    for (int64_t bb = 0; bb <= a; ++bb) {
                        const int cb = (int)(T[bb] % C);
                        F[a * k + bb] += a_r[a] * a_r[bb] * (p[ca] * (ca == cb ? 1.0 : 0.0) - p[ca] * p[cb]);
                    }
                }
            }
        for (int64_t a = 0; a < k; ++a)
            for (int64_t c = 0; c < a; ++c) F[c * k + a] = F[a * k + c];
        for (int64_t a = 0; a < k; ++a) d[a] = -g[a];
        rc = spd_solve(k, F, d);
        if (rc != ORC_OK) break;
        double gd = 0.0, dmax = 0.0, xmax = 1.0;
        for (int64_t a = 0; a < k; ++a) {
            gd += g[a] * d[a];
            dmax = fmax(dmax, fabs(d[a]));
            xmax = fmax(xmax, fabs(x[a]));
        }
        if (dmax <= 1e-13 * xmax) {
            for (int64_t a = 0; a < k; ++a) x[a] += d[a];
            break;
        }
        const int resolve = -gd > 1e-12 * (1.0 + fabs(f));   /* as in the logistic refit */
        double alpha = 1.0, fn = f;
        for (int ls = 0; ls < 60; ++ls, alpha *= 0.5) {
            for (int64_t a = 0; a < k; ++a) xn[a] = x[a] + alpha * d[a];
            fn = softmax_refit_f(pb, gamma, k, T, xn, w);
            if (!resolve || fn <= f + 1e-4 * alpha * gd) break;
        }
        memcpy(x, xn, sizeof(double) * (size_t)k);
        f = fn;
    }
    free(F); free(g); free(d); free(xn); free(a_r);
    return rc;
}

/* dense ridge = refit on the full index set. */
int orc_ridge_dense(const orc_problem* pb, double gamma, double* x) {
    int64_t* T = (int64_t*)malloc(sizeof(int64_t) * (size_t)pb->n);
    for (int64_t l = 0; l < pb->n; ++l) T[l] = l;
    int rc = orc_refit_ls(pb, gamma, pb->n, T, x);
    free(T);
    return rc;
}

/* S:413-421 best subset: enumerate all supports of size <= kappa (ascending size,
 * lexicographic within a size), restricted ridge on pooled moments
 * G = sum A_i^T A_i, h = sum A_i^T b_i, bb = sum ||b_i||^2.
 * Objective at the restricted optimum: bb - h_T^T x_T (since (2G_TT + I/gamma) x_T = 2 h_T). */
int orc_best_subset(const orc_problem* pb, double gamma, int64_t kappa,
                    int64_t* support, int64_t* support_len, double* x, double* objective) {
    const int64_t n = pb->n;
    if (pb->loss != ORC_LS || pb->C != 1) return ORC_ERR_INVALID;
    if (n > 64 || kappa > 8) return ORC_ERR_INVALID;
    double* G = (double*)calloc((size_t)(n * n), sizeof(double));
    double* h = (double*)calloc((size_t)n, sizeof(double));
    double bb = 0.0;
    for (int i = 0; i < pb->N; ++i)
        for (int64_t r = 0; r < pb->m[i]; ++r) {
            const double* a = pb->A[i] + r * n;
            for (int64_t p = 0; p < n; ++p) {
                h[p] += a[p] * pb->b[i][r];
                for (int64_t q2 = 0; q2 < n; ++q2) G[p * n + q2] += a[p] * a[q2];
            }
            bb += pb->b[i][r] * pb->b[i][r];
        }
    double best = bb;                 /* empty support */
    int64_t best_T[8], best_k = 0;
    double best_x[8];
    int64_t T[8];
    double F[64], xs[8];
    for (int64_t k = 1; k <= kappa && k <= n; ++k) {
        for (int64_t a = 0; a < k; ++a) T[a] = a;
        for (;;) {
            for (int64_t a = 0; a < k; ++a) {
                for (int64_t b2 = 0; b2 < k; ++b2) F[a * k + b2] = 2.0 * G[T[a] * n + T[b2]] + (a == b2 ? 1.0 / gamma : 0.0);
                xs[a] = 2.0 * h[T[a]];
            }
            if (spd_solve(k, F, xs) == ORC_OK) {
                double obj = bb;
                for (int64_t a = 0; a < k; ++a) obj -= h[T[a]] * xs[a];
                if (obj < best) {
                    best = obj; best_k = k;
                    for (int64_t a = 0; a < k; ++a) { best_T[a] = T[a]; best_x[a] = xs[a]; }
                }
            }
            int64_t p = k - 1;
            while (p >= 0 && T[p] == n - k + p) --p;
            if (p < 0) break;
            ++T[p];
            for (int64_t a = p + 1; a < k; ++a) T[a] = T[a - 1] + 1;
        }
    }
    for (int64_t l = 0; l < n; ++l) x[l] = 0.0;
    for (int64_t a = 0; a < best_k; ++a) { support[a] = best_T[a]; x[best_T[a]] = best_x[a]; }
    *support_len = best_k;
    *objective = best;
    free(G); free(h);
    return ORC_OK;
}
