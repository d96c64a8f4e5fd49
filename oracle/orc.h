/*
 * orc.h -- declarations of the FP64 CPU ORACLE for Bi-cADMM (arXiv 2405.16267).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load liborc.so.  The product path
 * (paper_2405_16267_b200/, include/) never includes, links or calls anything here,
 * and this tree never includes anything from the product path.
 *
 * Citation keys: P:n = reference PAPER.md line n; S:n = reference SPEC.md line n;
 * "DESIGN R<k>" = reading k listed in DESIGN.md section "Readings of the paper".
 *
 * Conventions (shared with the product only through DESIGN.md, never through code):
 *   - A_i is row-major m_i x n with leading dimension n (oracle keeps lda = n).
 *   - x, z, s, u are n*C vectors laid out as X[l*C + c] (row-major n x C).
 *   - p, omega_bar, nu, S are m_i*C vectors laid out as W[r*C + c].
 *   - labels b: LS real; logistic/hinge +-1; softmax class id in [0,C) stored as double.
 *   - feature blocks: contiguous column ranges [col_start[j], col_start[j+1]).
 */
#ifndef ORC_H
#define ORC_H
#include <stdint.h>

enum { ORC_LS = 0, ORC_LOGISTIC = 1, ORC_SOFTMAX = 2, ORC_HINGE = 3 };
enum { ORC_OK = 0, ORC_ERR_INVALID = -1, ORC_ERR_DIM = -2, ORC_ERR_DOMAIN = -3,
       ORC_ERR_INFEASIBLE = -4, ORC_ERR_NOMEM = -5 };

typedef struct {
    int32_t N, M, C, loss;
    int64_t n;
    const int64_t* m;          /* [N] rows per node */
    const double* const* A;    /* [N] row-major m_i x n */
    const double* const* b;    /* [N] labels, m_i entries */
    const int64_t* col_start;  /* [M+1] block boundaries */
} orc_problem;

typedef struct {
    int64_t kappa;
    double rho_c, alpha, rho_l, gamma;
    double eps_p, eps_d, eps_b;
    int32_t max_outer;
    int32_t inner_fixed;       /* > 0: exactly this many sweeps per outer iteration */
    double eps_inner;          /* tol mode (inner_fixed == 0) */
    int32_t max_inner;
    int32_t refit;             /* LS only: ridge refit on the support */
} orc_params;

typedef struct {
    double* z;            /* [n*C] final consensus */
    double* s;            /* [n*C] */
    double* t;            /* [1] */
    double* v;            /* [1] */
    double* x;            /* [N][n*C] final node estimates x_i */
    double* u;            /* [N][n*C] */
    double* trace;        /* [max_outer][ORC_TRACE_COLS] or NULL */
    int32_t* inner_counts;/* [max_outer][N] or NULL */
    double* z_trace;      /* [max_outer][n*C] or NULL */
    double* x_trace;      /* [max_outer][N][n*C] or NULL */
    int64_t* support;     /* [kappa] */
    int64_t* support_len; /* [1] */
    double* x_final;      /* [n*C] */
    double* objective;    /* [1] objective (1) at x_final */
    int32_t* iters;       /* [1] */
    int32_t* converged;   /* [1] */
    double* timings;      /* [4]: setup_s, inner_s, outer_s, total_s (wall) or NULL */
    double* nu;           /* [sum_i m_i*C] final inner duals nu_i (Eq. (23)), nodes concatenated, or NULL */
    double* step_s;       /* [max_outer] wall seconds of each outer iteration (inner + global step) or NULL;
                             timing only (bench.py's reference arm times exactly K steps after W) */
} orc_result;

#define ORC_TRACE_COLS 6  /* p_r, d_r, b_r, t, v, tau */

/* ---- losses / objective ---- */
double orc_phi(int loss, int C, const double* w, double b);
int    orc_loss_value(int loss, int C, int64_t m, const double* w, const double* b, double* out);
int    orc_objective(const orc_problem* pb, double gamma, const double* x, double* out);
int64_t orc_kappa_from_sparsity(int64_t n, double s_l);

/* ---- Theorem 1 geometry ---- */
int orc_l0_witness(int64_t n, const double* x, int64_t kappa, double* s, double* t);
int orc_check_theorem1(int64_t n, const double* x, const double* s, double t, double kappa, double tol);
void orc_proj_l1_epigraph(int64_t n, const double* z, double t, double* z_out, double* t_out);

/* ---- per-sample prox (22) ---- */
int orc_prox_omega(int loss, int C, int M, double rho_l, double b, const double* p, double* omega);

/* ---- global step (7b), (13), (14) ---- */
void orc_zt_update(int64_t len, int N, double rho_c, double rho_b, const double* wbar,
                   const double* s, double v, double* z, double* t, double* tau);
void orc_s_update(int64_t len, int64_t kappa, const double* z, double t, double v,
                  double* s, double* mcap);
void orc_zt_pgd(int64_t len, int N, double rho_c, double rho_b, const double* wbar,
                const double* s, double v, double step_tol, int max_steps, double* z, double* t);

/* ---- linear algebra used by the inner loop ---- */
void orc_gemv(int64_t m, int64_t nj, const double* A, int64_t lda, int C, const double* x, double* y);
void orc_gemv_t(int64_t m, int64_t nj, const double* A, int64_t lda, int C, const double* q, double* y);
int  orc_block_factor(int64_t m, int64_t nj, const double* A, int64_t lda, double rho_l, double c, double* L);
void orc_chol_solve(int64_t nj, const double* L, int C, const double* rhs, double* x);

/* ---- driver (Algorithm 1 with Algorithm 2 inside; Eq. (7) order) ---- */
int orc_run(const orc_problem* pb, const orc_params* pr, const int32_t* schedule, orc_result* res);

/* ---- validators ---- */
int orc_prox_direct_ls(int64_t m, int64_t n, const double* A, const double* b, double rho_c,
                       double c, const double* z, const double* u, double* x);
int orc_ridge_dense(const orc_problem* pb, double gamma, double* x);
int orc_refit_ls(const orc_problem* pb, double gamma, int64_t k, const int64_t* T, double* x);
/* Logistic refit on T by damped Newton (DESIGN R29); x: start (z on T) in, minimiser out. */
int orc_refit_logistic(const orc_problem* pb, double gamma, int64_t k, const int64_t* T, double* x);
/* Softmax refit on the entry support T of vec(X) (DESIGN R29), same damped Newton. */
int orc_refit_softmax(const orc_problem* pb, double gamma, int64_t k, const int64_t* T, double* x);
int orc_best_subset(const orc_problem* pb, double gamma, int64_t kappa,
                    int64_t* support, int64_t* support_len, double* x, double* objective);

#endif
