/*
 * bicadmm.h -- C ABI of the B200-native Bi-cADMM hot path (arXiv 2405.16267).
 *
 * One library, libbicadmm.so, hand-written CUDA for sm_100a.  Plain pointers and
 * sizes only; no torch types.  Citation keys: P:n = PAPER.md line n (Section /
 * Equation / Algorithm given beside it), S:n = SPEC.md line n, "DESIGN Rk" =
 * reading k in DESIGN.md section 4 (where the paper is silent or garbled).
 *
 * The problem (Problem (1)):
 *     min_x  sum_i l_i(A_i x - b_i) + (1/(2 gamma)) ||x||_2^2   s.t. ||x||_0 <= kappa
 * solved by Bi-cADMM: the outer bilinear-consensus iteration (Eqs. (7a)-(7e), (9),
 * (13), (14), (15); Algorithm 1) around the node-level sharing-ADMM
 * sub-solver over feature blocks A_ij (Eqs. (16)-(24); Algorithm 2).
 *
 * MEMORY AND OWNERSHIP
 *   - A_ij and b_i are DEVICE memory BORROWED from the caller; never written; must
 *     outlive the handle.  A_ij is row-major: element (r, l) of block (i, j),
 *     0 <= r < m_i, 0 <= l < n_j = col_start[j+1] - col_start[j], lives at
 *     A[r * lda + l].  The element type is the problem dtype (double or float).
 *     Alignment: the A pointer must be 16-byte aligned and lda a multiple of
 *     4 elements (128-bit vector loads); else BICADMM_ERR_INVALID.
 *   - The workspace is DEVICE memory provided by the caller (e.g. a torch
 *     tensor), at least bicadmm_workspace_size() bytes, 256-byte aligned.  The
 *     library performs no cudaMalloc of device memory.  It holds the cached
 *     block factors H_ij = (rho_l A_ij^T A_ij + c I)^-1, c = 1/(N gamma) + rho_c
 *     (DESIGN R17), all iterates (FP64) and scratch.
 *   - All work is enqueued on the caller's CUDA stream (cudaStream_t passed as
 *     void*; NULL = legacy default stream).  bicadmm_iterate / bicadmm_solve
 *     synchronise that stream once per outer iteration to read 6 scalars.
 *   - Handles are used by one host thread at a time; distinct handles are
 *     independent.
 *
 * ERRORS
 *   Every call returns a bicadmm_rc; nothing throws or aborts across the ABI.
 *   Non-convergence is not an error (report.converged = 0).  After a
 *   CUDA or NCCL failure the handle accepts only bicadmm_destroy and
 *   bicadmm_last_error.
 */
#ifndef BICADMM_H
#define BICADMM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BICADMM_ABI_VERSION 1

typedef enum {
    BICADMM_OK = 0,
    BICADMM_ERR_INVALID = -1,   /* bad parameter: kappa outside [0, n*C], penalty <= 0, alpha outside (0,1],
                                   tolerance < 0, alignment, NULL pointer */
    BICADMM_ERR_DIM = -2,       /* length/shape mismatch */
    BICADMM_ERR_DOMAIN = -3,    /* label outside {-1,+1} (logistic/hinge) or [0,C) (softmax) */
    BICADMM_ERR_PLACEMENT = -4, /* local blocks not a valid placement (duplicate, missing node labels) */
    BICADMM_ERR_OOM = -5,       /* workspace smaller than bicadmm_workspace_size() */
    BICADMM_ERR_CUDA = -6,      /* CUDA runtime failure; handle is dead */
    BICADMM_ERR_NCCL = -7,      /* NCCL failure; handle is dead */
    BICADMM_ERR_STATE = -8      /* call not valid in the handle's state */
} bicadmm_rc;

/* Loss l_i (LS without 1/2 per P:259; DESIGN R12): per sample phi(w, b):
 *   LS (w-b)^2, LOGISTIC ln(1+e^{-bw}) b in {-1,+1}, HINGE max(0, 1-bw) b in {-1,+1},
 *   SOFTMAX logsumexp(w) - w_b, w in R^C, b a class id in [0, C) stored as a number. */
typedef enum { BICADMM_LS = 0, BICADMM_LOGISTIC = 1, BICADMM_SOFTMAX = 2, BICADMM_HINGE = 3 } bicadmm_loss;

/* Storage type of A_ij, b_i and H_ij.  Iterates and all reductions are FP64 in both
 * modes (DESIGN R23). */
typedef enum { BICADMM_F64 = 0, BICADMM_F32 = 1 } bicadmm_dtype;

/* One feature block A_ij resident on this rank (Eq. (17)). */
typedef struct {
    int32_t node;       /* i in [0, N) */
    int32_t block;      /* j in [0, M) */
    const void* A;      /* device pointer, see MEMORY above */
    int64_t lda;        /* row stride in elements, >= n_j, multiple of 4 */
    void* ready_event;  /* optional cudaEvent_t (NULL = A and b_i already written): recorded by the
                           caller after A_ij and the labels b_i were written on another stream.
                           bicadmm_setup makes its stream wait on it right before the first read
                           of this block (its Gram, a0), so host->device copies of later blocks
                           overlap the factorisation of earlier ones; every such wait precedes the
                           return of bicadmm_setup in stream order.  Not retained after setup. */
} bicadmm_block;

/* bicadmm_setup(A, b, loss, ...) of the north star: the data half. */
typedef struct {
    int32_t N;                   /* nodes (sample shards) */
    int32_t M;                   /* feature blocks per node */
    int32_t C;                   /* classes: 1, or >= 2 for SOFTMAX (DESIGN R13) */
    int32_t loss;                /* bicadmm_loss */
    int32_t dtype;               /* bicadmm_dtype */
    int32_t n_blocks;            /* number of entries in blocks[] (blocks on this rank) */
    int64_t n;                   /* features */
    const int64_t* m;            /* host [N]: m_i rows of node i */
    const int64_t* col_start;    /* host [M+1]: block j owns columns [col_start[j], col_start[j+1]),
                                    col_start[0] = 0, col_start[M] = n, strictly increasing,
                                    every col_start[j] a multiple of 4 (DESIGN R16) */
    const bicadmm_block* blocks; /* host [n_blocks]; (node, block) pairs distinct */
    const void* const* b;        /* host [N]: device pointer to labels of node i (m_i entries, dtype);
                                    may be NULL for a node with no local block */
} bicadmm_problem;

/* bicadmm_setup(..., kappa, rho, lambda) of the north star: the parameter half. */
typedef struct {
    int64_t kappa;        /* sparsity budget, 0 <= kappa <= n*C */
    double rho_c;         /* consensus penalty rho_c > 0 */
    double alpha;         /* rho_b = alpha * rho_c, alpha in (0, 1] */
    double rho_l;         /* inner sharing penalty rho_l > 0 (DESIGN R8) */
    double lambda;        /* ridge weight 1/gamma > 0 of (1/(2 gamma))||x||^2 (DESIGN R24) */
    double eps_p, eps_d, eps_b;  /* absolute tolerances on p_r, d_r, b_r (Eq. (15)) */
    int32_t max_outer;    /* cap on outer iterations for bicadmm_solve */
    int32_t inner_fixed;  /* > 0: exactly this many inner sweeps per outer iteration;
                             0: tolerance mode (eps_inner, max_inner), DESIGN R7 */
    double eps_inner;     /* tol mode: stop node i when ||abar-obar|| <= eps_inner sqrt(m_i C)
                             and ||x_i^new - x_i^old|| <= eps_inner */
    int32_t max_inner;    /* tol mode cap */
    int32_t refit;        /* refit on the final support: LS closed-form ridge (DESIGN R19), logistic and softmax
                             damped Newton (DESIGN R29; multi-rank: node sums over the ranks); hinge: x_final = z on T */
    int32_t sweep;        /* inner-sweep schedule: 0 = auto (the fastest measured: the CTA-pair single-pass
                             kernel for tall single-block nodes with C == 1 and rows >= 5.5 KB; else, on a
                             single rank with C == 1 and nodes whose blocks and factors fit one CTA's
                             shared memory, whole inner loops in one CTA per node (kind 5); else
                             two-pass; BICADMM_FIELD_SWEEP_KIND reports the choice),
                             1 = two-pass (A streamed by GEMV-T then by GEMV, paper-literal order),
                             2 = fused single HBM pass (needs every node's blocks on this rank,
                             C == 1, tall blocks of an even width up to 13,432 (FP64) / 13,824 (FP32)
                             columns and 16-byte row pitches, else
                             BICADMM_ERR_INVALID).  Same algebra (Eqs. (22)-(24));
                             results agree to rounding. */
} bicadmm_params;

/* Result of bicadmm_iterate: the last outer iteration's Eq. (15) residuals. */
typedef struct {
    int32_t outer_iters;   /* total outer iterations done so far */
    int32_t inner_sweeps;  /* inner sweeps done by this call (max over local nodes) */
    double p_r, d_r, b_r;  /* Eq. (15) */
    double t, v, tau;      /* consensus l1 bound t, scaled bilinear multiplier v, (7b) root tau */
    int32_t converged;     /* all three residuals <= their tolerances */
} bicadmm_step_info;

typedef struct {
    int32_t converged;
    int32_t outer_iters;
    int64_t inner_sweeps;   /* total over the solve (max over nodes per outer iteration) */
    int64_t support_len;    /* |support| <= kappa */
    double objective;       /* Problem (1) at x_final (DESIGN R20) */
    double p_r, d_r, b_r;
    double ms_setup;        /* setup: Gram + factor (device time, CUDA events) */
    double ms_solve;        /* iterations + finalize (device time) */
} bicadmm_report;

/* Fields readable with bicadmm_get (FP64 unless noted; lengths in elements). */
typedef enum {
    BICADMM_FIELD_Z = 0,        /* n*C: consensus z (row-major n x C) */
    BICADMM_FIELD_S = 1,        /* n*C: s in S^kappa */
    BICADMM_FIELD_SCALARS = 2,  /* 6: t, v, tau, p_r, d_r, b_r */
    BICADMM_FIELD_X_LOCAL = 3,  /* per local block in blocks[] order: n_j*C each, concatenated */
    BICADMM_FIELD_U_LOCAL = 4,  /* same layout as X_LOCAL */
    BICADMM_FIELD_SUPPORT = 5,  /* int64 [support_len], ascending (after solve/finalize) */
    BICADMM_FIELD_X_FINAL = 6,  /* n*C (after solve/finalize) */
    BICADMM_FIELD_TRACE = 7,    /* host-side trace: outer_iters rows x 6 (p_r, d_r, b_r, t, v, tau) */
    BICADMM_FIELD_WBAR = 8,     /* n*C: last consensus average */
    BICADMM_FIELD_NU = 9,       /* per local node (ascending node id): m_i*C each, concatenated */
    BICADMM_FIELD_INNER_COUNTS = 10, /* int32 [outer_iters x N] inner sweeps per (outer, node) */
    BICADMM_FIELD_LAUNCHES = 11, /* int64 [1]: kernels this handle has launched so far */
    BICADMM_FIELD_PHASE_MS = 12, /* double [BICADMM_NPHASE]: device time per phase accumulated while
                                    profiling is on (CUDA events on the handle's stream) */
    BICADMM_FIELD_PHASE_COUNT = 13, /* int64 [BICADMM_NPHASE]: kernel launches per phase while profiling */
    BICADMM_FIELD_SWEEP_KIND = 14, /* int32 [2]: inner-sweep implementation chosen at setup (0 two-pass,
                                     4 the CTA-pair single-pass kernel k_fused4, 5 small nodes' inner
                                     loops in one CTA each) and the number of local Woodbury (fat) blocks */
    BICADMM_FIELD_P_LOCAL = 15,  /* per local block in blocks[] order: p_ij = A_ij x_ij of the last sweep
                                    (m_i*C each, concatenated; property checks at full size) */
    BICADMM_FIELD_R_LOCAL = 16   /* per local block: r_ij = rho_l A_ij^T q + rho_c (z_j - u_ij) of the last
                                    sweep (n_j*C each; x_ij = H_ij r_ij; tall blocks only) */
} bicadmm_field;

/* Phases timed by bicadmm_set_profiling:
 *   0 GEMV-T partial pass over A_ij (a1+a2, the first HBM pass)   1 GEMV-T chunk reduce + Eq. (24) epilogue
 *   2 x = H r (a3)   3 p = A x (a4, the second HBM pass)   4 block sum + AllReduce (a5)
 *   5 prox + nu + delta (a6, a7)   6 global step: Collect, (7b), (13), (14), (9), (15) (a8-a12)
 *   7 fused single-pass sweep (a4 + a5 + a6 + a7 + the next sweep's a1/a2 partial products) */
#define BICADMM_NPHASE 8

typedef struct bicadmm_comm bicadmm_comm;
typedef struct bicadmm_handle bicadmm_handle;

int bicadmm_version(void);
const char* bicadmm_rc_string(int rc);

/* ---- multi-GPU plumbing (NCCL over NVLink) ----
 * Rank 0 calls bicadmm_get_unique_id and the caller broadcasts the
 * bicadmm_uid_size() bytes (e.g. torch.distributed); every rank then calls
 * bicadmm_comm_init.  group_color: ranks holding blocks of the same node set
 * share a color; the per-sweep m-vector AllReduce (Algorithm 2) runs over
 * that group, the per-outer n-vector AllReduce ("Collect") over all ranks.
 * NCCL is loaded at run time (libnccl.so.2); world == 1 needs no NCCL and a NULL
 * comm passed to bicadmm_setup means a single rank.  NCCL_ALGO / NCCL_PROTO are pinned
 * to Ring / Simple unless the caller set them (run-to-run identical reduction order).
 * bicadmm_setup on more than one rank is collective: it checks that every (node, block)
 * pair is held by exactly one rank and that each node group holds all blocks of its
 * nodes (else BICADMM_ERR_PLACEMENT on every rank). */
int bicadmm_uid_size(void);
int bicadmm_get_unique_id(void* uid_out);
int bicadmm_comm_init(int world, int rank, int device, const void* uid, int group_color, bicadmm_comm** out);
int bicadmm_comm_destroy(bicadmm_comm* comm);

/* ---- in-process emulated communicator (validation of the multi-rank path on one GPU) ----
 * G "ranks" as G handles of ONE process on one device, each driven by its own host thread
 * and its own stream: bicadmm_emu_group_create(G), then bicadmm_comm_init_emu for every
 * rank 0..G-1 (all before any bicadmm_setup), then each thread runs bicadmm_setup /
 * _iterate / _solve / _finalize on its handle concurrently, exactly as G processes would.
 * Every AllReduce of the method (Algorithm 2's per-sweep block sum; the outer
 * Collect) becomes a fixed-order device sum over the members' buffers (ascending
 * rank), ordered across the members' streams by CUDA events; the threads meet at host
 * barriers.  No kernel waits on another, so the ranks never need to run concurrently on
 * the device.  The group owns a scratch buffer per rank (cudaMalloc, freed by
 * bicadmm_emu_group_destroy, which must follow every bicadmm_comm_destroy of the group).
 * Errors: BICADMM_ERR_INVALID (G outside [1, 64], rank out of range or registered twice). */
typedef struct bicadmm_emu_group bicadmm_emu_group;
int bicadmm_emu_group_create(int world, bicadmm_emu_group** out);
int bicadmm_comm_init_emu(bicadmm_emu_group* group, int rank, int device, int group_color, bicadmm_comm** out);
int bicadmm_emu_group_destroy(bicadmm_emu_group* group);

/* Bytes of device workspace needed for this problem on this rank. */
int bicadmm_workspace_size(const bicadmm_problem* problem, const bicadmm_params* params, size_t* bytes);

/* Validate, register the borrowed blocks, zero all state (DESIGN R10) and build
 * every local factor H_ij (one-time; Eq. (24) normal equations).  stream is a
 * cudaStream_t.  The device current on the calling thread must own the pointers. */
int bicadmm_setup(const bicadmm_problem* problem, const bicadmm_params* params, bicadmm_comm* comm,
                  void* workspace, size_t workspace_bytes, void* stream, bicadmm_handle** out);

/* Run n_outer outer iterations of Eq. (7) order: inner sweeps (Algorithm 2),
 * Collect + (7b) + (13) + (14) + (9) + (15).  Fills *info (may be NULL). */
int bicadmm_iterate(bicadmm_handle* h, int n_outer, bicadmm_step_info* info);

/* Iterate until p_r <= eps_p, d_r <= eps_d, b_r <= eps_b or max_outer outer
 * iterations in total, then finalize (support, x_final, objective). */
int bicadmm_solve(bicadmm_handle* h, bicadmm_report* report);

/* Finalize now (support = top-kappa of |z| with z != 0; x_final; objective). */
int bicadmm_finalize(bicadmm_handle* h, bicadmm_report* report);

/* Replay per-(outer, node) inner sweep counts (row-major [n_rows x N]) instead of
 * the fixed/tol rule, starting at the next outer iteration (DESIGN R7). */
int bicadmm_set_schedule(bicadmm_handle* h, const int32_t* counts, int n_rows);

/* Copy a field to dst (device memory if on_device, else host). bytes must equal
 * the field's size exactly (BICADMM_ERR_DIM otherwise); query with dst = NULL,
 * which stores the size in *bytes_out. */
int bicadmm_get(bicadmm_handle* h, int field, void* dst, size_t bytes, int on_device, size_t* bytes_out);

/* Per-phase device timing with CUDA events (on = 1) for roofline reporting; resets
 * the accumulators.  Adds two events per phase per sweep, no host syncs. */
int bicadmm_set_profiling(bicadmm_handle* h, int on);

const char* bicadmm_last_error(const bicadmm_handle* h);
int bicadmm_destroy(bicadmm_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* BICADMM_H */
