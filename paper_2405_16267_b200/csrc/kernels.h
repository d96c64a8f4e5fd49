// kernels.h -- private launcher declarations of libbicadmm (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

namespace bic {

// ---------------------------------------------------------------- GEMV family
// y[r] = sum_l A[r, l] x[l]   ("Compute A_ij x_ij"; also x = H r, a3)
struct GemvDesc {
    const void* A;
    int64_t lda, rows, cols;
    const double* x;
    double* y;
    int64_t task_begin;  // filled by the launcher
    double* xt = nullptr;   // C > 1: scratch (cols * C) for the class-major copy of x
    double alpha = 1.0;     // y = alpha * (A x)
};
int launch_gemv(int dtype, GemvDesc* d, int nd, int grid_cap, cudaStream_t s, int C = 1);

// Packed symmetric H-apply (k_symv.cu): y = alpha * H x, H stored as lower 64x64 tiles.
struct SymvDesc {
    const void* H;      // symv_packed_elems(n) elements of the data dtype
    int64_t n;
    const double* x;
    double* y;
    double alpha = 1.0;
    double* part;       // symv_part_doubles(n) scratch
};
int64_t symv_packed_elems(int64_t n);
int64_t symv_part_doubles(int64_t n);
int launch_symv_packed(int dtype, const SymvDesc* d, int nd, cudaStream_t s);
int launch_symv_pack(int dtype, int64_t n, const double* G, int64_t ldg, void* Hp, cudaStream_t s);
int launch_gemv_c(int dtype, int C, GemvDesc* d, int nd, cudaStream_t s);
// DMMA (FP64 tensor pipe) variants for C > 1 (k_gemv_dmma.cu); BICADMM_GEMVC_DMMA=0 selects
// the scalar-FMA kernels of k_gemv_c.cu
bool gemv_c_dmma_enabled();
int launch_gemv_c_dmma(int dtype, int C, GemvDesc* d, int nd, cudaStream_t s);
int gemv_grid_cap(int dtype, int sm_count);  // persistent grid size (resident CTAs)

// r[l] = rho_l * sum_r A[r, l] (p[r] + delta[r]) + rho_c (z[l] - u[l])   (Eq. (24))
struct GemvTDesc {
    const void* A;
    int64_t lda, rows, cols;
    const double* p;      // A_ij x_ij from the previous sweep
    const double* delta;  // omega_bar - abar - nu of the node (may be null)
    const double* z;      // z_j (may be null)
    const double* u;      // u_ij (may be null)
    double* r;            // output
    double* partial;      // [nchunks][cols] scratch
    int64_t chunk_rows;
    int32_t nchunks, nstrips;
    int64_t cta_begin;    // filled by the launcher
};
// Choose chunk_rows / nchunks for a batch so the grid fills the GPU; returns
// scratch doubles needed by descriptor k in need[k].
void plan_gemv_t(int dtype, GemvTDesc* d, int nd, int sm_count, int64_t* need, int C = 1);
int launch_gemv_t(int dtype, GemvTDesc* d, int nd, double rho_l, double rho_c, cudaStream_t s,
                  cudaEvent_t mid = nullptr, int C = 1);
int launch_gemv_t_c_partial(int dtype, int C, GemvTDesc* d, int nd, cudaStream_t s);
int launch_gemv_t_c_dmma(int dtype, int C, GemvTDesc* d, int nd, cudaStream_t s);
int launch_gemv_t_reduce(GemvTDesc* d, int nd, double rho_l, double rho_c, cudaStream_t s, int C = 1);
int gemv_t_c_strip_width(int dtype);
int gemv_t_strip_width(int dtype);

// ---------------------------------------------------------------- prox (Eqs. (22), (23))
struct ProxNode {
    const void* b;        // labels (dtype)
    const double* p;      // local block products, np blocks x pstride
    const double* S;      // if non-null: the (all-reduced) block sum, used instead of p
    double* nu;
    double* delta;
    double* omega;        // optional output
    double* sq_partial;   // optional: per-CTA partial of ||abar - omega||^2 (tol mode)
    int64_t m, pstride;
    int32_t np;
    int64_t cta_begin;    // filled by the launcher
};
int launch_prox(int loss, int dtype, int C, int M, double rho_l, ProxNode* nodes, int nn, cudaStream_t s);

// Small nodes (k_prox.cu): K whole sweeps of a node in one CTA, A_ij and H_ij staged in shared
// memory (C == 1, tall blocks, every block of the node local).
constexpr int kSmallMaxBlocks = 8;
constexpr int kSmallMaxCols = 256;   // threads of k_small_sweeps: a node's columns fit one pass of them
constexpr size_t kSmallSmemMax = 220 * 1024;
struct SmallBlock {
    const void* A;       // A_ij (dtype), row stride lda
    int64_t lda, nj;
    int64_t c0;          // first column of the block in the n-vector (z)
    int64_t cs;          // first column of the block in the node's staged matrix
    const void* H;       // H_ij (dtype): packed lower 64 x 64 tiles (hpack) or nj x ldh
    int64_t ldh;
    int hpack;
    double *x, *r, *p;   // x_ij, r_ij (nj), p_ij (m)
    const double* u;     // u_ij (nj)
};
struct SmallNode {
    const void* b;
    double *nu, *delta, *omega;
    int64_t m, ncols;
    int nb;
    int nsplit, nsplit_m;   // inner-length splits of the column / row products (small_sweep_plan)
    SmallBlock blk[kSmallMaxBlocks];
};
void small_sweep_plan(SmallNode& N);
size_t small_sweep_smem_bytes(const SmallNode& N);
int launch_small_sweeps(int loss, int dtype, const SmallNode* nodes, int nn, const double* z, int K, int M,
                        double rho_l, double rho_c, cudaStream_t s);
int launch_psum(int C, ProxNode* nodes, int nn, double* const* S_out, cudaStream_t s);
constexpr int kProxThreads = 256;
// Per-CTA partials of sum_r phi((sum_j p_j)[r], b_r) for the objective (DESIGN R20).
int launch_loss(int loss, int dtype, int C, ProxNode* nodes, int nn, cudaStream_t s);

// ---------------------------------------------------------------- dense factor (a0)
// F = alpha A^T A + diag I (lower triangle or full) into FP64 G (ldg).
// FP64-accurate Gram on tcgen05 kind::i8 (Ozaki slices, k_gram_tc.cu): lower triangle of
// alpha A^T A + diag I into G (FP64, ldg); scratch of gram_tc_scratch_bytes() (slices + scales)
size_t gram_tc_scratch_bytes(int dtype, int64_t m, int64_t nj);
// General FP64-accurate product on the same engine: C = alpha A_op B_op + beta C (+ diag I),
// A_op(i, k) = A[i a_sl + k a_sr] (M x K), B_op(k, j) = B[j b_sl + k b_sr] (K x N), FP64 C.
// k_lo / k_hi: structural zeros skipped per tile (exact): k_lo 1: A_op(i, k) = 0 for k < i,
// 2: B_op(k, j) = 0 for k < j, 3: both (k >= max(i, j)); k_hi 1: A_op(i, k) = 0 for k > i,
// 2: B_op(k, j) = 0 for k > j.  lower: M == N, entries j <= i only (mirror: and C[j][i]).
struct OzGemm {
    int64_t M, N, K;
    const void* A; int64_t a_sl, a_sr;
    const void* B; int64_t b_sl, b_sr;
    bool same;        // B_op = A_op^T (one digit set)
    int dtype;        // of A and B
    double alpha, beta, diag;
    double* C; int64_t ldc;
    int lower, mirror, k_lo, k_hi;
};
size_t gemm_tc_scratch_bytes(int64_t M, int64_t N, int64_t K, bool same);
int launch_gemm_tc(const OzGemm& g, void* scratch, size_t scratch_bytes, cudaStream_t s);
bool gram_tc_enabled();
int launch_gram_tc(int dtype, int64_t m, int64_t nj, const void* A, int64_t lda, double alpha, double diag, double* G,
                   int64_t ldg, void* scratch, size_t scratch_bytes, cudaStream_t s);
int launch_gram(int dtype, int64_t m, int64_t nj, const void* A, int64_t lda, double alpha,
                double diag, double* G, int64_t ldg, bool full, cudaStream_t s);
// K = alpha A A^T + diag I (m x m, lower triangle or full) into FP64 G (ldg): the Woodbury
// kernel matrix of fat blocks (m_i < n_j).
int launch_gram_rows(int dtype, int64_t m, int64_t nj, const void* A, int64_t lda, double alpha,
                     double diag, double* G, int64_t ldg, cudaStream_t s);
// In-place: G (nj x nj FP64, lower triangle holding F) -> H = F^{-1} written to H (dtype, ldh).
// ws: FP64 scratch of factor_ws_doubles(nj) doubles.
size_t factor_ws_doubles(int64_t nj);
// One factor job: F (n x n lower, FP64, leading dim ldg; overwritten) -> H = F^{-1}
// (full symmetric, dtype hdtype, leading dim ldh); ws = factor_ws_doubles(n) FP64 scratch.
struct FactorJob {
    int64_t n;
    double* G;
    int64_t ldg;
    void* H;
    int64_t ldh;
    int hdtype;
    double* ws;
};
// All jobs' blocked Cholesky / inverse steps run in lockstep, up to 8 GEMMs per launch.
// tc_ws (optional): scratch for the large products on the tcgen05 Ozaki engine
// (>= factor_tc_scratch_bytes(n) for the largest n); null -> DMMA only.
int factor_inverse_batched(const FactorJob* jobs, int njobs, cudaStream_t s, void* tc_ws = nullptr,
                           size_t tc_bytes = 0);
size_t factor_tc_scratch_bytes(int64_t n);
int factor_inverse(int64_t nj, double* G, int64_t ldg, void* H, int64_t ldh, int dtype,
                   double* ws, cudaStream_t s);

// ---------------------------------------------------------------- outer step (a8-a12)
struct OuterScalars {   // device-resident scalars of the global step
    double t, v, tau, g, mcap, dz2, psi0, pad0;
    double p_r, d_r, b_r, pad1;
};
struct WsumIn {          // Collect inputs when k_zt computes wsum itself (x_all == nullptr: it reads wsum)
    const double* x_all = nullptr;
    const double* u_all = nullptr;
    int64_t stride = 0;
    int nl = 0;
};
int launch_zt(int64_t len, int N, double rho_c, double rho_b, double* wsum, const double* s,
              double* wbar, double* z, double* z_prev, OuterScalars* sc, cudaStream_t st, WsumIn cw = WsumIn{});
int launch_s_update(int64_t len, int64_t kappa, const double* z, double* s, OuterScalars* sc,
                    cudaStream_t st);
int launch_support(int64_t len, int64_t kappa, const double* z, int64_t* support, int64_t* count,
                   cudaStream_t st);

struct BlockVec {       // one local block's slice of the n*C vectors
    double* x;          // x_ij (n_j*C)
    double* u;          // u_ij
    int64_t c0, len;    // offset into the global n*C vector, length n_j*C
    int32_t node;       // global node id
    int64_t cta_begin;  // filled by the launcher
};
// wsum[l] = sum over local nodes (ascending) of x_i[l] + u_i[l]  ("Collect");
// x_all / u_all hold one full-length n*C vector per local node (zero off-rank).
int launch_wsum(int64_t len, int64_t stride, const double* x_all, const double* u_all, int n_local_nodes, double* wsum,
                cudaStream_t s);
// u_ij += x_ij - z_j and per-CTA partials of ||x_ij - z_j||^2.
int launch_u_update(BlockVec* bv, int nb, const double* z, double* partial, cudaStream_t s, int mode = 0);
int launch_seg_sums(const double* const* ptr, const int64_t* count, const int32_t* node, int n, double* out,
                    cudaStream_t s);
// node_sq[i] = sum over local blocks of node i (blocks[] order) of partials.
int launch_node_sq(const BlockVec* bv, int nb, const double* partial, int N, double* node_sq,
                   cudaStream_t s, OuterScalars* res = nullptr, double sqrtN_rho_c = 0.0);
int launch_residuals(int N, double sqrtN_rho_c, const double* node_sq, OuterScalars* sc, cudaStream_t s);
constexpr int kUThreads = 256;

// ---------------------------------------------------------------- single-pass sweep (k_fused4.cu)
constexpr int kF2MaxNodes = 32;
struct Fused2Args {
    const void* A[kF2MaxNodes];
    const void* b[kF2MaxNodes];
    const double* x[kF2MaxNodes];
    double* p[kF2MaxNodes];
    double* nu[kF2MaxNodes];
    double* delta[kF2MaxNodes];
    double* partial[kF2MaxNodes];     // [(cluster - cta_lo) x row groups][ncols]
    int64_t lda[kF2MaxNodes], ncols[kF2MaxNodes], row_off[kF2MaxNodes], cta_lo[kF2MaxNodes];
    int32_t active[kF2MaxNodes];      // inactive nodes (tol mode / schedule) keep all their state
    double* e2row[kF2MaxNodes];       // tol mode: per-row (abar - omega)^2 (else null)
    int nn;
    int64_t total_rows, max_cols_pad;
};
int launch_fused4(int dtype, const Fused2Args& a, int loss, double rho, int grid, cudaStream_t s);
int fused4_max_cols(int dtype);                     // bound of the compiled vector counts
bool fused4_plan_ok(int dtype, int64_t max_cols);  // a launch plan exists (ring of >= 4 slots, ...)
int fused4_groups(int dtype, int64_t max_cols);   // row groups of the CTA-pair sweep (partials per group)

// ---------------------------------------------------------------- finalize vectors (k_vec.cu)
int launch_dot(int64_t n, const double* a, const double* b, double* out, cudaStream_t s);
int launch_sum(int64_t n, const double* a, double* out, cudaStream_t s);   // fixed-order single-CTA sum
int launch_ridge_mask(int64_t n, const double* mask, const double* v, double lambda, double* y, cudaStream_t s);
int launch_cg_xr(int64_t n, const double* sc, const double* p, const double* Ap, double* x, double* r, cudaStream_t s);
int launch_cg_p(int64_t n, const double* sc, const double* r, double* p, cudaStream_t s);
int launch_to_f64(int dtype, int64_t n, const void* src, double* dst, cudaStream_t s);
// *bad = 1 if a label lies outside the loss domain (BICADMM_ERR_DOMAIN); *bad pre-zeroed
int launch_check_labels(int dtype, int loss, int C, int64_t n, const void* b, int* bad, cudaStream_t s);
// logistic refit on the support (k_vec.cu; DESIGN R29)
int launch_rf_gather(int dtype, const void* A, int64_t lda, int64_t m, int64_t c0, int64_t nj, const int64_t* sup,
                     const int64_t* cnt, double* AT, int64_t kp, int64_t row_off, cudaStream_t s, int C = 1);
int launch_rf_sm_rows(int64_t n, int C, const double* y, const double* W, double* G, double* P, double* objpart,
                      cudaStream_t s);
int launch_rf_sm_scale(int64_t n, int64_t kp, int C, const double* AT, const double* P, const int64_t* sup,
                       const int64_t* cnt, double* BT, double* U, cudaStream_t s);
int launch_rf_sm_combine(int64_t kp, int64_t ldf, int C, const int64_t* sup, const int64_t* cnt, double* F1,
                         const double* F2, cudaStream_t s);
int launch_rf_logit(int64_t n, const double* b, const double* w, double* psi, double* sd, double* objpart,
                    cudaStream_t s);
int64_t rf_logit_parts(int64_t n);
int launch_rf_scale_rows(int64_t n, int64_t kp, const double* AT, const double* sd, double* BT, cudaStream_t s);
int launch_rf_scatter(int64_t kp, const double* x, const int64_t* sup, const int64_t* cnt, double* xf, cudaStream_t s);
int launch_support_mask(int64_t cap, const int64_t* sup, const int64_t* cnt, double* mask, cudaStream_t s);
struct FatEw { const double* a; const double* b; const double* c; double* o; double* d; int64_t n; };
int launch_fat_ew(const FatEw* d, int nd, int mode, cudaStream_t s);   // k_vec.cu
int launch_axpy_into(int64_t n, const double* x, double* y, cudaStream_t s);          // y += x
int launch_axpy_scaled(int64_t n, double a, const double* x, double* y, cudaStream_t s);  // y += a x

}  // namespace bic
