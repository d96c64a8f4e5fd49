/*
 * bicadmm_ops.h -- primitive entry points of libbicadmm.so, one per step of the
 * Bi-cADMM hot path.  They run the SAME kernels the
 * solver runs (bicadmm.h) on caller-provided device buffers, so every step can be
 * parity-tested against the oracle in isolation.  All pointers are DEVICE
 * pointers unless named *_host; all vectors are FP64; matrices are `dtype`
 * (bicadmm_dtype) row-major with the alignment rules of bicadmm.h.  Calls that
 * return host scalars synchronise the stream.  Errors: bicadmm_rc.
 */
#ifndef BICADMM_OPS_H
#define BICADMM_OPS_H

#include "bicadmm.h"

#ifdef __cplusplus
extern "C" {
#endif

/* a4 ("Compute A_ij x_ij"): y[r] = sum_l A[r, l] x[l], r < m, l < nj. */
int bicadmm_op_gemv(int dtype, int64_t m, int64_t nj, const void* A, int64_t lda,
                    const double* x, double* y, void* stream);

/* a1+a2 (Eq. (24) normal equations, DESIGN R17):
 *   r[l] = rho_l * sum_r A[r, l] (p[r] + delta[r]) + rho_c (z[l] - u[l])
 * delta / z / u may be NULL (treated as 0).  ws >= bicadmm_op_gemv_t_ws(...) bytes. */
size_t bicadmm_op_gemv_t_ws(int dtype, int64_t m, int64_t nj);
int bicadmm_op_gemv_t(int dtype, int64_t m, int64_t nj, const void* A, int64_t lda,
                      const double* p, const double* delta, const double* z, const double* u,
                      double rho_l, double rho_c, double* r, void* ws, size_t ws_bytes, void* stream);

/* a6+a7 (Eqs. (22), (23)) for one node with M blocks in total:
 *   abar = S / M; omega = prox_{phi(M.,b)/(M rho_l)}(abar + nu); nu += abar - omega;
 *   delta = omega - abar - nu   (the next sweep's q_ij = p_ij + delta, Eq. (24)).
 * S is the block sum (m x C); b labels (dtype); nu in/out; omega may be NULL. */
int bicadmm_op_prox(int loss, int dtype, int C, int64_t m, int M, double rho_l, const void* b,
                    const double* S, double* nu, double* delta, double* omega, void* stream);

/* a0 (DESIGN R17): H = (rho_l A^T A + c I)^{-1}, full symmetric
 * nj x nj, row stride ldh >= nj, stored as dtype.  ws >= bicadmm_op_block_factor_ws. */
size_t bicadmm_op_block_factor_ws(int64_t nj);
int bicadmm_op_block_factor(int dtype, int64_t m, int64_t nj, const void* A, int64_t lda,
                            double rho_l, double c, void* H, int64_t ldh,
                            void* ws, size_t ws_bytes, void* stream);

/* Gram step of a0 alone: G = alpha A^T A + diag I (full symmetric, FP64, ldg >= nj). */
int bicadmm_op_gram(int dtype, int64_t m, int64_t nj, const void* A, int64_t lda,
                    double alpha, double diag, double* G, int64_t ldg, void* stream);

/* The same Gram on the 5th-generation tensor cores: FP64-accurate
 * Ozaki-scheme emulation with int8 digits of the column-scaled A on tcgen05.mma kind::i8
 * (S = 7 round-to-nearest digits: 50 bits below each column's maximum), TMEM int32
 * accumulators, FP64 recombination.
 * Writes the LOWER triangle of G = alpha A^T A + diag I (FP64, ldg >= nj); the upper triangle
 * is left untouched.  ws: device scratch >= bicadmm_op_gram_tc_ws(dtype, m, nj) bytes
 * (caller-owned).  Errors: BICADMM_ERR_INVALID on bad sizes or a short workspace. */
size_t bicadmm_op_gram_tc_ws(int dtype, int64_t m, int64_t nj);
int bicadmm_op_gram_tc(int dtype, int64_t m, int64_t nj, const void* A, int64_t lda, double alpha, double diag,
                       double* G, int64_t ldg, void* ws, size_t ws_bytes, void* stream);

/* General product on the same tcgen05 Ozaki engine (used by the a0 factor for its large
 * GEMMs): C = alpha A_op B_op + beta C (+ diag on i == j), C FP64 row-major (ldc),
 *   A_op(i, k) = A[i a_sl + k a_sr]  (M x K),   B_op(k, j) = B[j b_sl + k b_sr]  (K x N),
 * A and B of the storage type dtype (device, caller-owned); rows of A_op and columns of B_op
 * are scaled by their own power of two.  flags: bit 0 lower (M == N; only entries j <= i
 * written), bit 1 mirror (also C[j][i]), bits 4-5 k_lo, bits 8-9 k_hi: operand zero
 * structure whose tiles are skipped exactly -- k_lo 1: A_op(i,k) = 0 for k < i, 2: B_op(k,j) = 0
 * for k < j, 3: zero unless k >= max(i, j); k_hi 1: A_op(i,k) = 0 for k > i, 2: B_op(k,j) = 0
 * for k > j.  same != 0: B_op = A_op^T (B, b_sl, b_sr ignored; one digit set).
 * ws: device scratch >= bicadmm_op_gemm_tc_ws(M, N, K, same) bytes.
 * Errors: BICADMM_ERR_INVALID on bad sizes / flags or a short workspace. */
size_t bicadmm_op_gemm_tc_ws(int64_t M, int64_t N, int64_t K, int same);
int bicadmm_op_gemm_tc(int dtype, int64_t M, int64_t N, int64_t K, const void* A, int64_t a_sl, int64_t a_sr,
                       const void* B, int64_t b_sl, int64_t b_sr, int same, double alpha, double beta, double diag,
                       double* C, int64_t ldc, int flags, void* ws, size_t ws_bytes, void* stream);

/* a10 ((7b); DESIGN R3): wbar = wsum / N; exact (z,t) minimiser by the
 * weighted soft-threshold with tau the root of N rho_c tau = rho_b (psi(tau) - v).
 * z_prev receives the old z; out_host[0..3] = t, tau, ||z - z_prev||^2, psi(0). */
int bicadmm_op_zt(int64_t len, int N, double rho_c, double rho_b, const double* wsum,
                  const double* s, double v, double* wbar, double* z, double* z_prev,
                  double* out_host, void* stream);

/* a11+a12 ((13) P:137, (14) P:142; DESIGN R4, R5): T = kappa largest |z_l|, ties
 * to the lower index; Mcap = sum_T |z|; s = clamp((t - v)/Mcap, -1, 1) sgn(z) 1_T;
 * g = z's - t.  out_host[0..2] = Mcap, g, v + g. */
int bicadmm_op_s_update(int64_t len, int64_t kappa, const double* z, double t, double v,
                        double* s, double* out_host, void* stream);

/* a13 (DESIGN R19): support = top-kappa of |z| among z_l != 0 (ties to the lower
 * index), written ascending into support (int64, capacity kappa); count_host[0] = size. */
int bicadmm_op_support(int64_t len, int64_t kappa, const double* z, int64_t* support,
                       int64_t* count_host, void* stream);

/* Total kernels launched by this library in this process (gpu_launches evidence). */
int64_t bicadmm_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* BICADMM_OPS_H */
