// ops.cu -- primitive entry points (include/bicadmm_ops.h): each runs the same
// kernels the solver runs, on caller buffers, so steps can be parity-tested alone.
// Ops that return host scalars use a small stream-ordered device allocation and
// synchronise; they are test/diagnostic entry points, not the solver's path.
#include <cuda_runtime.h>
#include <string.h>

#include "../../include/bicadmm.h"
#include "../../include/bicadmm_ops.h"
#include "common.cuh"
#include "kernels.h"

using namespace bic;

static int sm_count() {
    int dev = 0, sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, dev);
    return sm;
}

static bool aligned_ok(const void* A, int64_t lda) { return A && lda % 4 == 0 && ((uintptr_t)A) % 16 == 0; }

extern "C" int bicadmm_op_gemv(int dtype, int64_t m, int64_t nj, const void* A, int64_t lda, const double* x,
                               double* y, void* stream) {
    if (m < 0 || nj < 1 || lda < nj || !aligned_ok(A, lda) || !x || !y || ((uintptr_t)x) % 16) return BICADMM_ERR_INVALID;
    if (dtype != BICADMM_F64 && dtype != BICADMM_F32) return BICADMM_ERR_INVALID;
    GemvDesc d{A, lda, m, nj, x, y, 0};
    return launch_gemv(dtype, &d, 1, gemv_grid_cap(dtype, sm_count()), (cudaStream_t)stream);
}

static void gt_plan(int dtype, int64_t m, int64_t nj, GemvTDesc* d, int64_t* need) {
    *d = GemvTDesc{};
    d->rows = m;
    d->cols = nj;
    plan_gemv_t(dtype, d, 1, sm_count(), need);
}

extern "C" size_t bicadmm_op_gemv_t_ws(int dtype, int64_t m, int64_t nj) {
    GemvTDesc d;
    int64_t need = 0;
    gt_plan(dtype, m, nj, &d, &need);
    return sizeof(double) * (size_t)need;
}

extern "C" int bicadmm_op_gemv_t(int dtype, int64_t m, int64_t nj, const void* A, int64_t lda, const double* p,
                                 const double* delta, const double* z, const double* u, double rho_l, double rho_c,
                                 double* r, void* ws, size_t ws_bytes, void* stream) {
    if (m < 1 || nj < 1 || lda < nj || !aligned_ok(A, lda) || !p || !r) return BICADMM_ERR_INVALID;
    if (dtype != BICADMM_F64 && dtype != BICADMM_F32) return BICADMM_ERR_INVALID;
    GemvTDesc d;
    int64_t need = 0;
    gt_plan(dtype, m, nj, &d, &need);
    if (!ws || ws_bytes < sizeof(double) * (size_t)need) return BICADMM_ERR_OOM;
    d.A = A; d.lda = lda; d.p = p; d.delta = delta; d.z = z; d.u = u; d.r = r; d.partial = (double*)ws;
    return launch_gemv_t(dtype, &d, 1, rho_l, rho_c, (cudaStream_t)stream);
}

extern "C" int bicadmm_op_prox(int loss, int dtype, int C, int64_t m, int M, double rho_l, const void* b,
                               const double* S, double* nu, double* delta, double* omega, void* stream) {
    if (m < 1 || M < 1 || !(rho_l > 0) || !b || !S || !nu || !delta) return BICADMM_ERR_INVALID;
    if (loss < 0 || loss > 3 || (loss == BICADMM_SOFTMAX) != (C > 1) || C < 1 || C > 16) return BICADMM_ERR_INVALID;
    ProxNode p{};
    p.b = b; p.S = S; p.nu = nu; p.delta = delta; p.omega = omega; p.m = m; p.np = 0; p.pstride = 0;
    return launch_prox(loss, dtype, C, M, rho_l, &p, 1, (cudaStream_t)stream);
}

extern "C" size_t bicadmm_op_block_factor_ws(int64_t nj) {
    const int64_t ldg = (nj + 7) / 8 * 8;
    return sizeof(double) * ((size_t)(ldg * nj) + factor_ws_doubles(nj)) + 512;
}

extern "C" int bicadmm_op_block_factor(int dtype, int64_t m, int64_t nj, const void* A, int64_t lda, double rho_l,
                                       double c, void* H, int64_t ldh, void* ws, size_t ws_bytes, void* stream) {
    if (m < 1 || nj < 1 || lda < nj || !aligned_ok(A, lda) || !H || ldh < nj) return BICADMM_ERR_INVALID;
    if (!ws || ws_bytes < bicadmm_op_block_factor_ws(nj)) return BICADMM_ERR_OOM;
    const int64_t ldg = (nj + 7) / 8 * 8;
    double* G = (double*)(((uintptr_t)ws + 255) / 256 * 256);
    double* fws = G + ldg * nj;
    int rc = launch_gram(dtype, m, nj, A, lda, rho_l, c, G, ldg, false, (cudaStream_t)stream);
    if (rc) return rc;
    return factor_inverse(nj, G, ldg, H, ldh, dtype, fws, (cudaStream_t)stream);
}

extern "C" int bicadmm_op_gram(int dtype, int64_t m, int64_t nj, const void* A, int64_t lda, double alpha,
                               double diag, double* G, int64_t ldg, void* stream) {
    if (m < 1 || nj < 1 || lda < nj || !A || !G || ldg < nj) return BICADMM_ERR_INVALID;
    return launch_gram(dtype, m, nj, A, lda, alpha, diag, G, ldg, true, (cudaStream_t)stream);
}

extern "C" size_t bicadmm_op_gram_tc_ws(int dtype, int64_t m, int64_t nj) {
    return (m < 1 || nj < 1) ? 0 : gram_tc_scratch_bytes(dtype, m, nj);
}

extern "C" size_t bicadmm_op_gemm_tc_ws(int64_t M, int64_t N, int64_t K, int same) {
    return (M < 1 || N < 1 || K < 0) ? 0 : gemm_tc_scratch_bytes(M, N, K, same != 0);
}

extern "C" int bicadmm_op_gemm_tc(int dtype, int64_t M, int64_t N, int64_t K, const void* A, int64_t a_sl,
                                  int64_t a_sr, const void* B, int64_t b_sl, int64_t b_sr, int same, double alpha,
                                  double beta, double diag, double* C, int64_t ldc, int flags, void* ws,
                                  size_t ws_bytes, void* stream) {
    if (M < 1 || N < 1 || K < 0 || !A || (!same && !B) || !C || ldc < N || !ws) return BICADMM_ERR_INVALID;
    if (dtype != BICADMM_F64 && dtype != BICADMM_F32) return BICADMM_ERR_INVALID;
    OzGemm g{};
    g.M = M; g.N = N; g.K = K;
    g.A = A; g.a_sl = a_sl; g.a_sr = a_sr;
    g.same = same != 0;
    g.B = g.same ? A : B; g.b_sl = g.same ? a_sl : b_sl; g.b_sr = g.same ? a_sr : b_sr;
    g.dtype = dtype; g.alpha = alpha; g.beta = beta; g.diag = diag; g.C = C; g.ldc = ldc;
    g.lower = flags & 1; g.mirror = (flags >> 1) & 1; g.k_lo = (flags >> 4) & 3; g.k_hi = (flags >> 8) & 3;
    return launch_gemm_tc(g, ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" int bicadmm_op_gram_tc(int dtype, int64_t m, int64_t nj, const void* A, int64_t lda, double alpha,
                                  double diag, double* G, int64_t ldg, void* ws, size_t ws_bytes, void* stream) {
    if (m < 1 || nj < 1 || lda < nj || !A || !G || ldg < nj || !ws) return BICADMM_ERR_INVALID;
    return launch_gram_tc(dtype, m, nj, A, lda, alpha, diag, G, ldg, ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" int bicadmm_op_zt(int64_t len, int N, double rho_c, double rho_b, const double* wsum, const double* s,
                             double v, double* wbar, double* z, double* z_prev, double* out_host, void* stream) {
    if (len < 1 || N < 1 || !wsum || !s || !wbar || !z || !z_prev || !out_host) return BICADMM_ERR_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    OuterScalars* sc = nullptr;
    BIC_CUDA(cudaMallocAsync((void**)&sc, sizeof(OuterScalars), st));
    OuterScalars h{};
    h.v = v;
    BIC_CUDA(cudaMemcpyAsync(sc, &h, sizeof(h), cudaMemcpyHostToDevice, st));
    int rc = launch_zt(len, N, rho_c, rho_b, const_cast<double*>(wsum), s, wbar, z, z_prev, sc, st);
    if (!rc) {
        BIC_CUDA(cudaMemcpyAsync(&h, sc, sizeof(h), cudaMemcpyDeviceToHost, st));
        BIC_CUDA(cudaStreamSynchronize(st));
        out_host[0] = h.t; out_host[1] = h.tau; out_host[2] = h.dz2; out_host[3] = h.psi0;
    }
    cudaFreeAsync(sc, st);
    return rc;
}

extern "C" int bicadmm_op_s_update(int64_t len, int64_t kappa, const double* z, double t, double v, double* s,
                                   double* out_host, void* stream) {
    if (len < 1 || kappa < 0 || !z || !s || !out_host) return BICADMM_ERR_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    OuterScalars* sc = nullptr;
    BIC_CUDA(cudaMallocAsync((void**)&sc, sizeof(OuterScalars), st));
    OuterScalars h{};
    h.t = t; h.v = v;
    BIC_CUDA(cudaMemcpyAsync(sc, &h, sizeof(h), cudaMemcpyHostToDevice, st));
    int rc = launch_s_update(len, kappa, z, s, sc, st);
    if (!rc) {
        BIC_CUDA(cudaMemcpyAsync(&h, sc, sizeof(h), cudaMemcpyDeviceToHost, st));
        BIC_CUDA(cudaStreamSynchronize(st));
        out_host[0] = h.mcap; out_host[1] = h.g; out_host[2] = h.v;
    }
    cudaFreeAsync(sc, st);
    return rc;
}

extern "C" int bicadmm_op_support(int64_t len, int64_t kappa, const double* z, int64_t* support, int64_t* count_host,
                                  void* stream) {
    if (len < 1 || kappa < 0 || !z || !support || !count_host) return BICADMM_ERR_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    int64_t* cnt = nullptr;
    BIC_CUDA(cudaMallocAsync((void**)&cnt, sizeof(int64_t), st));
    int rc = launch_support(len, kappa, z, support, cnt, st);
    if (!rc) {
        BIC_CUDA(cudaMemcpyAsync(count_host, cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        BIC_CUDA(cudaStreamSynchronize(st));
    }
    cudaFreeAsync(cnt, st);
    return rc;
}
