// k_vec.cu -- small vector kernels for finalisation: the
// least-squares ridge refit on the recovered support (DESIGN R19),
//   (2 sum_i A_iT^T A_iT + lambda I) x_T = 2 sum_i A_iT^T b_i,
// solved by conjugate gradients whose matrix-vector products are the same HBM
// GEMV / GEMV-T passes as the inner loop (x zero off the support).  The system is
// SPD and, for kappa << m with unit-norm columns, condition ~1, so CG reaches
// 1e-15 relative residual in a few tens of iterations.  Dot products are
// single-CTA fixed-order reductions (bit-identical on every rank).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace bic {

// out[0] = sum_l a[l] b[l] (fixed order)
__global__ void __launch_bounds__(1024) k_dot(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                                             double* out) {
    __shared__ double scratch[32];
    double s = 0.0;
    for (int64_t l = threadIdx.x; l < n; l += 1024) s += a[l] * b[l];
    s = block_sum(s, scratch);
    if (threadIdx.x == 0) *out = s;
}

int launch_dot(int64_t n, const double* a, const double* b, double* out, cudaStream_t s) {
    k_dot<<<1, 1024, 0, s>>>(n, a, b, out);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

__global__ void __launch_bounds__(1024) k_sum(int64_t n, const double* __restrict__ a, double* out) {
    __shared__ double scratch[32];
    double s = 0.0;
    for (int64_t l = threadIdx.x; l < n; l += 1024) s += a[l];
    s = block_sum(s, scratch);
    if (threadIdx.x == 0) *out = s;
}

int launch_sum(int64_t n, const double* a, double* out, cudaStream_t s) {
    k_sum<<<1, 1024, 0, s>>>(n, a, out);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

// y[l] = mask[l] * (y[l] + lambda * v[l])
__global__ void k_ridge_mask(int64_t n, const double* __restrict__ mask, const double* __restrict__ v, double lambda,
                             double* __restrict__ y) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l < n) y[l] = mask[l] * (y[l] + lambda * v[l]);
}

int launch_ridge_mask(int64_t n, const double* mask, const double* v, double lambda, double* y, cudaStream_t s) {
    k_ridge_mask<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, mask, v, lambda, y);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

// CG step with device scalars: sc[0] = rr, sc[1] = pAp  ->  alpha = rr / pAp;
// x += alpha p; r -= alpha Ap.
__global__ void k_cg_xr(int64_t n, const double* __restrict__ sc, const double* __restrict__ p,
                        const double* __restrict__ Ap, double* __restrict__ x, double* __restrict__ r) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= n) return;
    const double alpha = sc[1] != 0.0 ? sc[0] / sc[1] : 0.0;
    x[l] += alpha * p[l];
    r[l] -= alpha * Ap[l];
}

// p = r + (rr_new / rr) p   (sc[0] = rr, sc[2] = rr_new)
__global__ void k_cg_p(int64_t n, const double* __restrict__ sc, const double* __restrict__ r, double* __restrict__ p) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= n) return;
    const double beta = sc[0] != 0.0 ? sc[2] / sc[0] : 0.0;
    p[l] = r[l] + beta * p[l];
}

int launch_cg_xr(int64_t n, const double* sc, const double* p, const double* Ap, double* x, double* r, cudaStream_t s) {
    k_cg_xr<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, sc, p, Ap, x, r);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

int launch_cg_p(int64_t n, const double* sc, const double* r, double* p, cudaStream_t s) {
    k_cg_p<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, sc, r, p);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

// dst[l] = (double) src[l]  (labels in the storage dtype -> FP64)
template <typename T>
__global__ void k_to_f64(int64_t n, const T* __restrict__ src, double* __restrict__ dst) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l < n) dst[l] = (double)src[l];
}

int launch_to_f64(int dtype, int64_t n, const void* src, double* dst, cudaStream_t s) {
    if (dtype == BICADMM_F64) k_to_f64<double><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, (const double*)src, dst);
    else k_to_f64<float><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, (const float*)src, dst);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

// Label domain of the loss (bicadmm.h BICADMM_ERR_DOMAIN, DESIGN R12): logistic and
// hinge labels in {-1, +1}, softmax class ids integral in [0, C), LS labels finite.  Any
// violation sets *bad = 1 (pre-zeroed; read back once by bicadmm_setup).
template <typename T>
__global__ void k_check_labels(int64_t n, const T* __restrict__ b, int loss, int C, int* bad) {
    int my = 0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const double v = (double)b[r];
        bool ok;
        if (loss == BICADMM_LOGISTIC || loss == BICADMM_HINGE) ok = v == 1.0 || v == -1.0;
        else if (loss == BICADMM_SOFTMAX) ok = v >= 0.0 && v < (double)C && v == floor(v);
        else ok = isfinite(v);
        my |= ok ? 0 : 1;
    }
    if (__syncthreads_or(my) && threadIdx.x == 0) *bad = 1;
}

int launch_check_labels(int dtype, int loss, int C, int64_t n, const void* b, int* bad, cudaStream_t s) {
    if (n <= 0) return BICADMM_OK;
    const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, 1024);
    if (dtype == BICADMM_F64) k_check_labels<double><<<g, 256, 0, s>>>(n, (const double*)b, loss, C, bad);
    else k_check_labels<float><<<g, 256, 0, s>>>(n, (const float*)b, loss, C, bad);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

// mask[l] = 1 on the support list, else 0 (mask pre-zeroed)
__global__ void k_support_mask(const int64_t* __restrict__ sup, const int64_t* __restrict__ cnt, double* mask) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < *cnt) mask[sup[k]] = 1.0;
}

int launch_support_mask(int64_t cap, const int64_t* sup, const int64_t* cnt, double* mask, cudaStream_t s) {
    k_support_mask<<<(unsigned)((cap + 255) / 256), 256, 0, s>>>(sup, cnt, mask);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

__global__ void k_axpy(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l < n) y[l] += a * x[l];
}

int launch_axpy_into(int64_t n, const double* x, double* y, cudaStream_t s) { return launch_axpy_scaled(n, 1.0, x, y, s); }

int launch_axpy_scaled(int64_t n, double a, const double* x, double* y, cudaStream_t s) {
    if (n <= 0) return BICADMM_OK;
    k_axpy<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, a, x, y);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

// Woodbury fat-block sweep elementwise steps (R27), batched over blocks:
//   mode 0: o = a + b                       (q = p + delta;  zu = z - u uses mode 2)
//   mode 1: o = a + b + c, d = a - o        (p = q + t1 + y0, diff = q - p)
//   mode 2: o = a - b
// ----------------------------------------------------------------------------- logistic refit
// (DESIGN R29) on the support T, single rank: the support columns of every local row are
// gathered into a dense FP64 matrix AT (rows of all local nodes stacked, kp columns).
template <typename T>
__global__ void k_rf_gather(const T* __restrict__ A, int64_t lda, int64_t m, int64_t c0, int64_t nj,
                            const int64_t* __restrict__ sup, const int64_t* __restrict__ cnt, double* __restrict__ AT,
                            int64_t kp, int64_t row_off, int C) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m * kp) return;
    const int64_t r = e / kp, a = e % kp;
    if (a >= *cnt) return;
    const int64_t l = sup[a] / C;   // entry l*C + c of vec(X) -> feature l
    if (l < c0 || l >= c0 + nj) return;
    AT[(row_off + r) * kp + a] = (double)A[r * lda + (l - c0)];
}

int launch_rf_gather(int dtype, const void* A, int64_t lda, int64_t m, int64_t c0, int64_t nj, const int64_t* sup,
                     const int64_t* cnt, double* AT, int64_t kp, int64_t row_off, cudaStream_t s, int C) {
    const int64_t n = m * kp;
    if (n <= 0) return BICADMM_OK;
    const unsigned g = (unsigned)((n + 255) / 256);
    if (dtype == BICADMM_F64) k_rf_gather<double><<<g, 256, 0, s>>>(static_cast<const double*>(A), lda, m, c0, nj, sup, cnt, AT, kp, row_off, C);
    else k_rf_gather<float><<<g, 256, 0, s>>>(static_cast<const float*>(A), lda, m, c0, nj, sup, cnt, AT, kp, row_off, C);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

// per row r: sp = sigma(b w); psi = -b (1 - sp) (the loss derivative); sd = sqrt(sp (1 - sp))
// (root of the second derivative); objective partials ln(1 + exp(-b w)) per CTA (fixed order)
constexpr int kRfThreads = 256;
__global__ void __launch_bounds__(kRfThreads) k_rf_logit(int64_t n, const double* __restrict__ b,
                                                         const double* __restrict__ w, double* __restrict__ psi,
                                                         double* __restrict__ sd, double* __restrict__ objpart) {
    __shared__ double scratch[32];
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double f = 0.0;
    if (r < n) {
        const double y = -b[r] * w[r];
        f = y > 0.0 ? y + log1p(exp(-y)) : log1p(exp(y));
        if (psi) {
            const double sp = 1.0 / (1.0 + exp(y));   // sigma(b w)
            psi[r] = -b[r] * (1.0 - sp);
            sd[r] = sqrt(sp * (1.0 - sp));
        }
    }
    f = block_sum(f, scratch);
    if (threadIdx.x == 0) objpart[blockIdx.x] = f;
}

int launch_rf_logit(int64_t n, const double* b, const double* w, double* psi, double* sd, double* objpart,
                    cudaStream_t s) {
    if (n <= 0) return BICADMM_OK;
    k_rf_logit<<<(unsigned)((n + kRfThreads - 1) / kRfThreads), kRfThreads, 0, s>>>(n, b, w, psi, sd, objpart);
    BIC_LAUNCHED();
    return BICADMM_OK;
}
int64_t rf_logit_parts(int64_t n) { return (n + kRfThreads - 1) / kRfThreads; }

// BT = diag(sd) AT (row scaling), so BT^T BT = AT^T diag(sp (1 - sp)) AT
__global__ void k_rf_scale_rows(int64_t n, int64_t kp, const double* __restrict__ AT, const double* __restrict__ sd,
                                double* __restrict__ BT) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n * kp) BT[e] = sd[e / kp] * AT[e];
}

int launch_rf_scale_rows(int64_t n, int64_t kp, const double* AT, const double* sd, double* BT, cudaStream_t s) {
    if (n * kp <= 0) return BICADMM_OK;
    k_rf_scale_rows<<<(unsigned)((n * kp + 255) / 256), 256, 0, s>>>(n, kp, AT, sd, BT);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

// softmax rows: p = softmax(w_r) (C classes), objective partials logsumexp(w) - w_y,
// G = p - e_y (gradient weights; null in objective-only mode) and P = p
__global__ void __launch_bounds__(kRfThreads) k_rf_sm_rows(int64_t n, int C, const double* __restrict__ y,
                                                           const double* __restrict__ W, double* __restrict__ G,
                                                           double* __restrict__ P, double* __restrict__ objpart) {
    __shared__ double scratch[32];
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double f = 0.0;
    if (r < n) {
        const double* w = W + r * C;
        double mx = w[0];
        for (int c = 1; c < C; ++c) mx = fmax(mx, w[c]);
        double se = 0.0;
        for (int c = 0; c < C; ++c) se += exp(w[c] - mx);
        const int yy = (int)y[r];
        f = mx + log(se) - w[yy];
        if (G) {
            for (int c = 0; c < C; ++c) {
                const double p = exp(w[c] - mx) / se;
                P[r * C + c] = p;
                G[r * C + c] = p - (c == yy ? 1.0 : 0.0);
            }
        }
    }
    f = block_sum(f, scratch);
    if (threadIdx.x == 0) objpart[blockIdx.x] = f;
}

int launch_rf_sm_rows(int64_t n, int C, const double* y, const double* W, double* G, double* P, double* objpart,
                      cudaStream_t s) {
    if (n <= 0) return BICADMM_OK;
    k_rf_sm_rows<<<(unsigned)((n + kRfThreads - 1) / kRfThreads), kRfThreads, 0, s>>>(n, C, y, W, G, P, objpart);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

// softmax Hessian factors: BT[r][a] = sqrt(p_{r,c_a}) AT[r][a], U[r][a] = p_{r,c_a} AT[r][a]
// (c_a = sup[a] % C; padding columns of AT are zero)
__global__ void k_rf_sm_scale(int64_t n, int64_t kp, int C, const double* __restrict__ AT, const double* __restrict__ P,
                              const int64_t* __restrict__ sup, const int64_t* __restrict__ cnt, double* __restrict__ BT,
                              double* __restrict__ U) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * kp) return;
    const int64_t r = e / kp, a = e % kp;
    const double p = a < *cnt ? P[r * C + sup[a] % C] : 0.0;
    BT[e] = sqrt(p) * AT[e];
    U[e] = p * AT[e];
}

int launch_rf_sm_scale(int64_t n, int64_t kp, int C, const double* AT, const double* P, const int64_t* sup,
                       const int64_t* cnt, double* BT, double* U, cudaStream_t s) {
    if (n * kp <= 0) return BICADMM_OK;
    k_rf_sm_scale<<<(unsigned)((n * kp + 255) / 256), 256, 0, s>>>(n, kp, C, AT, P, sup, cnt, BT, U);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

// lower triangle: F1 <- [c_a == c_b] F1 - F2 (the softmax Hessian from its two Grams; the
// ridge is already on F1's diagonal, padding rows/columns keep lambda I)
__global__ void k_rf_sm_combine(int64_t kp, int64_t ldf, int C, const int64_t* __restrict__ sup,
                                const int64_t* __restrict__ cnt, double* __restrict__ F1, const double* __restrict__ F2) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= kp * kp) return;
    const int64_t a = e / kp, b = e % kp;
    if (b > a) return;
    const int64_t k = *cnt;
    if (a >= k || b >= k) return;
    const bool same = (sup[a] % C) == (sup[b] % C);
    const double v = (same ? F1[a * ldf + b] : (a == b ? F1[a * ldf + b] : 0.0)) - F2[a * ldf + b];
    F1[a * ldf + b] = v;
}

int launch_rf_sm_combine(int64_t kp, int64_t ldf, int C, const int64_t* sup, const int64_t* cnt, double* F1,
                         const double* F2, cudaStream_t s) {
    k_rf_sm_combine<<<(unsigned)((kp * kp + 255) / 256), 256, 0, s>>>(kp, ldf, C, sup, cnt, F1, F2);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

__global__ void k_rf_scatter(const double* __restrict__ x, const int64_t* __restrict__ sup,
                             const int64_t* __restrict__ cnt, double* __restrict__ xf) {
    const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a < *cnt) xf[sup[a]] = x[a];
}

int launch_rf_scatter(int64_t kp, const double* x, const int64_t* sup, const int64_t* cnt, double* xf, cudaStream_t s) {
    k_rf_scatter<<<(unsigned)((kp + 255) / 256), 256, 0, s>>>(x, sup, cnt, xf);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

struct FatEwBatch { FatEw d[kMaxDesc]; int64_t begin[kMaxDesc + 1]; int nd; };

__global__ void k_fat_ew(const FatEwBatch B, int mode) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= B.begin[B.nd]) return;
    int k = 0;
    while (k + 1 < B.nd && g >= B.begin[k + 1]) ++k;
    const FatEw& e = B.d[k];
    const int64_t l = g - B.begin[k];
    const double a = e.a[l], b = e.b ? e.b[l] : 0.0;
    if (mode == 0) e.o[l] = a + b;
    else if (mode == 2) e.o[l] = a - b;
    else {
        const double o = (a + b) + e.c[l];
        e.o[l] = o;
        e.d[l] = a - o;
    }
}

int launch_fat_ew(const FatEw* d, int nd, int mode, cudaStream_t s) {
    for (int base = 0; base < nd; base += kMaxDesc) {
        FatEwBatch B;
        B.nd = nd - base < kMaxDesc ? nd - base : kMaxDesc;
        int64_t t = 0;
        for (int k = 0; k < B.nd; ++k) { B.d[k] = d[base + k]; B.begin[k] = t; t += B.d[k].n; }
        B.begin[B.nd] = t;
        if (t == 0) continue;
        k_fat_ew<<<(unsigned)((t + 255) / 256), 256, 0, s>>>(B, mode);
        BIC_LAUNCHED();
    }
    return BICADMM_OK;
}

}  // namespace bic
