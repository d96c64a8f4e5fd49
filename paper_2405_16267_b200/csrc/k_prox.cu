// k_prox.cu -- per-sample loss prox and dual update of the node-level sharing
// ADMM (Eqs. (22), (23)), fused with the q-vector
// formation of the next sweep (a1, Eq. (24)).
//
// For node i and sample r (C classes for softmax):
//   S     = sum_j A_ij x_ij            (block sum; P:244 AllReduce when blocks span GPUs)
//   abar  = S / M
//   omega = argmin_w phi(M w, b_r) + (M rho_l / 2) ||w - (abar + nu)||^2   (22)
//   nu   += abar - omega               (23)
//   delta = omega - abar - nu          (so q_ij = p_ij + delta, Eq. (24))
// "the omega-update splits entirely into m_i scalar optimization problems":
// one thread per sample.  LS and hinge are closed forms; logistic uses a
// safeguarded Newton iteration (bracket [p - 1/rho_l, p + 1/rho_l]); softmax a
// damped Newton step with the Sherman-Morrison inverse of M(diag pi - pi pi^T) + rho_l I.
#include "common.cuh"
#include "kernels.h"
#include <cfloat>
#include <algorithm>

namespace bic {

struct ProxBatch {
    ProxNode n[kMaxDesc];
    int nn;
    int64_t total_ctas;
};

__device__ __forceinline__ double sigmoid(double a) {
    if (a >= 0.0) return 1.0 / (1.0 + exp(-a));
    const double e = exp(a);
    return e / (1.0 + e);
}

__device__ __forceinline__ double prox_logistic(int M, double rho, double b, double p, double w0) {
    // root of g(w) = -b sigma(-b M w) + rho (w - p), g' = M sigma (1 - sigma) + rho > 0;
    // Newton from w0 (the previous sweep's omega of this sample, same root) when inside the bracket
    double lo = p - 1.0 / rho, hi = p + 1.0 / rho;
    double w = (w0 > lo && w0 < hi) ? w0 : p;
    const double Md = (double)M;
    for (int it = 0; it < 60; ++it) {
        const double sg = sigmoid(-b * Md * w);
        const double g = -b * sg + rho * (w - p);
        if (g > 0.0) hi = w; else lo = w;
        const double gp = Md * sg * (1.0 - sg) + rho;
        const double step = g / gp;
        // converged: accept the Newton step (checked BEFORE the bracket safeguard, which
        // would otherwise turn an ulp-sized step landing on the bracket into a bisection)
        if (fabs(step) <= 4.0 * DBL_EPSILON * fmax(1.0, fabs(w))) { w -= step; break; }
        double wn = w - step;
        if (!(wn > lo && wn < hi)) wn = 0.5 * (lo + hi);
        w = wn;
    }
    return w;
}

__device__ __forceinline__ double prox_hinge(int M, double rho, double b, double p) {
    const double pp = b * p, Md = (double)M;
    double y;
    if (Md * pp > 1.0) y = pp;
    else if (Md * (pp + 1.0 / rho) < 1.0) y = pp + 1.0 / rho;
    else y = 1.0 / Md;
    return b * y;
}

template <int CM>
__device__ double softmax_obj(int C, double Md, double rho, int y, const double* p, const double* w) {
    double mx = -INFINITY;
    for (int c = 0; c < C; ++c) mx = fmax(mx, Md * w[c]);
    double se = 0.0, q = 0.0;
    for (int c = 0; c < C; ++c) { se += exp(Md * w[c] - mx); q += (w[c] - p[c]) * (w[c] - p[c]); }
    return mx + log(se) - Md * w[y] + 0.5 * Md * rho * q;
}

template <int CM>
__device__ void prox_softmax(int C, int M, double rho, int y, const double* p, double* w) {
    const double Md = (double)M;
    double pi[CM], g[CM], d[CM], tr[CM];
    for (int c = 0; c < C; ++c) w[c] = p[c];
    for (int it = 0; it < 100; ++it) {
        double mx = -INFINITY;
        for (int c = 0; c < C; ++c) mx = fmax(mx, Md * w[c]);
        double se = 0.0;
        for (int c = 0; c < C; ++c) { pi[c] = exp(Md * w[c] - mx); se += pi[c]; }
        for (int c = 0; c < C; ++c) pi[c] /= se;
        // H = D - M pi pi^T, D = rho + M pi  =>  H^{-1} g = D^{-1} g + M D^{-1} pi (pi^T D^{-1} g) / (1 - M pi^T D^{-1} pi)
        double a = 0.0, bden = 0.0;
        for (int c = 0; c < C; ++c) {
            g[c] = pi[c] - (c == y ? 1.0 : 0.0) + rho * (w[c] - p[c]);
            const double Dc = rho + Md * pi[c];
            a += pi[c] * g[c] / Dc;
            bden += pi[c] * pi[c] / Dc;
        }
        const double coef = Md * a / (1.0 - Md * bden);
        double dmax = 0.0, wmax = 1.0;
        for (int c = 0; c < C; ++c) d[c] = (g[c] + coef * pi[c]) / (rho + Md * pi[c]);
        const double f0 = softmax_obj<CM>(C, Md, rho, y, p, w);
        double step = 1.0;
        for (int ls = 0; ls < 60; ++ls) {
            for (int c = 0; c < C; ++c) tr[c] = w[c] - step * d[c];
            if (softmax_obj<CM>(C, Md, rho, y, p, tr) <= f0 + 1e-12 * (1.0 + fabs(f0))) break;
            step *= 0.5;
        }
        for (int c = 0; c < C; ++c) {
            const double dc = step * d[c];
            dmax = fmax(dmax, fabs(dc));
            w[c] -= dc;
            wmax = fmax(wmax, fabs(w[c]));
        }
        if (dmax <= 4.0 * DBL_EPSILON * wmax) break;
    }
}

template <typename T, int LOSS, int CM>
__global__ void __launch_bounds__(kProxThreads) k_prox(const __grid_constant__ ProxBatch B, int C, int M,
                                                       double rho) {
    __shared__ double scratch[32];
    const int64_t cta = blockIdx.x;
    int ni = 0;
    while (ni + 1 < B.nn && cta >= B.n[ni + 1].cta_begin) ++ni;
    const ProxNode& P = B.n[ni];
    const int64_t r = (cta - P.cta_begin) * kProxThreads + threadIdx.x;
    double sq = 0.0;
    if (r < P.m) {
        const double Md = (double)M;
        const double bl = (double)static_cast<const T*>(P.b)[r];
        double abar[CM], pa[CM], om[CM];
        for (int c = 0; c < C; ++c) {
            double S;
            if (P.S) {
                S = P.S[r * C + c];
            } else {
                S = 0.0;
                for (int j = 0; j < P.np; ++j) S += P.p[j * P.pstride + r * C + c];
            }
            abar[c] = S / Md;
            pa[c] = abar[c] + P.nu[r * C + c];
        }
        if constexpr (LOSS == BICADMM_LS) {
            om[0] = (2.0 * bl + rho * pa[0]) / (2.0 * Md + rho);
        } else if constexpr (LOSS == BICADMM_LOGISTIC) {
            // Newton warm start: the previous sweep's omega of this sample (P.omega holds it)
            const double w0 = P.omega ? P.omega[r] : pa[0];
            om[0] = prox_logistic(M, rho, bl, pa[0], w0);
        } else if constexpr (LOSS == BICADMM_HINGE) {
            om[0] = prox_hinge(M, rho, bl, pa[0]);
        } else {
            prox_softmax<CM>(C, M, rho, (int)bl, pa, om);
        }
        for (int c = 0; c < C; ++c) {
            const double nu = P.nu[r * C + c] + abar[c] - om[c];
            P.nu[r * C + c] = nu;
            P.delta[r * C + c] = om[c] - abar[c] - nu;
            if (P.omega) P.omega[r * C + c] = om[c];
            const double e = abar[c] - om[c];
            sq += e * e;
        }
    }
    if (P.sq_partial) {
        const double s = block_sum(sq, scratch);
        if (threadIdx.x == 0) P.sq_partial[cta - P.cta_begin] = s;
    }
}

int launch_prox(int loss, int dtype, int C, int M, double rho_l, ProxNode* nodes, int nn, cudaStream_t s) {
    if (C > 16 || (loss == BICADMM_SOFTMAX) != (C > 1)) return BICADMM_ERR_INVALID;
    for (int base = 0; base < nn; base += kMaxDesc) {
        ProxBatch B;
        B.nn = nn - base < kMaxDesc ? nn - base : kMaxDesc;
        int64_t t = 0;
        for (int k = 0; k < B.nn; ++k) {
            B.n[k] = nodes[base + k];
            B.n[k].cta_begin = t;
            t += (B.n[k].m + kProxThreads - 1) / kProxThreads;
        }
        B.total_ctas = t;
        if (t == 0) continue;
        const unsigned g = (unsigned)t;
#define BIC_PROX(T)                                                                              \
    switch (loss) {                                                                              \
    case BICADMM_LS: k_prox<T, BICADMM_LS, 1><<<g, kProxThreads, 0, s>>>(B, C, M, rho_l); break; \
    case BICADMM_LOGISTIC: k_prox<T, BICADMM_LOGISTIC, 1><<<g, kProxThreads, 0, s>>>(B, C, M, rho_l); break; \
    case BICADMM_HINGE: k_prox<T, BICADMM_HINGE, 1><<<g, kProxThreads, 0, s>>>(B, C, M, rho_l); break; \
    default: k_prox<T, BICADMM_SOFTMAX, 16><<<g, kProxThreads, 0, s>>>(B, C, M, rho_l); break; \
    }
        if (dtype == BICADMM_F64) { BIC_PROX(double) } else { BIC_PROX(float) }
#undef BIC_PROX
        BIC_LAUNCHED();
    }
    return BICADMM_OK;
}

// Objective (1) data term: per-CTA partial sums of phi((sum_j p_j)[r], b_r)
// into sq_partial (fixed-order block sums).
template <typename T, int LOSS, int CM>
__global__ void __launch_bounds__(kProxThreads) k_loss(const __grid_constant__ ProxBatch B, int C) {
    __shared__ double scratch[32];
    const int64_t cta = blockIdx.x;
    int ni = 0;
    while (ni + 1 < B.nn && cta >= B.n[ni + 1].cta_begin) ++ni;
    const ProxNode& P = B.n[ni];
    const int64_t r = (cta - P.cta_begin) * kProxThreads + threadIdx.x;
    double f = 0.0;
    if (r < P.m) {
        const double bl = (double)static_cast<const T*>(P.b)[r];
        double w[CM];
        for (int c = 0; c < C; ++c) {
            double S = 0.0;
            if (P.S) S = P.S[r * C + c];
            else for (int j = 0; j < P.np; ++j) S += P.p[j * P.pstride + r * C + c];
            w[c] = S;
        }
        if constexpr (LOSS == BICADMM_LS) { const double e = w[0] - bl; f = e * e; }
        else if constexpr (LOSS == BICADMM_LOGISTIC) {
            const double a = -bl * w[0];
            f = a > 0.0 ? a + log1p(exp(-a)) : log1p(exp(a));
        } else if constexpr (LOSS == BICADMM_HINGE) { f = fmax(0.0, 1.0 - bl * w[0]); }
        else {
            double mx = -INFINITY, se = 0.0;
            for (int c = 0; c < C; ++c) mx = fmax(mx, w[c]);
            for (int c = 0; c < C; ++c) se += exp(w[c] - mx);
            f = mx + log(se) - w[(int)bl];
        }
    }
    const double s = block_sum(f, scratch);
    if (threadIdx.x == 0) P.sq_partial[cta - P.cta_begin] = s;
}

int launch_loss(int loss, int dtype, int C, ProxNode* nodes, int nn, cudaStream_t s) {
    for (int base = 0; base < nn; base += kMaxDesc) {
        ProxBatch B;
        B.nn = nn - base < kMaxDesc ? nn - base : kMaxDesc;
        int64_t t = 0;
        for (int k = 0; k < B.nn; ++k) {
            B.n[k] = nodes[base + k];
            B.n[k].cta_begin = t;
            t += (B.n[k].m + kProxThreads - 1) / kProxThreads;
        }
        if (t == 0) continue;
        const unsigned g = (unsigned)t;
#define BIC_LOSS(T)                                                                          \
    switch (loss) {                                                                          \
    case BICADMM_LS: k_loss<T, BICADMM_LS, 1><<<g, kProxThreads, 0, s>>>(B, C); break;       \
    case BICADMM_LOGISTIC: k_loss<T, BICADMM_LOGISTIC, 1><<<g, kProxThreads, 0, s>>>(B, C); break; \
    case BICADMM_HINGE: k_loss<T, BICADMM_HINGE, 1><<<g, kProxThreads, 0, s>>>(B, C); break; \
    default: k_loss<T, BICADMM_SOFTMAX, 16><<<g, kProxThreads, 0, s>>>(B, C); break;          \
    }
        if (dtype == BICADMM_F64) { BIC_LOSS(double) } else { BIC_LOSS(float) }
#undef BIC_LOSS
        BIC_LAUNCHED();
    }
    return BICADMM_OK;
}

// S_out[k][r] = sum over the node's local blocks (ascending) of p  -- the local
// contribution handed to the cross-GPU AllReduce (Algorithm 2).
__global__ void __launch_bounds__(256) k_psum(const __grid_constant__ ProxBatch B, double* const* S_out_dev_unused,
                                              int C) {
    (void)S_out_dev_unused;
    const int64_t cta = blockIdx.x;
    int ni = 0;
    while (ni + 1 < B.nn && cta >= B.n[ni + 1].cta_begin) ++ni;
    const ProxNode& P = B.n[ni];
    const int64_t e = (cta - P.cta_begin) * 256 + threadIdx.x;
    if (e >= P.m * C) return;
    double S = 0.0;
    for (int j = 0; j < P.np; ++j) S += P.p[j * P.pstride + e];
    const_cast<double*>(P.S)[e] = S;
}

int launch_psum(int C, ProxNode* nodes, int nn, double* const* /*S_out*/, cudaStream_t s) {
    for (int base = 0; base < nn; base += kMaxDesc) {
        ProxBatch B;
        B.nn = nn - base < kMaxDesc ? nn - base : kMaxDesc;
        int64_t t = 0;
        for (int k = 0; k < B.nn; ++k) {
            B.n[k] = nodes[base + k];
            B.n[k].cta_begin = t;
            t += (B.n[k].m * C + 255) / 256;
        }
        if (t == 0) continue;
        k_psum<<<(unsigned)t, 256, 0, s>>>(B, nullptr, C);
        BIC_LAUNCHED();
    }
    return BICADMM_OK;
}

}  // namespace bic

namespace bic {

// ----------------------------------------------------------------------------- small nodes
// Whole inner loops of small nodes in one CTA each (configs[0]-sized problems are launch-
// bound: ~70 graph launches per outer iteration, 3 us each).  The node's blocks A_ij and
// their factors H_ij are staged into shared memory once; then K sweeps of Eqs. (22)-(24),
// each: q_j = p_j + delta; r_j = rho_l A_j^T q_j + rho_c (z_j - u_j); x_j = H_j r_j;
// p_j = A_j x_j; per sample S = sum_j p_j, abar = S / M, omega = prox(abar + nu) (22),
// nu += abar - omega (23), delta = omega - abar - nu -- the same algebra, state and prox
// functions as the two-pass sweep, every sum sequential in a fixed order.
constexpr int kSmallBatchNodes = 24;   // nodes per launch (kernel parameter space: 32 KB)
constexpr int kSmallThreads = kSmallMaxCols;   // one CTA per node (512 and 1024 measured no faster)
struct SmallSweepBatch {
    SmallNode n[kSmallBatchNodes];
    int nn;
};

__device__ __forceinline__ double small_h(const SmallBlock& B, int64_t r, int64_t c, bool f64) {
    if (B.hpack) {   // lower 64 x 64 tiles, tile (I, J), I >= J, at I(I+1)/2 + J (k_symv.cu)
        if (r < c) { const int64_t t = r; r = c; c = t; }
        const int64_t I = r >> 6, J = c >> 6, e = (I * (I + 1) / 2 + J) * 4096 + (r & 63) * 64 + (c & 63);
        return f64 ? static_cast<const double*>(B.H)[e] : (double)static_cast<const float*>(B.H)[e];
    }
    const int64_t e = r * B.ldh + c;
    return f64 ? static_cast<const double*>(B.H)[e] : (double)static_cast<const float*>(B.H)[e];
}

template <typename T, int LOSS>
__global__ void __launch_bounds__(kSmallThreads) k_small_sweeps(const __grid_constant__ SmallSweepBatch SB, const double* z, int K,
                                                      int M, double rho_l, double rho_c) {
    extern __shared__ double sm[];
    const SmallNode& N = SB.n[blockIdx.x];
    // 32-bit indices: everything below lives in one CTA's shared memory (< 2^15 doubles)
    const int m = (int)N.m, n = (int)N.ncols;
    const int nb = N.nb;
    // shared layout: A (m x n, blocks side by side), H_j (n_j x n_j each), z - u (n), r (n),
    // x (n), p (nb x m), nu, delta, omega, b (m)
    double* As = sm;
    // row strides padded to an odd number of doubles: lanes walking rows (the A x and H r
    // products) then hit distinct bank pairs (an even stride such as 50 is a 4-way conflict)
    const int lda = n | 1;
    double* Hs = As + m * lda;
    int hoff[kSmallMaxBlocks], bcs[kSmallMaxBlocks + 1];
    int hsz = 0;
    for (int j = 0; j < nb; ++j) {
        hoff[j] = hsz;
        hsz += (int)(N.blk[j].nj * (N.blk[j].nj | 1));
        bcs[j] = (int)N.blk[j].cs;
    }
    bcs[nb] = n;
    double* zu = Hs + hsz;
    double* rs = zu + n;
    double* xs = rs + n;
    double* ps = xs + n;
    double* nus = ps + nb * m;
    double* dls = nus + m;
    double* oms = dls + m;
    double* bs = oms + m;
    const int tid = threadIdx.x, nt = blockDim.x;
    const bool f64 = sizeof(T) == 8;
    // staging: 8 independent global loads per thread in flight before their shared stores
    // (a load -> store chain per element costs one L2/HBM latency each: ~10 us per launch)
    constexpr int U = 8;
    for (int j = 0; j < nb; ++j) {
        const SmallBlock& B = N.blk[j];
        const T* A = static_cast<const T*>(B.A);
        const int nj = (int)B.nj, cs = bcs[j];
        for (int e0 = 0; e0 < m * nj; e0 += U * nt) {
            double v[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int e = e0 + k * nt + tid;
                v[k] = e < m * nj ? (double)A[(int64_t)(e / nj) * B.lda + e % nj] : 0.0;
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int e = e0 + k * nt + tid;
                if (e < m * nj) As[(e / nj) * lda + cs + e % nj] = v[k];
            }
        }
        for (int e0 = 0; e0 < nj * nj; e0 += U * nt) {
            double v[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int e = e0 + k * nt + tid;
                v[k] = e < nj * nj ? small_h(B, e / nj, e % nj, f64) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int e = e0 + k * nt + tid;
                if (e < nj * nj) Hs[hoff[j] + (e / nj) * (nj | 1) + e % nj] = v[k];
            }
        }
        for (int l = tid; l < nj; l += nt) {
            zu[cs + l] = z[B.c0 + l] - B.u[l];
            xs[cs + l] = B.x[l];
        }
        for (int r = tid; r < m; r += nt) ps[j * m + r] = B.p[r];
    }
    for (int r = tid; r < m; r += nt) {
        nus[r] = N.nu[r];
        dls[r] = N.delta[r];
        oms[r] = N.omega ? N.omega[r] : 0.0;
        bs[r] = (double)static_cast<const T*>(N.b)[r];
    }
    __syncthreads();
    const double Md = (double)M;
    // every product splits its inner length over S = nt / outputs threads (partials in a
    // [S][outputs] scratch, then summed by the output's thread in ascending split order)
    double* part = bs + m;   // scratch: max(n, m) * ns doubles (small_sweep_smem_bytes)
    const int ns = N.nsplit;
    const int nsm = N.nsplit_m;
    auto block_of = [&](int l) {
        int j = 0;
        while (j + 1 < nb && l >= bcs[j + 1]) ++j;
        return j;
    };
    // Per-thread work, fixed for all K sweeps (hoisted: the index arithmetic was ~40 % of the
    // instructions of a sweep).  Column phases: n <= kSmallThreads (build_small), so a thread
    // owns at most one (column, split) slice.  Row phase: the first (row, split) item here,
    // further items (nb m nsm > kSmallThreads) computed in the loop.
    const bool colw = tid < n * ns;
    const int cl = colw ? tid % n : 0, csp = colw ? tid / n : 0;
    const int cj = block_of(cl);
    const int cr0 = m * csp / ns, cr1 = m * (csp + 1) / ns;
    const int hnj = bcs[cj + 1] - bcs[cj];
    const int hc0 = hnj * csp / ns, hc1 = hnj * (csp + 1) / ns;
    const double* aT = As + cl;
    const double* pT = ps + cj * m;
    const double* Hrow = Hs + hoff[cj] + (cl - bcs[cj]) * (hnj | 1);
    const double* rj = rs + bcs[cj];
    const int nbm = nb * m;
    struct RowItem { int o, sp, c0, c1; const double* a; const double* x; };
    auto row_item = [&](int e) {
        RowItem it;
        it.o = e % nbm;
        it.sp = e / nbm;
        const int j = it.o / m, r = it.o % m;
        const int nj = bcs[j + 1] - bcs[j];
        it.c0 = nj * it.sp / nsm;
        it.c1 = nj * (it.sp + 1) / nsm;
        it.a = As + r * lda + bcs[j];
        it.x = xs + bcs[j];
        return it;
    };
    const RowItem ri0 = row_item(tid);
    for (int s = 0; s < K; ++s) {
        // r = rho_l A^T (p + delta) + rho_c (z - u): outputs = columns, inner = rows
        if (colw) {
            double acc = 0.0;
#pragma unroll 4
            for (int r = cr0; r < cr1; ++r) acc = fma(aT[r * lda], pT[r] + dls[r], acc);
            part[csp * n + cl] = acc;
        }
        __syncthreads();
        if (tid < n) {
            double acc = 0.0;
            for (int sp = 0; sp < ns; ++sp) acc += part[sp * n + tid];
            rs[tid] = rho_l * acc + rho_c * zu[tid];
        }
        __syncthreads();
        // x_j = H_j r_j: outputs = the block's rows, inner = its columns
        if (colw) {
            double acc = 0.0;
#pragma unroll 4
            for (int c = hc0; c < hc1; ++c) acc = fma(Hrow[c], rj[c], acc);
            part[csp * n + cl] = acc;
        }
        __syncthreads();
        if (tid < n) {
            double acc = 0.0;
            for (int sp = 0; sp < ns; ++sp) acc += part[sp * n + tid];
            xs[tid] = acc;
        }
        __syncthreads();
        // p_j = A_j x_j: outputs = (block, row), inner = the block's columns
        for (int e = tid; e < nbm * nsm; e += nt) {
            const RowItem it = e == tid ? ri0 : row_item(e);
            double acc = 0.0;
#pragma unroll 4
            for (int c = it.c0; c < it.c1; ++c) acc = fma(it.a[c], it.x[c], acc);
            part[it.sp * nbm + it.o] = acc;
        }
        __syncthreads();
        // block sums and the per-sample prox (22)-(23): one thread per row
        for (int r = tid; r < m; r += nt) {
            double S = 0.0;
            for (int j = 0; j < nb; ++j) {
                double acc = 0.0;
                for (int sp = 0; sp < nsm; ++sp) acc += part[sp * nbm + j * m + r];
                ps[j * m + r] = acc;
                S += acc;
            }
            const double abar = S / Md, pa = abar + nus[r];
            double om;
            if constexpr (LOSS == BICADMM_LS) om = (2.0 * bs[r] + rho_l * pa) / (2.0 * Md + rho_l);
            else if constexpr (LOSS == BICADMM_LOGISTIC) om = prox_logistic(M, rho_l, bs[r], pa, N.omega ? oms[r] : pa);
            else om = prox_hinge(M, rho_l, bs[r], pa);
            const double nu = nus[r] + abar - om;
            nus[r] = nu;
            dls[r] = om - abar - nu;
            oms[r] = om;
        }
        __syncthreads();
    }
    for (int j = 0; j < nb; ++j) {
        const SmallBlock& B = N.blk[j];
        const int nj = (int)B.nj, cs = bcs[j];
        for (int l = tid; l < nj; l += nt) {
            B.x[l] = xs[cs + l];
            B.r[l] = rs[cs + l];
        }
        for (int r = tid; r < m; r += nt) B.p[r] = ps[j * m + r];
    }
    for (int r = tid; r < m; r += nt) {
        N.nu[r] = nus[r];
        N.delta[r] = dls[r];
        if (N.omega) N.omega[r] = oms[r];
    }
}

size_t small_sweep_smem_bytes(const SmallNode& N) {
    int64_t hsz = 0;
    for (int j = 0; j < N.nb; ++j) hsz += N.blk[j].nj * (N.blk[j].nj | 1);   // odd row strides
    const int64_t scratch = std::max<int64_t>(N.ncols * N.nsplit, (int64_t)N.nb * N.m * N.nsplit_m);
    return sizeof(double) * (size_t)(N.m * (N.ncols | 1) + hsz + 3 * N.ncols + N.nb * N.m + 4 * N.m + scratch);
}
// splits of the inner length per output (kSmallThreads threads per CTA)
void small_sweep_plan(SmallNode& N) {
    N.nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(16, kSmallThreads / std::max<int64_t>(1, N.ncols)));
    N.nsplit_m = (int)std::max<int64_t>(1, std::min<int64_t>(16, kSmallThreads / std::max<int64_t>(1, (int64_t)N.nb * N.m)));
}

int launch_small_sweeps(int loss, int dtype, const SmallNode* nodes, int nn, const double* z, int K, int M,
                        double rho_l, double rho_c, cudaStream_t s) {
    if (loss == BICADMM_SOFTMAX) return BICADMM_ERR_INVALID;
    for (int base = 0; base < nn; base += kSmallBatchNodes) {
        SmallSweepBatch B;
        B.nn = nn - base < kSmallBatchNodes ? nn - base : kSmallBatchNodes;
        size_t smem = 0;
        for (int k = 0; k < B.nn; ++k) {
            B.n[k] = nodes[base + k];
            smem = smem > small_sweep_smem_bytes(B.n[k]) ? smem : small_sweep_smem_bytes(B.n[k]);
        }
        if (smem > kSmallSmemMax) return BICADMM_ERR_INVALID;
#define BIC_SMALL(T, L)                                                                                      \
    {                                                                                                        \
        static bool set = false;                                                                             \
        if (!set) {                                                                                          \
            if (cudaFuncSetAttribute(k_small_sweeps<T, L>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                                     (int)kSmallSmemMax) != cudaSuccess)                                     \
                return BICADMM_ERR_CUDA;                                                                     \
            set = true;                                                                                      \
        }                                                                                                    \
        k_small_sweeps<T, L><<<B.nn, kSmallThreads, smem, s>>>(B, z, K, M, rho_l, rho_c);                              \
    }
        if (dtype == BICADMM_F64) {
            if (loss == BICADMM_LS) BIC_SMALL(double, BICADMM_LS)
            else if (loss == BICADMM_LOGISTIC) BIC_SMALL(double, BICADMM_LOGISTIC)
            else BIC_SMALL(double, BICADMM_HINGE)
        } else {
            if (loss == BICADMM_LS) BIC_SMALL(float, BICADMM_LS)
            else if (loss == BICADMM_LOGISTIC) BIC_SMALL(float, BICADMM_LOGISTIC)
            else BIC_SMALL(float, BICADMM_HINGE)
        }
#undef BIC_SMALL
        BIC_LAUNCHED();
    }
    return BICADMM_OK;
}

}  // namespace bic
