// k_factor.cu -- one-time block factor of the x-update.
//
// Eq. (24)'s x_ij-step is the ridge least-squares problem whose normal equations
// (DESIGN R17) are  (rho_l A_ij^T A_ij + c I) x = rho_l A_ij^T q + rho_c (z_j - u_ij),
// c = 1/(N gamma) + rho_c.  We build H_ij = F^{-1} explicitly once, so every sweep's
// solve is one more HBM-streamed GEMV (a3) instead of two latency-bound
// triangular solves:
//   G = A^T A                       (FP64 tensor-core DMMA tiles, SASS DMMA.8x8x4)
//   F = rho_l G + c I;  F = L L^T   (right-looking blocked Cholesky, nb = 64)
//   W = L^{-1}                      (blocked forward substitution, GEMM-shaped)
//   H = W^T W                       (DMMA, triangular K range, mirrored)
// FP64 tensor cores exist on sm_100a only as mma.sync DMMA; tcgen05 has no f64
// kind.  In FP32 mode the factor is still built in FP64 and H rounded once.
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace bic {

constexpr int BM = 64, BN = 64, BK = 16, PAD = 4;
constexpr int kGemmThreads = 128;

struct GemmArgs {
    int64_t M, N, K;
    double alpha, beta, diag;
    const void* A; int64_t lda;
    const void* B; int64_t ldb;
    void* C; int64_t ldc;
    int lower_only;   // skip tiles strictly above the diagonal
    int mirror;       // also write the transpose into the upper triangle
    int tri_k;        // K range starts at max(m0, n0) (lower-triangular operands)
    // Triangular operands whose zero half is skipped tile by tile (the skipped products are
    // exact zeros, so the result is bit-identical to the full product):
    int k_lo;         // 0: K from 0; 1: A(i,k) = 0 for k < i -> from m0; 2: B(k,j) = 0 for k < j -> from n0
    int k_hi;         // 0: K to K; 1: A(i,k) = 0 for k > i -> to m0 + BM; 2: B(k,j) = 0 for k > j -> to n0 + BN
};

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// A(i, k): A_KFAST -> A[i*lda + k] (stored M x K), else A[k*lda + i] (stored K x M)
// B(k, j): B_KFAST -> B[j*ldb + k] (stored N x K), else B[k*ldb + j] (stored K x N)
// Up to kMaxBatch independent GEMMs per launch (blockIdx.z): the setup factors all local
// blocks of equal step count in lockstep, so the small per-step Cholesky / inverse GEMMs
// of several blocks share one launch.
constexpr int kMaxBatch = 8;
struct GemmBatch {
    GemmArgs g[kMaxBatch];
    int n;
};

template <typename TIN, typename TOUT, bool A_KFAST, bool B_KFAST>
__global__ void __launch_bounds__(kGemmThreads) k_gemm_dmma(const __grid_constant__ GemmBatch bt) {
    __shared__ double As[2][BK][BM + PAD];
    __shared__ double Bs[2][BK][BN + PAD];
    const GemmArgs& g = bt.g[blockIdx.z];
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
    if (m0 >= g.M || n0 >= g.N) return;
    if (g.lower_only && n0 > m0 + BM - 1) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 1, wn = warp & 1;
    const int grp = lane >> 2, tig = lane & 3;
    const TIN* A = static_cast<const TIN*>(g.A);
    const TIN* B = static_cast<const TIN*>(g.B);

    int64_t kb = 0;
    if (g.tri_k) kb = (m0 > n0 ? m0 : n0) / BK * BK;
    if (g.k_lo == 1) kb = m0 / BK * BK;
    if (g.k_lo == 2) kb = n0 / BK * BK;
    int64_t K = g.K;
    if (g.k_hi == 1 && m0 + BM < K) K = m0 + BM;
    if (g.k_hi == 2 && n0 + BN < K) K = n0 + BN;

    double regA[8], regB[8];
    auto gload = [&](int64_t k0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int idx = tid + kGemmThreads * e;
            int ii, kk;
            if (A_KFAST) { ii = idx >> 4; kk = idx & 15; } else { kk = idx >> 6; ii = idx & 63; }
            const int64_t gi = m0 + ii, gk = k0 + kk;
            double v = 0.0;
            if (gi < g.M && gk < K) v = (double)(A_KFAST ? A[gi * g.lda + gk] : A[gk * g.lda + gi]);
            regA[e] = v;
            int jj;
            if (B_KFAST) { jj = idx >> 4; kk = idx & 15; } else { kk = idx >> 6; jj = idx & 63; }
            const int64_t gj = n0 + jj, gk2 = k0 + kk;
            double w = 0.0;
            if (gj < g.N && gk2 < K) w = (double)(B_KFAST ? B[gj * g.ldb + gk2] : B[gk2 * g.ldb + gj]);
            regB[e] = w;
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int idx = tid + kGemmThreads * e;
            int ii, kk;
            if (A_KFAST) { ii = idx >> 4; kk = idx & 15; } else { kk = idx >> 6; ii = idx & 63; }
            As[buf][kk][ii] = regA[e];
            int jj;
            if (B_KFAST) { jj = idx >> 4; kk = idx & 15; } else { kk = idx >> 6; jj = idx & 63; }
            Bs[buf][kk][jj] = regB[e];
        }
    };

    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    if (kb < K) {
        gload(kb);
        sstore(0);
        __syncthreads();
        int buf = 0;
        for (int64_t k0 = kb; k0 < K; k0 += BK) {
            const bool more = k0 + BK < K;
            if (more) gload(k0 + BK);
#pragma unroll
            for (int ks = 0; ks < BK; ks += 4) {
                double af[4], bf[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    af[t] = As[buf][ks + tig][wm * 32 + t * 8 + grp];
                    bf[t] = Bs[buf][ks + tig][wn * 32 + t * 8 + grp];
                }
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
            }
            if (more) {
                sstore(buf ^ 1);
                __syncthreads();
                buf ^= 1;
            }
        }
    }
    TOUT* C = static_cast<TOUT*>(g.C);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t i = m0 + wm * 32 + a * 8 + grp;
                const int64_t j = n0 + wn * 32 + b * 8 + tig * 2 + h;
                if (i >= g.M || j >= g.N) continue;
                double v = g.alpha * acc[a][b][h];
                if (g.beta != 0.0) v += g.beta * (double)C[i * g.ldc + j];
                if (i == j) v += g.diag;
                C[i * g.ldc + j] = (TOUT)v;
                if (g.mirror && i > j) C[j * g.ldc + i] = (TOUT)v;
            }
}

template <typename TIN, typename TOUT, bool AK, bool BK_>
static int gemm_batched(const GemmArgs* gs, int n, cudaStream_t s) {
    GemmBatch bt{};
    bt.n = 0;
    int64_t mx = 0, nx = 0;
    for (int k = 0; k < n; ++k) {
        if (gs[k].M <= 0 || gs[k].N <= 0) continue;
        bt.g[bt.n++] = gs[k];
        mx = gs[k].M > mx ? gs[k].M : mx;
        nx = gs[k].N > nx ? gs[k].N : nx;
    }
    if (bt.n == 0) return BICADMM_OK;
    dim3 grid((unsigned)((nx + BN - 1) / BN), (unsigned)((mx + BM - 1) / BM), (unsigned)bt.n);
    k_gemm_dmma<TIN, TOUT, AK, BK_><<<grid, kGemmThreads, 0, s>>>(bt);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

template <typename TIN, typename TOUT, bool AK, bool BK_>
static int gemm(const GemmArgs& g, cudaStream_t s) {
    return gemm_batched<TIN, TOUT, AK, BK_>(&g, 1, s);
}

int launch_gram(int dtype, int64_t m, int64_t nj, const void* A, int64_t lda, double alpha, double diag,
                double* G, int64_t ldg, bool full, cudaStream_t s) {
    GemmArgs g{};
    g.M = nj; g.N = nj; g.K = m;
    g.alpha = alpha; g.beta = 0.0; g.diag = diag;
    g.A = A; g.lda = lda; g.B = A; g.ldb = lda; g.C = G; g.ldc = ldg;
    g.lower_only = 1; g.mirror = full ? 1 : 0; g.tri_k = 0;
    // A^T A: A(i,k) = A[k*lda + i] (stored K x M), B(k,j) = A[k*lda + j] (stored K x N)
    if (dtype == BICADMM_F64) return gemm<double, double, false, false>(g, s);
    return gemm<float, double, false, false>(g, s);
}

int launch_gram_rows(int dtype, int64_t m, int64_t nj, const void* A, int64_t lda, double alpha, double diag,
                     double* G, int64_t ldg, cudaStream_t s) {
    GemmArgs g{};
    g.M = m; g.N = m; g.K = nj;
    g.alpha = alpha; g.beta = 0.0; g.diag = diag;
    g.A = A; g.lda = lda; g.B = A; g.ldb = lda; g.C = G; g.ldc = ldg;
    g.lower_only = 1; g.mirror = 0; g.tri_k = 0;
    // A A^T: A(i,k) = A[i*lda + k] (stored M x K), B(k,j) = A[j*lda + k] (stored N x K)
    if (dtype == BICADMM_F64) return gemm<double, double, true, true>(g, s);
    return gemm<float, double, true, true>(g, s);
}

// ------------------------------------------------------------------ Cholesky diag block
// One CTA factors the kn x kn diagonal block (kn <= 64) of F in place (lower, upper
// zeroed) and writes W_kk = L_kk^{-1} (lower) into Wd.  Unblocked right-looking
// Cholesky in shared memory with the inverse formed by the same elimination steps.
constexpr int NB = 64;
constexpr int kDiagThreads = 256;

struct DiagBatch {
    double* F[kMaxBatch];
    double* Wd[kMaxBatch];
    int64_t ldf[kMaxBatch], ldw[kMaxBatch];
    int kn[kMaxBatch];
    int* info[kMaxBatch];
};

__global__ void __launch_bounds__(kDiagThreads) k_chol_diag(const __grid_constant__ DiagBatch db) {
    double* F = db.F[blockIdx.x];
    double* Wd = db.Wd[blockIdx.x];
    const int64_t ldf = db.ldf[blockIdx.x], ldw = db.ldw[blockIdx.x];
    const int kn = db.kn[blockIdx.x];
    int* info = db.info[blockIdx.x];
    extern __shared__ double sm[];
    double (*L)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(sm);
    double (*W)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(sm + NB * (NB + 1));
    const int tid = threadIdx.x;
    for (int e = tid; e < kn * kn; e += kDiagThreads) {
        const int i = e / kn, j = e % kn;
        L[i][j] = j <= i ? F[i * ldf + j] : 0.0;
        W[i][j] = i == j ? 1.0 : 0.0;
    }
    __syncthreads();
    // Right-looking Cholesky with the inverse built alongside by the same row operations
    // on [L | I] (forward elimination): step j scales column j of L and row j of W by
    // 1/sqrt(d_j), then subtracts L[i][j] x (row j) from rows i > j of both.  Two barriers
    // per column; 16 x 16 thread grid over the update regions.
    const int tx = tid & 15, ty = tid >> 4;
    for (int j = 0; j < kn; ++j) {
        double d = L[j][j];
        if (!(d > 0.0)) {
            if (tid == 0) atomicExch(info, 1);
            d = 1.0;
        }
        const double rl = 1.0 / sqrt(d);
        __syncthreads();   // every thread has read the pivot before it is overwritten
        if (tid < 64) {
            const int i = j + tid;
            if (i < kn) L[i][j] = i == j ? sqrt(d) : L[i][j] * rl;
        } else if (tid < 128) {
            const int c = tid - 64;
            if (c <= j) W[j][c] *= rl;
        }
        __syncthreads();
        for (int i = j + 1 + ty; i < kn; i += 16) {
            const double lij = L[i][j];
            for (int k = j + 1 + tx; k <= i; k += 16) L[i][k] -= lij * L[k][j];
            for (int c = tx; c <= j; c += 16) W[i][c] -= lij * W[j][c];
        }
        __syncthreads();
    }
    for (int e = tid; e < kn * kn; e += kDiagThreads) {
        const int i = e / kn, j = e % kn;
        F[i * ldf + j] = j <= i ? L[i][j] : 0.0;
        Wd[i * ldw + j] = j <= i ? W[i][j] : 0.0;
    }
}

static int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

size_t factor_ws_doubles(int64_t nj) {
    const int64_t ld = round_up(nj, 8);
    // W (nj x ld), the recursion's panel scratch (<= (nj/2 + NB) x ld), info
    return (size_t)(ld * nj + (nj / 2 + NB + 8) * ld + 8);
}

// ------------------------------------------------------------------ recursive factor
// chol_inv(F, n) -> L (in F, lower) and W = L^{-1} (in W), all jobs in lockstep (equal n):
//   n <= NB : k_chol_diag
//   else    : n1 = NB * ceil(n / 2 / NB), n2 = n - n1
//             (L11, W11) = chol_inv(F11)
//             L21 = F21 W11^T                (GEMM, via scratch X)
//             F22 -= L21 L21^T               (lower tiles)
//             (L22, W22) = chol_inv(F22)
//             W21 = -W22 (L21 W11)           (two GEMMs, via X)
// The same flops as the blocked right-looking factor + blocked inverse, but in GEMMs of
// size n/2, n/4, ... instead of rank-64 updates (which are bound by the C read/write).
struct RecJob {
    double* F;   // job's F at (0, 0), leading dim ldf
    int64_t ldf;
    double* W;   // job's W at (0, 0), leading dim ldw
    int64_t ldw;
    double* X;   // scratch (>= (n/2 + NB) x ldw)
    int* info;
};

// Large products of the recursion go to the tcgen05 Ozaki engine (k_gram_tc.cu: FP64-accurate,
// ~2x the DMMA rate at these sizes), one job at a time through the shared scratch; the small
// ones stay on the batched DMMA kernel.  Structural zeros (k_lo / k_hi / tri_k) are skipped
// exactly on both paths.
struct FactorTc {
    void* ws = nullptr;
    size_t bytes = 0;
};
constexpr double kTcMinVolume = 8.0e9;   // M N K (~2000^3): below it the DMMA batch wins

template <bool AK, bool BK_>
static int gemm_factor(const GemmArgs* ga, int nj, const FactorTc* tc, cudaStream_t s) {
    const GemmArgs& g0 = ga[0];
    if (tc && tc->ws && (double)g0.M * (double)g0.N * (double)g0.K >= kTcMinVolume &&
        gemm_tc_scratch_bytes(g0.M, g0.N, g0.K, false) <= tc->bytes) {
        for (int k = 0; k < nj; ++k) {
            const GemmArgs& g = ga[k];
            OzGemm o{};
            o.M = g.M; o.N = g.N; o.K = g.K;
            o.A = g.A;
            o.a_sl = AK ? g.lda : 1; o.a_sr = AK ? 1 : g.lda;      // A(i,k): AK -> A[i lda + k]
            o.B = g.B;
            o.b_sl = BK_ ? g.ldb : 1; o.b_sr = BK_ ? 1 : g.ldb;    // B(k,j): BK -> B[j ldb + k]
            o.same = o.A == o.B && o.a_sl == o.b_sl && o.a_sr == o.b_sr;
            o.dtype = BICADMM_F64;
            o.alpha = g.alpha; o.beta = g.beta; o.diag = g.diag; o.C = static_cast<double*>(g.C); o.ldc = g.ldc;
            o.lower = g.lower_only; o.mirror = g.mirror;
            o.k_lo = g.tri_k ? 3 : g.k_lo; o.k_hi = g.k_hi;
            const int rc = launch_gemm_tc(o, tc->ws, tc->bytes, s);
            if (rc) return rc;
        }
        return BICADMM_OK;
    }
    return gemm_batched<double, double, AK, BK_>(ga, nj, s);
}

static int chol_inv_rec(const RecJob* J, int nj, int64_t n, int64_t off, const FactorTc* tc, cudaStream_t s) {
    if (n <= NB) {
        DiagBatch db{};
        for (int k = 0; k < nj; ++k) {
            db.F[k] = J[k].F + off * J[k].ldf + off; db.ldf[k] = J[k].ldf;
            db.Wd[k] = J[k].W + off * J[k].ldw + off; db.ldw[k] = J[k].ldw;
            db.kn[k] = (int)n; db.info[k] = J[k].info;
        }
        k_chol_diag<<<nj, kDiagThreads, sizeof(double) * 2 * NB * (NB + 1), s>>>(db);
        BIC_LAUNCHED();
        return BICADMM_OK;
    }
    int64_t n1 = (n / 2 + NB - 1) / NB * NB;
    if (n1 >= n) n1 = n - NB;
    const int64_t n2 = n - n1;
    int rc = chol_inv_rec(J, nj, n1, off, tc, s);
    if (rc) return rc;
    GemmArgs ga[kMaxBatch];
    // X = F21 W11^T  (n2 x n1 x n1): A(i,k) = F21[i][k] (K-fast), B(k,j) = W11[j][k] (K-fast)
    for (int k = 0; k < nj; ++k) {
        GemmArgs g{};
        g.M = n2; g.N = n1; g.K = n1; g.alpha = 1.0; g.beta = 0.0; g.diag = 0.0;
        g.A = J[k].F + (off + n1) * J[k].ldf + off; g.lda = J[k].ldf;
        g.B = J[k].W + off * J[k].ldw + off; g.ldb = J[k].ldw;
        g.C = J[k].X; g.ldc = J[k].ldw; g.k_hi = 2;
        ga[k] = g;
    }
    rc = gemm_factor<true, true>(ga, nj, tc, s);
    if (rc) return rc;
    for (int k = 0; k < nj; ++k)   // L21 = X
        BIC_CUDA(cudaMemcpy2DAsync(J[k].F + (off + n1) * J[k].ldf + off, sizeof(double) * J[k].ldf, J[k].X,
                                   sizeof(double) * J[k].ldw, sizeof(double) * n1, n2, cudaMemcpyDeviceToDevice, s));
    // F22 -= L21 L21^T (lower tiles): A(i,k) = L21[i][k], B(k,j) = L21[j][k]
    for (int k = 0; k < nj; ++k) {
        GemmArgs g{};
        g.M = n2; g.N = n2; g.K = n1; g.alpha = -1.0; g.beta = 1.0; g.diag = 0.0;
        g.A = J[k].F + (off + n1) * J[k].ldf + off; g.lda = J[k].ldf;
        g.B = g.A; g.ldb = J[k].ldf;
        g.C = J[k].F + (off + n1) * J[k].ldf + off + n1; g.ldc = J[k].ldf; g.lower_only = 1;
        ga[k] = g;
    }
    rc = gemm_factor<true, true>(ga, nj, tc, s);
    if (rc) return rc;
    rc = chol_inv_rec(J, nj, n2, off + n1, tc, s);
    if (rc) return rc;
    // X = L21 W11 (n2 x n1 x n1): A(i,k) = L21[i][k], B(k,j) = W11[k][j] (N-fast)
    for (int k = 0; k < nj; ++k) {
        GemmArgs g{};
        g.M = n2; g.N = n1; g.K = n1; g.alpha = 1.0; g.beta = 0.0; g.diag = 0.0;
        g.A = J[k].F + (off + n1) * J[k].ldf + off; g.lda = J[k].ldf;
        g.B = J[k].W + off * J[k].ldw + off; g.ldb = J[k].ldw;
        g.C = J[k].X; g.ldc = J[k].ldw; g.k_lo = 2;
        ga[k] = g;
    }
    rc = gemm_factor<true, false>(ga, nj, tc, s);
    if (rc) return rc;
    // W21 = -W22 X (n2 x n1 x n2): A(i,k) = W22[i][k], B(k,j) = X[k][j]
    for (int k = 0; k < nj; ++k) {
        GemmArgs g{};
        g.M = n2; g.N = n1; g.K = n2; g.alpha = -1.0; g.beta = 0.0; g.diag = 0.0;
        g.A = J[k].W + (off + n1) * J[k].ldw + off + n1; g.lda = J[k].ldw;
        g.B = J[k].X; g.ldb = J[k].ldw;
        g.C = J[k].W + (off + n1) * J[k].ldw + off; g.ldc = J[k].ldw; g.k_hi = 1;
        ga[k] = g;
    }
    return gemm_factor<true, false>(ga, nj, tc, s);
}

size_t factor_tc_scratch_bytes(int64_t n) { return gemm_tc_scratch_bytes(n, n, n, false); }

static bool factor_rec_enabled() {
    static const bool on = [] { const char* e = getenv("BICADMM_FACTOR_REC"); return !(e && atoi(e) == 0); }();
    return on;
}

static int factor_inverse_rec(const FactorJob* jobs, int njobs, const FactorTc* tc, cudaStream_t s) {
    const int64_t n = jobs[0].n;
    const int hdtype = jobs[0].hdtype;
    RecJob J[kMaxBatch];
    for (int k = 0; k < njobs; ++k) {
        if (jobs[k].n != n || jobs[k].hdtype != hdtype) return BICADMM_ERR_INVALID;
        const int64_t ldw = round_up(n, 8);
        J[k].F = jobs[k].G; J[k].ldf = jobs[k].ldg;
        J[k].W = jobs[k].ws; J[k].ldw = ldw;
        J[k].X = jobs[k].ws + ldw * n;
        J[k].info = reinterpret_cast<int*>(J[k].X + (n / 2 + NB + 8) * ldw);
        BIC_CUDA(cudaMemsetAsync(J[k].W, 0, sizeof(double) * (size_t)(ldw * n), s));
        BIC_CUDA(cudaMemsetAsync(J[k].info, 0, sizeof(int), s));
    }
    static bool attr_set = false;
    if (!attr_set) {
        BIC_CUDA(cudaFuncSetAttribute(k_chol_diag, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(sizeof(double) * 2 * NB * (NB + 1))));
        attr_set = true;
    }
    int rc = chol_inv_rec(J, njobs, n, 0, tc, s);
    if (rc) return rc;
    GemmArgs ga[kMaxBatch];
    for (int k = 0; k < njobs; ++k) {   // H = W^T W (W lower: K range from max(m0, n0)); lower tiles mirrored
        GemmArgs g{};
        g.M = n; g.N = n; g.K = n; g.alpha = 1.0; g.beta = 0.0; g.diag = 0.0;
        g.A = J[k].W; g.lda = J[k].ldw; g.B = J[k].W; g.ldb = J[k].ldw; g.C = jobs[k].H; g.ldc = jobs[k].ldh;
        g.lower_only = 1; g.mirror = 1; g.tri_k = 1;
        ga[k] = g;
    }
    rc = hdtype == BICADMM_F64 ? gemm_factor<false, false>(ga, njobs, tc, s)
                               : gemm_batched<double, float, false, false>(ga, njobs, s);
    if (rc) return rc;
    int hinfo[kMaxBatch] = {};
    for (int k = 0; k < njobs; ++k) BIC_CUDA(cudaMemcpyAsync(&hinfo[k], J[k].info, sizeof(int), cudaMemcpyDeviceToHost, s));
    BIC_CUDA(cudaStreamSynchronize(s));
    for (int k = 0; k < njobs; ++k)
        if (hinfo[k]) return BICADMM_ERR_INVALID;
    return BICADMM_OK;
}

int factor_inverse_batched(const FactorJob* jobs, int njobs, cudaStream_t s, void* tc_ws, size_t tc_bytes) {
    FactorTc tc;
    tc.ws = gram_tc_enabled() ? tc_ws : nullptr;
    tc.bytes = tc_bytes;
    if (njobs > 0 && factor_rec_enabled()) {
        // recursive (large-GEMM) variant, one lockstep batch per distinct size
        std::vector<FactorJob> rest(jobs, jobs + njobs);
        while (!rest.empty()) {
            std::vector<FactorJob> same, other;
            for (auto& j : rest) (j.n == rest[0].n && j.hdtype == rest[0].hdtype && same.size() < kMaxBatch ? same : other).push_back(j);
            const int rc = factor_inverse_rec(same.data(), (int)same.size(), &tc, s);
            if (rc) return rc;
            rest.swap(other);
        }
        return BICADMM_OK;
    }
    if (njobs <= 0) return BICADMM_OK;
    if (njobs > kMaxBatch) {
        for (int b = 0; b < njobs; b += kMaxBatch) {
            const int rc = factor_inverse_batched(jobs + b, njobs - b < kMaxBatch ? njobs - b : kMaxBatch, s);
            if (rc) return rc;
        }
        return BICADMM_OK;
    }
    const int hdtype = jobs[0].hdtype;
    for (int k = 1; k < njobs; ++k)
        if (jobs[k].hdtype != hdtype) return BICADMM_ERR_INVALID;
    int64_t ldw[kMaxBatch], nblk[kMaxBatch], nblk_max = 0;
    double *W[kMaxBatch], *X[kMaxBatch];
    int* info[kMaxBatch];
    for (int k = 0; k < njobs; ++k) {
        const int64_t nj = jobs[k].n;
        ldw[k] = round_up(nj, 8);
        W[k] = jobs[k].ws;                  // nj x ldw, lower triangular L^{-1}
        X[k] = jobs[k].ws + ldw[k] * nj;    // NB x ldw scratch
        info[k] = reinterpret_cast<int*>(X[k] + NB * ldw[k]);
        BIC_CUDA(cudaMemsetAsync(W[k], 0, sizeof(double) * (size_t)(ldw[k] * nj), s));
        BIC_CUDA(cudaMemsetAsync(info[k], 0, sizeof(int), s));
        nblk[k] = (nj + NB - 1) / NB;
        nblk_max = nblk[k] > nblk_max ? nblk[k] : nblk_max;
    }
    const size_t diag_smem = sizeof(double) * 2 * NB * (NB + 1);
    static bool attr_set = false;
    if (!attr_set) {
        BIC_CUDA(cudaFuncSetAttribute(k_chol_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)diag_smem));
        attr_set = true;
    }
    GemmArgs ga[kMaxBatch];
    // right-looking blocked Cholesky of F (lower triangle of G), all jobs in lockstep
    for (int64_t kbk = 0; kbk < nblk_max; ++kbk) {
        DiagBatch db{};
        int nd = 0;
        for (int k = 0; k < njobs; ++k) {
            if (kbk >= nblk[k]) continue;
            const int64_t k0 = kbk * NB, kn = jobs[k].n - k0 < NB ? jobs[k].n - k0 : NB;
            db.F[nd] = jobs[k].G + k0 * jobs[k].ldg + k0; db.ldf[nd] = jobs[k].ldg;
            db.Wd[nd] = W[k] + k0 * ldw[k] + k0; db.ldw[nd] = ldw[k];
            db.kn[nd] = (int)kn; db.info[nd] = info[k];
            ++nd;
        }
        k_chol_diag<<<nd, kDiagThreads, diag_smem, s>>>(db);
        BIC_LAUNCHED();
        int np = 0;
        for (int k = 0; k < njobs; ++k) {   // panel: L21 = F21 W_kk^T (in place; all K read before write)
            if (kbk >= nblk[k]) continue;
            const int64_t k0 = kbk * NB, kn = jobs[k].n - k0 < NB ? jobs[k].n - k0 : NB, rest = jobs[k].n - k0 - kn;
            if (rest <= 0) continue;
            double* F21 = jobs[k].G + (k0 + kn) * jobs[k].ldg + k0;
            GemmArgs g{};
            g.M = rest; g.N = kn; g.K = kn; g.alpha = 1.0; g.beta = 0.0; g.diag = 0.0;
            g.A = F21; g.lda = jobs[k].ldg; g.B = W[k] + k0 * ldw[k] + k0; g.ldb = ldw[k]; g.C = F21; g.ldc = jobs[k].ldg;
            ga[np++] = g;
        }
        int rc = gemm_batched<double, double, true, true>(ga, np, s);
        if (rc) return rc;
        np = 0;
        for (int k = 0; k < njobs; ++k) {   // trailing: F22 -= L21 L21^T (lower tiles)
            if (kbk >= nblk[k]) continue;
            const int64_t k0 = kbk * NB, kn = jobs[k].n - k0 < NB ? jobs[k].n - k0 : NB, rest = jobs[k].n - k0 - kn;
            if (rest <= 0) continue;
            double* F21 = jobs[k].G + (k0 + kn) * jobs[k].ldg + k0;
            GemmArgs g{};
            g.M = rest; g.N = rest; g.K = kn; g.alpha = -1.0; g.beta = 1.0; g.diag = 0.0;
            g.A = F21; g.lda = jobs[k].ldg; g.B = F21; g.ldb = jobs[k].ldg;
            g.C = jobs[k].G + (k0 + kn) * jobs[k].ldg + (k0 + kn); g.ldc = jobs[k].ldg; g.lower_only = 1;
            ga[np++] = g;
        }
        rc = gemm_batched<double, double, true, true>(ga, np, s);
        if (rc) return rc;
    }
    // W = L^{-1}: block row i:  W_i,<i = -W_ii (L_i,<i W_<i,<i)
    for (int64_t ib = 1; ib < nblk_max; ++ib) {
        int np = 0;
        for (int k = 0; k < njobs; ++k) {
            if (ib >= nblk[k]) continue;
            const int64_t i0 = ib * NB, in = jobs[k].n - i0 < NB ? jobs[k].n - i0 : NB;
            GemmArgs g{};
            g.M = in; g.N = i0; g.K = i0; g.alpha = 1.0; g.beta = 0.0; g.diag = 0.0;
            g.A = jobs[k].G + i0 * jobs[k].ldg; g.lda = jobs[k].ldg; g.B = W[k]; g.ldb = ldw[k]; g.C = X[k];
            g.ldc = ldw[k];
            ga[np++] = g;
        }
        int rc = gemm_batched<double, double, true, false>(ga, np, s);
        if (rc) return rc;
        np = 0;
        for (int k = 0; k < njobs; ++k) {
            if (ib >= nblk[k]) continue;
            const int64_t i0 = ib * NB, in = jobs[k].n - i0 < NB ? jobs[k].n - i0 : NB;
            GemmArgs g{};
            g.M = in; g.N = i0; g.K = in; g.alpha = -1.0; g.beta = 0.0; g.diag = 0.0;
            g.A = W[k] + i0 * ldw[k] + i0; g.lda = ldw[k]; g.B = X[k]; g.ldb = ldw[k]; g.C = W[k] + i0 * ldw[k];
            g.ldc = ldw[k];
            ga[np++] = g;
        }
        rc = gemm_batched<double, double, true, false>(ga, np, s);
        if (rc) return rc;
    }
    // H = W^T W  (W lower: K range from max(m0, n0)); lower tiles mirrored
    for (int k = 0; k < njobs; ++k) {
        GemmArgs g{};
        g.M = jobs[k].n; g.N = jobs[k].n; g.K = jobs[k].n; g.alpha = 1.0; g.beta = 0.0; g.diag = 0.0;
        g.A = W[k]; g.lda = ldw[k]; g.B = W[k]; g.ldb = ldw[k]; g.C = jobs[k].H; g.ldc = jobs[k].ldh;
        g.lower_only = 1; g.mirror = 1; g.tri_k = 1;
        ga[k] = g;
    }
    int rc = hdtype == BICADMM_F64 ? gemm_batched<double, double, false, false>(ga, njobs, s)
                                   : gemm_batched<double, float, false, false>(ga, njobs, s);
    if (rc) return rc;
    int hinfo[kMaxBatch] = {};
    for (int k = 0; k < njobs; ++k) BIC_CUDA(cudaMemcpyAsync(&hinfo[k], info[k], sizeof(int), cudaMemcpyDeviceToHost, s));
    BIC_CUDA(cudaStreamSynchronize(s));
    for (int k = 0; k < njobs; ++k)
        if (hinfo[k]) return BICADMM_ERR_INVALID;
    return BICADMM_OK;
}

int factor_inverse(int64_t nj, double* G, int64_t ldg, void* H, int64_t ldh, int dtype, double* ws,
                   cudaStream_t s) {
    FactorJob j{nj, G, ldg, H, ldh, dtype, ws};
    return factor_inverse_batched(&j, 1, s);
}

}  // namespace bic
