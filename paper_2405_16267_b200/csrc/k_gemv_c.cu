// k_gemv_c.cu -- multi-class (softmax, C >= 2) variants of the two HBM passes
// (SURVEY 8(a) a2-a4 with X in R^{n x C}; DESIGN R13).  A is still streamed once per
// pass; each element now feeds C FMAs (2.5 flop/B at C = 10 in FP64).
//
//   gemv_c   : Y[r, c] = sum_l A[r, l] X[l, c]          (X, Y row-major n x C / m x C)
//   gemv_t_c : R[l, c] = rho_l sum_r A[r, l] Q[r, c] + rho_c (Z[l, c] - U[l, c]),  Q = P + Delta
//
// gemv_c: X is first transposed to class-major XT (C x n, a tiny kernel) so that a
// warp's X loads are coalesced like its A loads; a warp-task is R = 4 rows, so each
// XT vector load from L1 feeds 4 rows (L1 traffic ~2.5x the HBM traffic at C = 10).
// gemv_t_c: each lane owns 2 vector slots of a 128-column (FP64) strip and 2 rows are
// in flight per warp; the C-vector q of a row is a warp-broadcast load.
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace bic {

template <typename T> struct VecC;
template <> struct VecC<double> { using V = double2; static constexpr int n = 2; };
template <> struct VecC<float> { using V = float4; static constexpr int n = 4; };

__device__ __forceinline__ double vget(const double2& v, int e) { return e == 0 ? v.x : v.y; }
__device__ __forceinline__ double vget(const float4& v, int e) {
    return e == 0 ? (double)v.x : e == 1 ? (double)v.y : e == 2 ? (double)v.z : (double)v.w;
}

// ----------------------------------------------------------------------------- X -> XT
struct TransBatch {
    const double* x[kMaxDesc];
    double* xt[kMaxDesc];
    int64_t cols[kMaxDesc], cta_begin[kMaxDesc];
    int nd;
};

__global__ void k_transpose_c(const __grid_constant__ TransBatch B, int C) {
    const int64_t cta = blockIdx.x;
    int di = 0;
    while (di + 1 < B.nd && cta >= B.cta_begin[di + 1]) ++di;
    const int64_t e = (cta - B.cta_begin[di]) * 256 + threadIdx.x;   // over cols * C (source order)
    if (e >= B.cols[di] * C) return;
    const int64_t l = e / C, c = e % C;
    B.xt[di][c * B.cols[di] + l] = B.x[di][e];
}

static int transpose_batch(const GemvDesc* d, int nd, int C, cudaStream_t s) {
    for (int base = 0; base < nd; base += kMaxDesc) {
        TransBatch B;
        B.nd = nd - base < kMaxDesc ? nd - base : kMaxDesc;
        int64_t t = 0;
        for (int k = 0; k < B.nd; ++k) {
            B.x[k] = d[base + k].x;
            B.xt[k] = d[base + k].xt;
            if (!B.xt[k]) return BICADMM_ERR_INVALID;
            B.cols[k] = d[base + k].cols;
            B.cta_begin[k] = t;
            t += (B.cols[k] * C + 255) / 256;
        }
        if (t == 0) continue;
        k_transpose_c<<<(unsigned)t, 256, 0, s>>>(B, C);
        BIC_LAUNCHED();
    }
    return BICADMM_OK;
}

// ----------------------------------------------------------------------------- GEMV, C columns
struct GemvBatchC {
    GemvDesc d[kMaxDesc];
    int nd;
    int64_t total_tasks;
};

constexpr int kGemvCThreads = 256;

static int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

template <typename T, int CM, int kGemvCR>
__global__ void __launch_bounds__(kGemvCThreads) k_gemv_c(const __grid_constant__ GemvBatchC B, int C) {
    using V = typename VecC<T>::V;
    constexpr int VN = VecC<T>::n;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (kGemvCThreads / 32);
    for (int64_t task = (int64_t)blockIdx.x * (kGemvCThreads / 32) + (threadIdx.x >> 5); task < B.total_tasks;
         task += nwarps) {
        int di = 0;
        while (di + 1 < B.nd && task >= B.d[di + 1].task_begin) ++di;
        const GemvDesc& D = B.d[di];
        const int64_t r0 = (task - D.task_begin) * kGemvCR;
        const T* rowp[kGemvCR];
#pragma unroll
        for (int rr = 0; rr < kGemvCR; ++rr)
            rowp[rr] = static_cast<const T*>(D.A) + (r0 + rr < D.rows ? r0 + rr : D.rows - 1) * D.lda;
        double acc[kGemvCR][CM];
#pragma unroll
        for (int rr = 0; rr < kGemvCR; ++rr)
#pragma unroll
            for (int c = 0; c < CM; ++c) acc[rr][c] = 0.0;
        const double* xt = D.xt;
        const int64_t cols = D.cols;
        for (int64_t l = (int64_t)lane * VN; l < cols; l += 32 * VN) {
            double a[kGemvCR][VN];
            if (l + VN <= cols) {
#pragma unroll
                for (int rr = 0; rr < kGemvCR; ++rr) {
                    const V v = ld_stream(reinterpret_cast<const V*>(rowp[rr] + l));
#pragma unroll
                    for (int e = 0; e < VN; ++e) a[rr][e] = vget(v, e);
                }
            } else {
#pragma unroll
                for (int rr = 0; rr < kGemvCR; ++rr)
#pragma unroll
                    for (int e = 0; e < VN; ++e) a[rr][e] = l + e < cols ? (double)rowp[rr][l + e] : 0.0;
            }
#pragma unroll
            for (int c = 0; c < CM; ++c) {
                if (c >= C) break;
                double xv[VN];
#pragma unroll
                for (int e = 0; e < VN; ++e) xv[e] = l + e < cols ? __ldg(xt + c * cols + l + e) : 0.0;
#pragma unroll
                for (int rr = 0; rr < kGemvCR; ++rr)
#pragma unroll
                    for (int e = 0; e < VN; ++e) acc[rr][c] = fma(a[rr][e], xv[e], acc[rr][c]);
            }
        }
#pragma unroll
        for (int rr = 0; rr < kGemvCR; ++rr)
#pragma unroll
            for (int c = 0; c < CM; ++c) {
                if (c < C) {
                    const double sum = warp_sum(acc[rr][c]);
                    if (lane == 0 && r0 + rr < D.rows) D.y[(r0 + rr) * C + c] = D.alpha * sum;
                }
            }
    }
}

template <typename T, int R>
static void gemv_c_dispatch_r(int C, unsigned g, cudaStream_t s, const GemvBatchC& B) {
    if (C <= 2) k_gemv_c<T, 2, R><<<g, kGemvCThreads, 0, s>>>(B, C);
    else if (C <= 4) k_gemv_c<T, 4, R><<<g, kGemvCThreads, 0, s>>>(B, C);
    else if (C <= 8) k_gemv_c<T, 8, R><<<g, kGemvCThreads, 0, s>>>(B, C);
    else if (C <= 10) k_gemv_c<T, 10, R><<<g, kGemvCThreads, 0, s>>>(B, C);
    else k_gemv_c<T, 16, R><<<g, kGemvCThreads, 0, s>>>(B, C);
}

// rows per warp-task (BICADMM_GEMVC_R in {1, 2, 4}; tuning)
static int gemv_c_rows() {
    static int r = [] { int v = env_int("BICADMM_GEMVC_R", 2); return (v == 1 || v == 2 || v == 4) ? v : 2; }();
    return r;
}

template <typename T>
static void gemv_c_dispatch(int C, unsigned g, cudaStream_t s, const GemvBatchC& B) {
    switch (gemv_c_rows()) {
    case 1: gemv_c_dispatch_r<T, 1>(C, g, s, B); break;
    case 4: gemv_c_dispatch_r<T, 4>(C, g, s, B); break;
    default: gemv_c_dispatch_r<T, 2>(C, g, s, B); break;
    }
}

int launch_gemv_c(int dtype, int C, GemvDesc* d, int nd, cudaStream_t s) {
    if (C < 2 || C > 16) return BICADMM_ERR_INVALID;
    if (gemv_c_dmma_enabled()) return launch_gemv_c_dmma(dtype, C, d, nd, s);   // k_gemv_dmma.cu
    int rc = transpose_batch(d, nd, C, s);
    if (rc) return rc;
    for (int base = 0; base < nd; base += kMaxDesc) {
        GemvBatchC B;
        B.nd = nd - base < kMaxDesc ? nd - base : kMaxDesc;
        int64_t t = 0;
        for (int k = 0; k < B.nd; ++k) {
            B.d[k] = d[base + k];
            B.d[k].task_begin = t;
            t += (B.d[k].rows + gemv_c_rows() - 1) / gemv_c_rows();
        }
        B.total_tasks = t;
        if (t == 0) continue;
        int64_t blocks = (t + (kGemvCThreads / 32) - 1) / (kGemvCThreads / 32);
        if (blocks > 0x7fffffff) blocks = 0x7fffffff;
        if (dtype == BICADMM_F64) gemv_c_dispatch<double>(C, (unsigned)blocks, s, B);
        else gemv_c_dispatch<float>(C, (unsigned)blocks, s, B);
        BIC_LAUNCHED();
    }
    return BICADMM_OK;
}

// ----------------------------------------------------------------------------- GEMV-T, C columns
constexpr int kGtCWarps = 8;
constexpr int kGtCThreads = 32 * kGtCWarps;
// vector slots per lane: 2 x double2 (FP64) or 1 x float4 (FP32) -> 128-column strips
template <typename T> __host__ __device__ constexpr int gtc_slots() { return sizeof(T) == 8 ? 2 : 1; }

int gemv_t_c_strip_width(int dtype) { (void)dtype; return gemv_c_dmma_enabled() ? 256 : 128; }

struct GemvTBatchC {
    GemvTDesc d[kMaxDesc];
    int nd;
    int64_t total_ctas;
};

template <typename T, int CM, int U>
__global__ void __launch_bounds__(kGtCThreads) k_gemv_t_partial_c(const __grid_constant__ GemvTBatchC B, int C) {
    using V = typename VecC<T>::V;
    constexpr int VN = VecC<T>::n;
    constexpr int S = gtc_slots<T>();
    constexpr int W = 32 * S * VN;
    extern __shared__ double red[];   // [kGtCWarps][W][C]
    const int64_t cta = blockIdx.x;
    int di = 0;
    while (di + 1 < B.nd && cta >= B.d[di + 1].cta_begin) ++di;
    const GemvTDesc& D = B.d[di];
    const int64_t local = cta - D.cta_begin;
    const int strip = (int)(local % D.nstrips);
    const int64_t chunk = local / D.nstrips;
    const int64_t c_strip = (int64_t)strip * W;
    const int64_t rb = chunk * D.chunk_rows;
    const int64_t re = rb + D.chunk_rows < D.rows ? rb + D.chunk_rows : D.rows;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double acc[S * VN][CM];
#pragma unroll
    for (int e = 0; e < S * VN; ++e)
#pragma unroll
        for (int c = 0; c < CM; ++c) acc[e][c] = 0.0;
    const T* A = static_cast<const T*>(D.A);
    for (int64_t r0 = rb + w; r0 < re; r0 += (int64_t)kGtCWarps * U) {
        double a[U][S * VN];
#pragma unroll
        for (int u = 0; u < U; ++u) {           // U rows' loads in flight before the FMAs
            const int64_t r = r0 + (int64_t)kGtCWarps * u;
            const T* row = A + (r < re ? r : rb) * D.lda;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const int64_t cl = c_strip + (int64_t)(lane + 32 * s) * VN;
                if (cl + VN <= D.cols) {
                    const V v = ld_stream(reinterpret_cast<const V*>(row + cl));
#pragma unroll
                    for (int e = 0; e < VN; ++e) a[u][s * VN + e] = vget(v, e);
                } else {
#pragma unroll
                    for (int e = 0; e < VN; ++e) a[u][s * VN + e] = cl + e < D.cols ? (double)row[cl + e] : 0.0;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t r = r0 + (int64_t)kGtCWarps * u;
            if (r >= re) break;
#pragma unroll
            for (int c = 0; c < CM; ++c) {
                if (c >= C) break;
                const double q = D.p[r * C + c] + (D.delta ? D.delta[r * C + c] : 0.0);
#pragma unroll
                for (int e = 0; e < S * VN; ++e) acc[e][c] = fma(a[u][e], q, acc[e][c]);
            }
        }
    }
    // red[w][col][c]
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
        for (int e = 0; e < VN; ++e) {
            const int col = (lane + 32 * s) * VN + e;
#pragma unroll
            for (int c = 0; c < CM; ++c)
                if (c < C) red[((size_t)w * W + col) * C + c] = acc[s * VN + e][c];
        }
    __syncthreads();
    double* out = D.partial + chunk * D.cols * C;
    for (int k = threadIdx.x; k < W * C; k += kGtCThreads) {
        const int col = k / C;
        if (c_strip + col >= D.cols) continue;
        double sum = 0.0;
#pragma unroll
        for (int ww = 0; ww < kGtCWarps; ++ww) sum += red[(size_t)ww * W * C + k];
        out[c_strip * C + k] = sum;
    }
}

template <typename T, int CM, int U>
static int launch_tc_u(unsigned g, int C, cudaStream_t s, const GemvTBatchC& B) {
    constexpr int W = 32 * gtc_slots<T>() * VecC<T>::n;
    const size_t smem = sizeof(double) * kGtCWarps * W * C;
    static bool set = false;
    if (!set) {
        if (cudaFuncSetAttribute(k_gemv_t_partial_c<T, CM, U>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(sizeof(double) * kGtCWarps * W * CM)) != cudaSuccess)
            return BICADMM_ERR_CUDA;
        set = true;
    }
    k_gemv_t_partial_c<T, CM, U><<<g, kGtCThreads, smem, s>>>(B, C);
    return BICADMM_OK;
}

// rows in flight per warp (BICADMM_GTC_U in {1, 2, 4}; tuning)
template <typename T, int CM>
static int launch_tc(unsigned g, int C, cudaStream_t s, const GemvTBatchC& B) {
    static int u = [] { int v = env_int("BICADMM_GTC_U", 2); return (v == 1 || v == 2 || v == 4) ? v : 2; }();
    if (u == 1) return launch_tc_u<T, CM, 1>(g, C, s, B);
    if (u == 4) return launch_tc_u<T, CM, 4>(g, C, s, B);
    return launch_tc_u<T, CM, 2>(g, C, s, B);
}

template <typename T>
static int gemv_t_c_dispatch(int C, unsigned g, cudaStream_t s, const GemvTBatchC& B) {
    if (C <= 2) return launch_tc<T, 2>(g, C, s, B);
    if (C <= 4) return launch_tc<T, 4>(g, C, s, B);
    if (C <= 8) return launch_tc<T, 8>(g, C, s, B);
    if (C <= 10) return launch_tc<T, 10>(g, C, s, B);
    return launch_tc<T, 16>(g, C, s, B);
}

int launch_gemv_t_c_partial(int dtype, int C, GemvTDesc* d, int nd, cudaStream_t s) {
    if (gemv_c_dmma_enabled()) return launch_gemv_t_c_dmma(dtype, C, d, nd, s);   // k_gemv_dmma.cu
    for (int base = 0; base < nd; base += kMaxDesc) {
        GemvTBatchC B;
        B.nd = nd - base < kMaxDesc ? nd - base : kMaxDesc;
        int64_t t = 0;
        for (int k = 0; k < B.nd; ++k) {
            B.d[k] = d[base + k];
            B.d[k].cta_begin = t;
            t += (int64_t)B.d[k].nstrips * B.d[k].nchunks;
        }
        B.total_ctas = t;
        if (t == 0) continue;
        int rc = dtype == BICADMM_F64 ? gemv_t_c_dispatch<double>(C, (unsigned)t, s, B)
                                      : gemv_t_c_dispatch<float>(C, (unsigned)t, s, B);
        if (rc) return rc;
        BIC_LAUNCHED();
    }
    return BICADMM_OK;
}

}  // namespace bic
