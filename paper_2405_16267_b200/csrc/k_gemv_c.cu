// k_gemv_c.cu -- multi-class (softmax, C >= 2) variants of the two HBM passes
// (SURVEY 8(a) a2-a4 with X in R^{n x C}; DESIGN R13).  The feature matrix is
// still streamed once per pass; each element now feeds C FMAs, so at C = 10 the
// pass is ~2.5 flop/B in FP64 -- still under the FP64 ridge of B200.
//
//   gemv_c   : Y[r, c] = sum_l A[r, l] X[l, c]          (X, Y row-major n x C / m x C)
//   gemv_t_c : R[l, c] = rho_l sum_r A[r, l] Q[r, c] + rho_c (Z[l, c] - U[l, c]),  Q = P + Delta
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace bic {

struct GemvBatchC {
    GemvDesc d[kMaxDesc];
    int nd;
    int64_t total_tasks;
};

template <typename T> struct VecC;
template <> struct VecC<double> { using V = double2; static constexpr int n = 2; };
template <> struct VecC<float> { using V = float4; static constexpr int n = 4; };

__device__ __forceinline__ double vget(const double2& v, int e) { return e == 0 ? v.x : v.y; }
__device__ __forceinline__ double vget(const float4& v, int e) {
    return e == 0 ? (double)v.x : e == 1 ? (double)v.y : e == 2 ? (double)v.z : (double)v.w;
}

constexpr int kGemvCThreads = 256;

// one warp per row; lane owns one vector slot per 32*VN columns
template <typename T, int CM>
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
        const int64_t r = task - D.task_begin;
        const T* row = static_cast<const T*>(D.A) + r * D.lda;
        double acc[CM];
#pragma unroll
        for (int c = 0; c < CM; ++c) acc[c] = 0.0;
        for (int64_t l = (int64_t)lane * VN; l < D.cols; l += 32 * VN) {
            if (l + VN <= D.cols) {
                const V a = ld_stream(reinterpret_cast<const V*>(row + l));
#pragma unroll
                for (int e = 0; e < VN; ++e) {
                    const double ae = vget(a, e);
                    const double* xr = D.x + (l + e) * C;
#pragma unroll
                    for (int c = 0; c < CM; ++c)
                        if (c < C) acc[c] = fma(ae, __ldg(xr + c), acc[c]);
                }
            } else {
                for (int64_t e = l; e < D.cols; ++e) {
                    const double ae = (double)row[e];
#pragma unroll
                    for (int c = 0; c < CM; ++c)
                        if (c < C) acc[c] = fma(ae, __ldg(D.x + e * C + c), acc[c]);
                }
            }
        }
#pragma unroll
        for (int c = 0; c < CM; ++c) {
            if (c < C) {
                const double s = warp_sum(acc[c]);
                if (lane == 0) D.y[r * C + c] = s;
            }
        }
    }
}

template <typename T>
static void gemv_c_dispatch(int C, unsigned g, cudaStream_t s, const GemvBatchC& B) {
    if (C <= 2) k_gemv_c<T, 2><<<g, kGemvCThreads, 0, s>>>(B, C);
    else if (C <= 4) k_gemv_c<T, 4><<<g, kGemvCThreads, 0, s>>>(B, C);
    else if (C <= 8) k_gemv_c<T, 8><<<g, kGemvCThreads, 0, s>>>(B, C);
    else if (C <= 10) k_gemv_c<T, 10><<<g, kGemvCThreads, 0, s>>>(B, C);
    else k_gemv_c<T, 16><<<g, kGemvCThreads, 0, s>>>(B, C);
}

int launch_gemv_c(int dtype, int C, GemvDesc* d, int nd, cudaStream_t s) {
    if (C < 2 || C > 16) return BICADMM_ERR_INVALID;
    for (int base = 0; base < nd; base += kMaxDesc) {
        GemvBatchC B;
        B.nd = nd - base < kMaxDesc ? nd - base : kMaxDesc;
        int64_t t = 0;
        for (int k = 0; k < B.nd; ++k) {
            B.d[k] = d[base + k];
            B.d[k].task_begin = t;
            t += B.d[k].rows;
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
constexpr int kGtCWarps = 4;
constexpr int kGtCThreads = 32 * kGtCWarps;

int gemv_t_c_strip_width(int dtype) { return 32 * (dtype == BICADMM_F64 ? 2 : 4); }

struct GemvTBatchC {
    GemvTDesc d[kMaxDesc];
    int nd;
    int64_t total_ctas;
};

template <typename T, int CM>
__global__ void __launch_bounds__(kGtCThreads) k_gemv_t_partial_c(const __grid_constant__ GemvTBatchC B, int C) {
    using V = typename VecC<T>::V;
    constexpr int VN = VecC<T>::n;
    constexpr int W = 32 * VN;
    extern __shared__ double red[];   // [kGtCWarps][W * CM]
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
    double acc[VN][CM];
#pragma unroll
    for (int e = 0; e < VN; ++e)
#pragma unroll
        for (int c = 0; c < CM; ++c) acc[e][c] = 0.0;
    const T* A = static_cast<const T*>(D.A);
    const int64_t cl = c_strip + (int64_t)lane * VN;
    for (int64_t r = rb + w; r < re; r += kGtCWarps) {
        double q[CM];
#pragma unroll
        for (int c = 0; c < CM; ++c)
            q[c] = c < C ? D.p[r * C + c] + (D.delta ? D.delta[r * C + c] : 0.0) : 0.0;
        const T* row = A + r * D.lda;
        if (cl + VN <= D.cols) {
            const V a = ld_stream(reinterpret_cast<const V*>(row + cl));
#pragma unroll
            for (int e = 0; e < VN; ++e) {
                const double ae = vget(a, e);
#pragma unroll
                for (int c = 0; c < CM; ++c) acc[e][c] = fma(ae, q[c], acc[e][c]);
            }
        } else {
#pragma unroll
            for (int e = 0; e < VN; ++e)
                if (cl + e < D.cols) {
                    const double ae = (double)row[cl + e];
#pragma unroll
                    for (int c = 0; c < CM; ++c) acc[e][c] = fma(ae, q[c], acc[e][c]);
                }
        }
    }
#pragma unroll
    for (int e = 0; e < VN; ++e)
#pragma unroll
        for (int c = 0; c < CM; ++c) red[(size_t)w * W * CM + (lane * VN + e) * CM + c] = acc[e][c];
    __syncthreads();
    double* out = D.partial + chunk * D.cols * C;
    for (int k = threadIdx.x; k < W * CM; k += kGtCThreads) {
        const int col = k / CM, c = k % CM;
        if (c >= C || c_strip + col >= D.cols) continue;
        double s = 0.0;
#pragma unroll
        for (int ww = 0; ww < kGtCWarps; ++ww) s += red[(size_t)ww * W * CM + k];
        out[(c_strip + col) * C + c] = s;
    }
}

template <typename T, int CM>
static int launch_tc(unsigned g, int C, cudaStream_t s, const GemvTBatchC& B) {
    constexpr int W = 32 * VecC<T>::n;
    const size_t smem = sizeof(double) * kGtCWarps * W * CM;
    static bool set = false;
    if (!set) {
        if (cudaFuncSetAttribute(k_gemv_t_partial_c<T, CM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
            return BICADMM_ERR_CUDA;
        set = true;
    }
    k_gemv_t_partial_c<T, CM><<<g, kGtCThreads, smem, s>>>(B, C);
    return BICADMM_OK;
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
