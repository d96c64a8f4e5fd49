// k_gemv.cu -- the two HBM passes of every inner sweep.
//
//   gemv   : y = A x            ("Compute A_ij x_ij"; and x_ij = H_ij r_ij)
//   gemv_t : r = rho_l A^T (p + delta) + rho_c (z - u)   (Eq. (24) normal equations)
//
// Both are HBM-bound (0.25 flop/B in FP64): the design goal is to stream A once
// per pass at full bandwidth with 128-bit, coalesced, L1-bypassing loads and
// enough independent loads in flight per SM (~40 KB) to cover DRAM latency.
// Reductions are fixed-order (warp shuffle tree / per-chunk partials summed in
// chunk order), so results are bitwise reproducible.
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace bic {

std::atomic<int64_t> g_launches{0};

// ============================================================== GEMV
// One warp-task = R consecutive rows of one descriptor; warps stride over the
// flattened task list of all descriptors (one launch covers every local block).
struct GemvBatch {
    GemvDesc d[kMaxDesc];
    int nd;
    int64_t total_tasks;
};

constexpr int kGemvR = 1;          // rows per warp-task (measured best: R=1, 7.0 TB/s at C2, profiles/r01_microbench.jsonl)
constexpr int kGemvThreads = 256;

template <int R>
__device__ __forceinline__ void gemv_rows_f64(const GemvDesc& D, int64_t r0, int lane) {
    const double2* rowp[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
        int64_t r = r0 + rr < D.rows ? r0 + rr : D.rows - 1;
        rowp[rr] = reinterpret_cast<const double2*>(static_cast<const double*>(D.A) + r * D.lda);
    }
    const double2* xv = reinterpret_cast<const double2*>(D.x);
    double acc[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) acc[rr] = 0.0;
    const int64_t nvec = D.cols >> 1;
    int64_t v = lane;
    for (; v + 32 < nvec; v += 64) {
        const double2 xa = __ldg(xv + v), xb = __ldg(xv + v + 32);
        double2 a[R], b[R];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) { a[rr] = ld_stream(rowp[rr] + v); b[rr] = ld_stream(rowp[rr] + v + 32); }
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            acc[rr] = fma(a[rr].x, xa.x, acc[rr]);
            acc[rr] = fma(a[rr].y, xa.y, acc[rr]);
            acc[rr] = fma(b[rr].x, xb.x, acc[rr]);
            acc[rr] = fma(b[rr].y, xb.y, acc[rr]);
        }
    }
    if (v < nvec) {
        const double2 xa = __ldg(xv + v);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            const double2 a = ld_stream(rowp[rr] + v);
            acc[rr] = fma(a.x, xa.x, acc[rr]);
            acc[rr] = fma(a.y, xa.y, acc[rr]);
        }
    }
    if ((D.cols & 1) && lane == 0) {
        const int64_t c = D.cols - 1;
        const double xc = __ldg(D.x + c);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) acc[rr] = fma(reinterpret_cast<const double*>(rowp[rr])[c], xc, acc[rr]);
    }
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
        const double s = warp_sum(acc[rr]);
        if (lane == rr && r0 + rr < D.rows) D.y[r0 + rr] = D.alpha * s;
    }
}

template <int R>
__device__ __forceinline__ void gemv_rows_f32(const GemvDesc& D, int64_t r0, int lane) {
    const float4* rowp[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
        int64_t r = r0 + rr < D.rows ? r0 + rr : D.rows - 1;
        rowp[rr] = reinterpret_cast<const float4*>(static_cast<const float*>(D.A) + r * D.lda);
    }
    const double2* xv = reinterpret_cast<const double2*>(D.x);
    double acc[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) acc[rr] = 0.0;
    const int64_t nvec = D.cols >> 2;
    int64_t v = lane;
    for (; v + 32 < nvec; v += 64) {
        const double2 x0 = __ldg(xv + 2 * v), x1 = __ldg(xv + 2 * v + 1);
        const double2 y0 = __ldg(xv + 2 * (v + 32)), y1 = __ldg(xv + 2 * (v + 32) + 1);
        float4 a[R], b[R];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) { a[rr] = ld_stream(rowp[rr] + v); b[rr] = ld_stream(rowp[rr] + v + 32); }
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            acc[rr] = fma((double)a[rr].x, x0.x, acc[rr]);
            acc[rr] = fma((double)a[rr].y, x0.y, acc[rr]);
            acc[rr] = fma((double)a[rr].z, x1.x, acc[rr]);
            acc[rr] = fma((double)a[rr].w, x1.y, acc[rr]);
            acc[rr] = fma((double)b[rr].x, y0.x, acc[rr]);
            acc[rr] = fma((double)b[rr].y, y0.y, acc[rr]);
            acc[rr] = fma((double)b[rr].z, y1.x, acc[rr]);
            acc[rr] = fma((double)b[rr].w, y1.y, acc[rr]);
        }
    }
    if (v < nvec) {
        const double2 x0 = __ldg(xv + 2 * v), x1 = __ldg(xv + 2 * v + 1);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            const float4 a = ld_stream(rowp[rr] + v);
            acc[rr] = fma((double)a.x, x0.x, acc[rr]);
            acc[rr] = fma((double)a.y, x0.y, acc[rr]);
            acc[rr] = fma((double)a.z, x1.x, acc[rr]);
            acc[rr] = fma((double)a.w, x1.y, acc[rr]);
        }
    }
    const int64_t tail = D.cols - 4 * nvec;
    if (lane < tail) {
        const int64_t c = 4 * nvec + lane;
        const double xc = __ldg(D.x + c);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) acc[rr] = fma((double)reinterpret_cast<const float*>(rowp[rr])[c], xc, acc[rr]);
    }
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
        const double s = warp_sum(acc[rr]);
        if (lane == rr && r0 + rr < D.rows) D.y[r0 + rr] = D.alpha * s;
    }
}

template <typename T, int R>
__global__ void __launch_bounds__(kGemvThreads) k_gemv(const __grid_constant__ GemvBatch B) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (kGemvThreads / 32);
    for (int64_t task = (int64_t)blockIdx.x * (kGemvThreads / 32) + (threadIdx.x >> 5); task < B.total_tasks;
         task += nwarps) {
        int di = 0;
        while (di + 1 < B.nd && task >= B.d[di + 1].task_begin) ++di;
        const GemvDesc& D = B.d[di];
        const int64_t r0 = (task - D.task_begin) * R;
        if constexpr (sizeof(T) == 8) gemv_rows_f64<R>(D, r0, lane);
        else gemv_rows_f32<R>(D, r0, lane);
    }
}

// rows per warp-task: BICADMM_GEMV_R in {1, 2, 4, 8} (tuning), default kGemvR
static int gemv_rows_per_task() {
    static int r = [] {
        const char* e = getenv("BICADMM_GEMV_R");
        int v = e ? atoi(e) : kGemvR;
        return (v == 1 || v == 2 || v == 4 || v == 8) ? v : kGemvR;
    }();
    return r;
}

template <typename T>
static void gemv_dispatch(int R, unsigned blocks, cudaStream_t s, const GemvBatch& B) {
    switch (R) {
    case 1: k_gemv<T, 1><<<blocks, kGemvThreads, 0, s>>>(B); break;
    case 2: k_gemv<T, 2><<<blocks, kGemvThreads, 0, s>>>(B); break;
    case 8: k_gemv<T, 8><<<blocks, kGemvThreads, 0, s>>>(B); break;
    default: k_gemv<T, 4><<<blocks, kGemvThreads, 0, s>>>(B); break;
    }
}

int launch_gemv(int dtype, GemvDesc* d, int nd, int grid_cap, cudaStream_t s, int C) {
    if (C > 1) return launch_gemv_c(dtype, C, d, nd, s);
    const int R = gemv_rows_per_task();
    for (int base = 0; base < nd; base += kMaxDesc) {
        GemvBatch B;
        B.nd = nd - base < kMaxDesc ? nd - base : kMaxDesc;
        int64_t t = 0;
        for (int k = 0; k < B.nd; ++k) {
            B.d[k] = d[base + k];
            B.d[k].task_begin = t;
            t += (B.d[k].rows + R - 1) / R;
        }
        B.total_tasks = t;
        if (t == 0) continue;
        int64_t blocks = (t + (kGemvThreads / 32) - 1) / (kGemvThreads / 32);
        // default: one warp-task per warp (the block scheduler balances the tail);
        // BICADMM_GEMV_PERSISTENT=1 caps the grid at the resident CTA count instead
        static const bool persistent = getenv("BICADMM_GEMV_PERSISTENT") && atoi(getenv("BICADMM_GEMV_PERSISTENT"));
        if (persistent && blocks > grid_cap) blocks = grid_cap;
        if (blocks > 0x7fffffff) blocks = 0x7fffffff;
        if (dtype == BICADMM_F64) gemv_dispatch<double>(R, (unsigned)blocks, s, B);
        else gemv_dispatch<float>(R, (unsigned)blocks, s, B);
        BIC_LAUNCHED();
    }
    return BICADMM_OK;
}

int gemv_grid_cap(int dtype, int sm_count) {
    int occ = 0;
    if (dtype == BICADMM_F64) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gemv<double, kGemvR>, kGemvThreads, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gemv<float, kGemvR>, kGemvThreads, 0);
    if (occ < 1) occ = 1;
    return occ * sm_count;
}

// ============================================================== GEMV-T
// CTA-task = (descriptor, column strip of W columns, row chunk).  8 warps share
// the strip and interleave rows; each lane owns 4 vector slots of the strip
// (coalesced: one load instruction covers 512 contiguous bytes per warp).  The 8
// warp partials are summed in warp order in shared memory and written to
// partial[chunk][col]; a second kernel sums chunks in chunk order and applies the
// Eq. (24) epilogue.
constexpr int kGtThreads = 256;
constexpr int kGtWarps = kGtThreads / 32;
constexpr int kGtK = 4;  // vector slots per lane

template <typename T> struct VecOf;
template <> struct VecOf<double> { using V = double2; static constexpr int n = 2; };
template <> struct VecOf<float> { using V = float4; static constexpr int n = 4; };

int gemv_t_strip_width(int dtype) { return 32 * kGtK * (dtype == BICADMM_F64 ? 2 : 4); }

struct GemvTBatch {
    GemvTDesc d[kMaxDesc];
    int nd;
    int64_t total_ctas;
};

__device__ __forceinline__ void vfma(double* acc, const double2& a, double q) {
    acc[0] = fma(a.x, q, acc[0]);
    acc[1] = fma(a.y, q, acc[1]);
}
__device__ __forceinline__ void vfma(double* acc, const float4& a, double q) {
    acc[0] = fma((double)a.x, q, acc[0]);
    acc[1] = fma((double)a.y, q, acc[1]);
    acc[2] = fma((double)a.z, q, acc[2]);
    acc[3] = fma((double)a.w, q, acc[3]);
}

template <typename T>
__global__ void __launch_bounds__(kGtThreads) k_gemv_t_partial(const __grid_constant__ GemvTBatch B) {
    using V = typename VecOf<T>::V;
    constexpr int VN = VecOf<T>::n;
    constexpr int W = 32 * kGtK * VN;
    __shared__ double red[kGtWarps][W];

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

    double acc[kGtK * VN];
#pragma unroll
    for (int k = 0; k < kGtK * VN; ++k) acc[k] = 0.0;

    const T* A = static_cast<const T*>(D.A);
    const bool full = c_strip + W <= D.cols;
    if (full) {
        int64_t r = rb + w;
        for (; r + kGtWarps < re; r += 2 * kGtWarps) {
            const int64_t r2 = r + kGtWarps;
            double q1 = D.p[r], q2 = D.p[r2];
            if (D.delta) { q1 += D.delta[r]; q2 += D.delta[r2]; }
            const V* a1 = reinterpret_cast<const V*>(A + r * D.lda + c_strip) + lane;
            const V* a2 = reinterpret_cast<const V*>(A + r2 * D.lda + c_strip) + lane;
            V x1[kGtK], x2[kGtK];
#pragma unroll
            for (int k = 0; k < kGtK; ++k) { x1[k] = ld_stream(a1 + 32 * k); x2[k] = ld_stream(a2 + 32 * k); }
#pragma unroll
            for (int k = 0; k < kGtK; ++k) { vfma(acc + k * VN, x1[k], q1); vfma(acc + k * VN, x2[k], q2); }
        }
        if (r < re) {
            double q1 = D.p[r];
            if (D.delta) q1 += D.delta[r];
            const V* a1 = reinterpret_cast<const V*>(A + r * D.lda + c_strip) + lane;
#pragma unroll
            for (int k = 0; k < kGtK; ++k) vfma(acc + k * VN, ld_stream(a1 + 32 * k), q1);
        }
    } else {
        for (int64_t r = rb + w; r < re; r += kGtWarps) {
            double q1 = D.p[r];
            if (D.delta) q1 += D.delta[r];
            const T* row = A + r * D.lda;
#pragma unroll
            for (int k = 0; k < kGtK; ++k) {
                const int64_t c = c_strip + (int64_t)(32 * k + lane) * VN;
                if (c + VN <= D.cols) {
                    vfma(acc + k * VN, ld_stream(reinterpret_cast<const V*>(row + c)), q1);
                } else {
#pragma unroll
                    for (int e = 0; e < VN; ++e)
                        if (c + e < D.cols) acc[k * VN + e] = fma((double)row[c + e], q1, acc[k * VN + e]);
                }
            }
        }
    }
#pragma unroll
    for (int k = 0; k < kGtK; ++k)
#pragma unroll
        for (int e = 0; e < VN; ++e) red[w][(32 * k + lane) * VN + e] = acc[k * VN + e];
    __syncthreads();
    double* out = D.partial + chunk * D.cols;
    for (int c = threadIdx.x; c < W; c += kGtThreads) {
        double s = 0.0;
#pragma unroll
        for (int ww = 0; ww < kGtWarps; ++ww) s += red[ww][c];
        if (c_strip + c < D.cols) out[c_strip + c] = s;
    }
}

struct GemvTRedBatch {
    GemvTDesc d[kMaxDesc];
    int nd;
    int64_t cta_begin[kMaxDesc];
};

__global__ void __launch_bounds__(256) k_gemv_t_reduce(const __grid_constant__ GemvTRedBatch B, double rho_l,
                                                       double rho_c, int C) {
    const int64_t cta = blockIdx.x;
    int di = 0;
    while (di + 1 < B.nd && cta >= B.cta_begin[di + 1]) ++di;
    const GemvTDesc& D = B.d[di];
    const int64_t c = (cta - B.cta_begin[di]) * 256 + threadIdx.x;
    const int64_t ncomp = D.cols * C;
    if (c >= ncomp) return;
    double s = 0.0;
    for (int k = 0; k < D.nchunks; ++k) s += D.partial[(int64_t)k * ncomp + c];
    double r = rho_l * s;
    if (D.z || D.u) r += rho_c * ((D.z ? D.z[c] : 0.0) - (D.u ? D.u[c] : 0.0));
    D.r[c] = r;
}

void plan_gemv_t(int dtype, GemvTDesc* d, int nd, int sm_count, int64_t* need, int C) {
    const int W = C > 1 ? gemv_t_c_strip_width(dtype) : gemv_t_strip_width(dtype);
    int64_t total_strips = 0;
    for (int k = 0; k < nd; ++k) {
        d[k].nstrips = (int32_t)((d[k].cols + W - 1) / W);
        total_strips += d[k].nstrips;
    }
    // C = 1: ~192 CTAs per SM over the launch, i.e. short row chunks, so that the CTAs in
    // flight at any time touch a narrow band of rows (at 100 GB of A: 5.4 -> 6.2 TB/s, the
    // wide-band variant thrashes address translation); C > 1: 24.  BICADMM_GEMVT_CTAS_PER_SM
    // overrides (tuning)
    static const int env_per_sm = [] { const char* e = getenv("BICADMM_GEMVT_CTAS_PER_SM"); return e && atoi(e) > 0 ? atoi(e) : 0; }();
    const int per_sm = env_per_sm ? env_per_sm : (C > 1 ? 24 : 192);
    const int64_t target = (int64_t)sm_count * per_sm;
    int64_t chunks = total_strips > 0 ? (target + total_strips - 1) / total_strips : 1;
    if (chunks < 1) chunks = 1;
    for (int k = 0; k < nd; ++k) {
        int64_t cr = (d[k].rows + chunks - 1) / chunks;
        if (cr < 64) cr = 64;
        cr = (cr + 15) / 16 * 16;
        d[k].chunk_rows = cr;
        d[k].nchunks = (int32_t)((d[k].rows + cr - 1) / cr);
        if (d[k].nchunks < 1) d[k].nchunks = 1;
        need[k] = (int64_t)d[k].nchunks * d[k].cols * C;
    }
}

int launch_gemv_t(int dtype, GemvTDesc* d, int nd, double rho_l, double rho_c, cudaStream_t s, cudaEvent_t mid,
                  int C) {
    // all partial passes first (the HBM pass over A), then the chunk reductions
    if (C > 1) {
        int rc = launch_gemv_t_c_partial(dtype, C, d, nd, s);
        if (rc) return rc;
    }
    for (int base = 0; base < nd && C == 1; base += kMaxDesc) {
        GemvTBatch B;
        B.nd = nd - base < kMaxDesc ? nd - base : kMaxDesc;
        int64_t t = 0;
        for (int k = 0; k < B.nd; ++k) {
            B.d[k] = d[base + k];
            B.d[k].cta_begin = t;
            t += (int64_t)B.d[k].nstrips * B.d[k].nchunks;
        }
        B.total_ctas = t;
        if (t > 0) {
            if (dtype == BICADMM_F64) k_gemv_t_partial<double><<<(unsigned)t, kGtThreads, 0, s>>>(B);
            else k_gemv_t_partial<float><<<(unsigned)t, kGtThreads, 0, s>>>(B);
            BIC_LAUNCHED();
        }
    }
    if (mid) BIC_CUDA(record_event(mid, s));
    return launch_gemv_t_reduce(d, nd, rho_l, rho_c, s, C);
}

int launch_gemv_t_reduce(GemvTDesc* d, int nd, double rho_l, double rho_c, cudaStream_t s, int C) {
    for (int base = 0; base < nd; base += kMaxDesc) {
        GemvTRedBatch R;
        R.nd = nd - base < kMaxDesc ? nd - base : kMaxDesc;
        int64_t tr = 0;
        for (int k = 0; k < R.nd; ++k) {
            R.d[k] = d[base + k];
            R.cta_begin[k] = tr;
            tr += (R.d[k].cols * C + 255) / 256;
        }
        if (tr > 0) {
            k_gemv_t_reduce<<<(unsigned)tr, 256, 0, s>>>(R, rho_l, rho_c, C);
            BIC_LAUNCHED();
        }
    }
    return BICADMM_OK;
}

}  // namespace bic
