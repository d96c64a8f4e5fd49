// k_gemv_dmma.cu -- multi-class (softmax, C in [2, 16]) HBM passes on the FP64 tensor
// pipe (SURVEY 8(a) a2 and a4 with X in R^{n x C}; DESIGN R13, section 6).
//
//   gemv_c   : Y[r, c] = alpha sum_l A[r, l] X[l, c]          (X, Y row-major n x C / m x C)
//   gemv_t_c : partial[chunk][l, c] = sum_{r in chunk} A[r, l] Q[r, c],  Q = P + Delta
//
// At C = 10 each A element feeds 10 FMAs (2.5 flop/B in FP64): as scalar FFMA code the
// passes are issue-bound well below the HBM roofline.  Here both are skinny GEMMs on
// `mma.sync.m8n8k4.f64` (SASS DMMA): one instruction = 256 FMAs.  N = C is padded to
// 8 (C <= 8) or 16 (two n-tiles).  A stays streamed exactly once with 128-bit
// L1-bypassing loads; the K order inside a 4-wide DMMA step is permuted so that every
// thread's A elements are contiguous in memory (a sum over k is order-free up to
// rounding, and the order is fixed, so results are reproducible).
//
// Fragment layout of m8n8k4 (f64): thread (g = lane/4, t = lane%4) holds A[g][t],
// B[t][g] and D[g][2t], D[g][2t+1].
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace bic {

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// four consecutive elements as doubles (16-byte aligned for the vector path)
__device__ __forceinline__ void ld4(const double* p, double (&v)[4]) {
    const double2 a = ld_stream(reinterpret_cast<const double2*>(p));
    const double2 b = ld_stream(reinterpret_cast<const double2*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
__device__ __forceinline__ void ld4(const float* p, double (&v)[4]) {
    const float4 a = ld_stream(reinterpret_cast<const float4*>(p));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
}

// ----------------------------------------------------------------------------- GEMV (Y = A X)
// CTA = 256 rows (8 warps x 4 m-tiles).  X is staged through shared memory in k-chunks
// of 64 (64 x 16 doubles, zero-padded past n and C), double-buffered: the next chunk's
// global loads are issued before the current chunk's DMMAs and stored after them.  The
// B-fragment reads xs[k][c] for k = 16s + 4t + j, c = 8nt + g are bank-conflict-free
// with the swizzle c ^ 4((k >> 2) & 3) (= c ^ 4t).
struct GemvBatchD {
    GemvDesc d[kMaxDesc];
    int nd;
    int64_t total_tasks;
};
constexpr int kGdThreads = 256;
constexpr int kGdR = 4;                       // m-tiles per warp
constexpr int kGdRows = 8 * kGdR * (kGdThreads / 32);   // 256 rows per CTA
constexpr int kGdKC = 64;                     // k per staged chunk

__device__ __forceinline__ int xs_swz(int k, int c) { return k * 16 + (c ^ (4 * ((k >> 2) & 3))); }

// XC = 2: classes 8 and 9 (C = 9 or 10) as two DFMAs per element instead of a second,
// three-quarters-empty n-tile: DMMA and DFMA share the FP64 datapath (tools/fp64_rate.cu:
// 37 TFLOP/s DMMA, 33 DFMA, 33 mixed), so this is 10 classes of work instead of 16.
template <typename T, int NT, int XC = 0>
__global__ void __launch_bounds__(kGdThreads, 2) k_gemv_dmma(const __grid_constant__ GemvBatchD B, int C) {
    __shared__ double xs[2][kGdKC * 16];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
    const int64_t task = blockIdx.x;
    int di = 0;
    while (di + 1 < B.nd && task >= B.d[di + 1].task_begin) ++di;
    const GemvDesc& D = B.d[di];
    const int64_t r0 = (task - D.task_begin) * kGdRows + (int64_t)w * (8 * kGdR);
    const T* rowp[kGdR];
#pragma unroll
    for (int i = 0; i < kGdR; ++i) {
        const int64_t r = r0 + 8 * i + g;
        rowp[i] = static_cast<const T*>(D.A) + (r < D.rows ? r : D.rows - 1) * D.lda;
    }
    double acc[kGdR][NT][2];
    double accx[kGdR][XC > 0 ? XC : 1];   // classes 8.. of row 8i + g over this thread's k
#pragma unroll
    for (int i = 0; i < kGdR; ++i) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[i][nt][0] = acc[i][nt][1] = 0.0;
#pragma unroll
        for (int e = 0; e < (XC > 0 ? XC : 1); ++e) accx[i][e] = 0.0;
    }
    const int64_t cols = D.cols;
    const double* x = D.x;
    // staging: thread e holds elements e, e + 256, e + 512, e + 768 of the 64 x 16 chunk
    double st[4];
    auto load_chunk = [&](int64_t kc) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = threadIdx.x + kGdThreads * q, k = e >> 4, c = e & 15;
            st[q] = (kc + k < cols && c < C) ? __ldg(x + (kc + k) * C + c) : 0.0;
        }
    };
    auto store_chunk = [&](int buf) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = threadIdx.x + kGdThreads * q, k = e >> 4, c = e & 15;
            xs[buf][xs_swz(k, c)] = st[q];
        }
    };
    load_chunk(0);
    store_chunk(0);
    __syncthreads();
    int buf = 0;
    for (int64_t kc = 0; kc < cols; kc += kGdKC) {
        const bool more = kc + kGdKC < cols;
        if (more) load_chunk(kc + kGdKC);
#pragma unroll
        for (int s4 = 0; s4 < kGdKC / 16; ++s4) {
            const int64_t kk = kc + 16 * s4 + 4 * t;   // this thread's 4 k-indices
            double a[kGdR][4];
            if (kk + 4 <= cols) {
#pragma unroll
                for (int i = 0; i < kGdR; ++i) ld4(rowp[i] + kk, a[i]);
            } else {
#pragma unroll
                for (int i = 0; i < kGdR; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) a[i][j] = kk + j < cols ? (double)rowp[i][kk + j] : 0.0;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int kl = 16 * s4 + 4 * t + j;
                double b[NT];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) b[nt] = xs[buf][xs_swz(kl, nt * 8 + g)];
#pragma unroll
                for (int i = 0; i < kGdR; ++i)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) dmma(acc[i][nt], a[i][j], b[nt]);
                if constexpr (XC > 0) {
                    // X[k][8], X[k][9]: adjacent after the swizzle (8 ^ 4m, 9 ^ 4m)
                    const double2 xe = *reinterpret_cast<const double2*>(&xs[buf][xs_swz(kl, 8)]);
#pragma unroll
                    for (int i = 0; i < kGdR; ++i) {
                        accx[i][0] = fma(a[i][j], xe.x, accx[i][0]);
                        if (XC > 1) accx[i][XC > 1 ? 1 : 0] = fma(a[i][j], xe.y, accx[i][XC > 1 ? 1 : 0]);
                    }
                }
            }
        }
        if (more) store_chunk(buf ^ 1);
        __syncthreads();
        buf ^= 1;
    }
    if constexpr (XC > 0) {   // the 4 lanes t of a row group hold disjoint k: fixed-order butterfly
#pragma unroll
        for (int i = 0; i < kGdR; ++i)
#pragma unroll
            for (int e = 0; e < XC; ++e) {
                accx[i][e] += __shfl_xor_sync(0xffffffffu, accx[i][e], 1);
                accx[i][e] += __shfl_xor_sync(0xffffffffu, accx[i][e], 2);
            }
    }
#pragma unroll
    for (int i = 0; i < kGdR; ++i) {
        const int64_t r = r0 + 8 * i + g;
        if (r >= D.rows) continue;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int c = nt * 8 + 2 * t + e;
                if (c < C) D.y[r * C + c] = D.alpha * acc[i][nt][e];
            }
        if constexpr (XC > 0)
            if (t == 0)
#pragma unroll
                for (int e = 0; e < XC; ++e)
                    if (8 + e < C) D.y[r * C + 8 + e] = D.alpha * accx[i][e];
    }
}

bool gemv_c_dmma_enabled() {
    static bool on = [] { const char* e = getenv("BICADMM_GEMVC_DMMA"); return !(e && atoi(e) == 0); }();
    return on;
}

// 9 <= C <= 10: one n-tile on DMMA plus DFMA for classes 8-9 (BICADMM_GEMVC_MIXED=0: two n-tiles)
static bool gemv_c_mixed() {
    static const bool on = [] { const char* e = getenv("BICADMM_GEMVC_MIXED"); return !(e && atoi(e) == 0); }();
    return on;
}

int launch_gemv_c_dmma(int dtype, int C, GemvDesc* d, int nd, cudaStream_t s) {
    if (C < 2 || C > 16) return BICADMM_ERR_INVALID;
    for (int base = 0; base < nd; base += kMaxDesc) {
        GemvBatchD B;
        B.nd = nd - base < kMaxDesc ? nd - base : kMaxDesc;
        int64_t t = 0;
        for (int k = 0; k < B.nd; ++k) {
            B.d[k] = d[base + k];
            B.d[k].task_begin = t;
            t += (B.d[k].rows + kGdRows - 1) / kGdRows;
        }
        B.total_tasks = t;
        if (t == 0) continue;
        const unsigned blocks = (unsigned)t;
        if (dtype == BICADMM_F64) {
            if (C <= 8) k_gemv_dmma<double, 1><<<blocks, kGdThreads, 0, s>>>(B, C);
            else if (C <= 10 && gemv_c_mixed()) k_gemv_dmma<double, 1, 2><<<blocks, kGdThreads, 0, s>>>(B, C);
            else k_gemv_dmma<double, 2><<<blocks, kGdThreads, 0, s>>>(B, C);
        } else {
            if (C <= 8) k_gemv_dmma<float, 1><<<blocks, kGdThreads, 0, s>>>(B, C);
            else if (C <= 10 && gemv_c_mixed()) k_gemv_dmma<float, 1, 2><<<blocks, kGdThreads, 0, s>>>(B, C);
            else k_gemv_dmma<float, 2><<<blocks, kGdThreads, 0, s>>>(B, C);
        }
        BIC_LAUNCHED();
    }
    return BICADMM_OK;
}

// ----------------------------------------------------------------------------- GEMV-T partials
// CTA = (descriptor, 256-column strip, row chunk); warp w owns 32 columns of the strip
// and walks every row of the chunk, 4 rows per DMMA step, kGtdU steps per iteration
// (loads first).  Thread (g, t) loads 4 consecutive columns 4g..4g+3 of row r + t: the
// DMMA j uses M-index g <-> column 4g + j, so the 8 warps of a CTA read 2 KB contiguous
// per row.  No cross-warp reduction: partial[chunk][l][c] is written straight from D.
constexpr int kGtdThreads = 256;
constexpr int kGtdU = 4;

struct GemvTBatchD {
    GemvTDesc d[kMaxDesc];
    int nd;
    int64_t total_ctas;
};

// q = p + delta of the CTA's rows is staged through shared memory in slices of 64 rows
// (64 x 16 doubles, double-buffered like X above); the B-fragment reads qs[row][c] for
// row = 4u + t, c = 8nt + g are conflict-free with the swizzle c ^ 4(row & 3).
constexpr int kGtdRC = 64;
__device__ __forceinline__ int qs_swz(int r, int c) { return r * 16 + (c ^ (4 * (r & 3))); }

template <typename T, int NT>
__global__ void __launch_bounds__(kGtdThreads, 2) k_gemv_t_dmma(const __grid_constant__ GemvTBatchD B, int C) {
    __shared__ double qs[2][kGtdRC * 16];
    const int64_t cta = blockIdx.x;
    int di = 0;
    while (di + 1 < B.nd && cta >= B.d[di + 1].cta_begin) ++di;
    const GemvTDesc& D = B.d[di];
    const int64_t local = cta - D.cta_begin;
    const int strip = (int)(local % D.nstrips);
    const int64_t chunk = local / D.nstrips;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
    const int64_t l0 = (int64_t)strip * 256 + 32 * w + 4 * g;   // this thread's 4 columns
    const int64_t rb = chunk * D.chunk_rows;
    const int64_t re = rb + D.chunk_rows < D.rows ? rb + D.chunk_rows : D.rows;
    const int64_t cols = D.cols;
    const bool vec = l0 + 4 <= cols;
    const T* A = static_cast<const T*>(D.A);
    double acc[4][NT][2];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[j][nt][0] = acc[j][nt][1] = 0.0;
    double st[4];
    auto load_slice = [&](int64_t rs) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = threadIdx.x + kGtdThreads * q, rr = e >> 4, c = e & 15;
            const int64_t r = rs + rr;
            st[q] = (r < re && c < C) ? D.p[r * C + c] + (D.delta ? D.delta[r * C + c] : 0.0) : 0.0;
        }
    };
    auto store_slice = [&](int buf) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = threadIdx.x + kGtdThreads * q, rr = e >> 4, c = e & 15;
            qs[buf][qs_swz(rr, c)] = st[q];
        }
    };
    load_slice(rb);
    store_slice(0);
    __syncthreads();
    int buf = 0;
    for (int64_t rs = rb; rs < re; rs += kGtdRC) {
        const bool more = rs + kGtdRC < re;
        if (more) load_slice(rs + kGtdRC);
#pragma unroll
        for (int u0 = 0; u0 < kGtdRC / 4; u0 += kGtdU) {
            double a[kGtdU][4];
#pragma unroll
            for (int u = 0; u < kGtdU; ++u) {   // kGtdU row-steps of loads in flight
                const int64_t r = rs + 4 * (u0 + u) + t;
                const bool ok = r < re;
                const T* row = A + (ok ? r : rb) * D.lda + l0;
                if (ok && vec) {
                    ld4(row, a[u]);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) a[u][j] = (ok && l0 + j < cols) ? (double)row[j] : 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < kGtdU; ++u) {
                const int rl = 4 * (u0 + u) + t;
                double q[NT];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) q[nt] = qs[buf][qs_swz(rl, nt * 8 + g)];
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) dmma(acc[j][nt], a[u][j], q[nt]);
            }
        }
        if (more) store_slice(buf ^ 1);
        __syncthreads();
        buf ^= 1;
    }
    // D[g][2t+e] of DMMA j: M-index g = column l0 + j of lane group g, class nt*8 + 2t + e
    double* out = D.partial + chunk * cols * C;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t l = l0 + j;
        if (l >= cols) continue;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int c = nt * 8 + 2 * t + e;
                if (c < C) out[l * C + c] = acc[j][nt][e];
            }
    }
}

// ----------------------------------------------------------------------------- GEMV-T, TMA-staged
// FP64, even C and even row widths: the CTA's A rows (32 x 256-column strip per stage) and
// the matching p / delta slices are moved by cp.async.bulk into a 3-stage shared-memory
// ring (one producer warp, mbarrier complete_tx), so ~200 KB per SM are in flight without
// spending registers on it.  Rows are padded to 260 doubles: with the column mapping
// g + 8j of the DMMA M-index, the 16 lanes of a half-warp read 4 rows x 32 contiguous
// bytes each, 32 bytes apart modulo 128 (conflict-free).
#ifndef BIC_TT_RS
#define BIC_TT_RS 32
#define BIC_TT_ST 3
#endif
constexpr int kTtW = 256, kTtRS = BIC_TT_RS, kTtLD = 260, kTtST = BIC_TT_ST;
// 16 consumer warps: warp w takes the 32 columns 32 (w & 7) + g + 8j of the strip and the
// row half w >> 3 of every stage (two independent accumulator sets per column, so twice
// the DMMA chains in flight: with 8 warps the FP64 tensor pipe idled on the DMMA -> DMMA
// dependency), summed in a fixed order (half 0 + half 1) at the end.
constexpr int kTtCW = 16;
constexpr int kTtThreads = 32 * kTtCW + 32;   // consumer warps + 1 producer warp
constexpr size_t kTtSmem = sizeof(double) * (size_t)kTtST * kTtRS * (kTtLD + 2 * 16);

__device__ __forceinline__ unsigned tt_smem(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tt_bulk(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     tt_smem(dst)),
                 "l"(src), "r"(bytes), "r"(tt_smem(bar))
                 : "memory");
}
__device__ __forceinline__ bool tt_try(uint64_t* b, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{ .reg .pred P; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
        : "=r"(ok) : "r"(tt_smem(b)), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void tt_wait(uint64_t* b, unsigned parity) {
    for (long long it = 0; !tt_try(b, parity); ++it)
        if (it > (1ll << 26)) asm volatile("trap;");
}

template <int NT, int XC = 0>
__global__ void __launch_bounds__(kTtThreads, 1) k_gemv_t_dmma_tma(const __grid_constant__ GemvTBatchD B, int C) {
    extern __shared__ __align__(128) unsigned char tt_sm[];
    double* As = reinterpret_cast<double*>(tt_sm);        // [ST][RS][LD]
    double* Ps = As + (size_t)kTtST * kTtRS * kTtLD;       // [ST][RS * C] (C <= 16)
    double* Ds = Ps + (size_t)kTtST * kTtRS * 16;
    __shared__ __align__(8) uint64_t full[kTtST], empty[kTtST];
    const int64_t cta = blockIdx.x;
    int di = 0;
    while (di + 1 < B.nd && cta >= B.d[di + 1].cta_begin) ++di;
    const GemvTDesc& D = B.d[di];
    const int64_t local = cta - D.cta_begin;
    const int strip = (int)(local % D.nstrips);
    const int64_t chunk = local / D.nstrips;
    const int64_t l0 = (int64_t)strip * kTtW, cols = D.cols;
    const int wcols = (int)(cols - l0 < kTtW ? cols - l0 : kTtW);
    const int64_t rb = chunk * D.chunk_rows;
    const int64_t re = rb + D.chunk_rows < D.rows ? rb + D.chunk_rows : D.rows;
    const int nstage = (int)((re - rb + kTtRS - 1) / kTtRS);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTtST; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tt_smem(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tt_smem(&empty[s])), "r"(kTtCW));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kTtCW) {
        // all 32 lanes issue copies (lane i: row i; lane 0 also the p / delta slices): one
        // thread issuing 34 bulk copies per stage was the stage-rate limit
        const double* A = static_cast<const double*>(D.A);
        for (int st = 0; st < nstage; ++st) {
            const int s = st % kTtST;
            const int64_t r0 = rb + (int64_t)st * kTtRS;
            const int nr = (int)(re - r0 < kTtRS ? re - r0 : kTtRS);
            const unsigned abytes = (unsigned)(wcols * 8), vbytes = (unsigned)(nr * C * 8);
            if (lane == 0) {
                if (st >= kTtST) tt_wait(&empty[s], (unsigned)((st / kTtST - 1) & 1));
                const unsigned total = abytes * nr + vbytes * (D.delta ? 2u : 1u);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tt_smem(&full[s])),
                             "r"(total) : "memory");
            }
            __syncwarp();
            double* as = As + (size_t)s * kTtRS * kTtLD;
            for (int i = lane; i < nr; i += 32) tt_bulk(as + i * kTtLD, A + (r0 + i) * D.lda + l0, abytes, &full[s]);
            if (lane == 0) {
                tt_bulk(Ps + (size_t)s * kTtRS * 16, D.p + r0 * C, vbytes, &full[s]);
                if (D.delta) tt_bulk(Ds + (size_t)s * kTtRS * 16, D.delta + r0 * C, vbytes, &full[s]);
            }
        }
        return;
    }
    const int g = lane >> 2, t = lane & 3;
    double acc[4][NT][2];
    double accx[4][XC > 0 ? XC : 1];   // classes 8.. of column cbase + 8j over this thread's rows
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[j][nt][0] = acc[j][nt][1] = 0.0;
#pragma unroll
        for (int e = 0; e < (XC > 0 ? XC : 1); ++e) accx[j][e] = 0.0;
    }
    const int cbase = 32 * (warp & 7) + g;   // this thread's columns cbase + 8j
    const int half = warp >> 3;               // rows [half RS/2, (half + 1) RS/2) of each stage
    for (int st = 0; st < nstage; ++st) {
        const int s = st % kTtST;
        tt_wait(&full[s], (unsigned)((st / kTtST) & 1));
        const int64_t r0 = rb + (int64_t)st * kTtRS;
        const int nr = (int)(re - r0 < kTtRS ? re - r0 : kTtRS);
        const double* as = As + (size_t)s * kTtRS * kTtLD;
        const double* ps = Ps + (size_t)s * kTtRS * 16;
        const double* ds = Ds + (size_t)s * kTtRS * 16;
#pragma unroll
        for (int uu = 0; uu < kTtRS / 8; ++uu) {
            const int i = 4 * (half * (kTtRS / 8) + uu) + t;
            const bool ok = i < nr;
            double a[4], q[NT];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int c = cbase + 8 * j;
                a[j] = (ok && c < wcols) ? as[i * kTtLD + c] : 0.0;
            }
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const int c = nt * 8 + g;
                q[nt] = (ok && c < C) ? ps[i * C + c] + (D.delta ? ds[i * C + c] : 0.0) : 0.0;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) dmma(acc[j][nt], a[j], q[nt]);
            if constexpr (XC > 0) {   // Q[row i][8], Q[row i][9] (C even: 16-byte aligned pair)
                double2 qe = make_double2(0.0, 0.0);
                if (ok) {
                    qe = *reinterpret_cast<const double2*>(ps + i * C + 8);
                    if (D.delta) {
                        const double2 de = *reinterpret_cast<const double2*>(ds + i * C + 8);
                        qe.x += de.x;
                        qe.y += de.y;
                    }
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    accx[j][0] = fma(a[j], qe.x, accx[j][0]);
                    if (XC > 1) accx[j][XC > 1 ? 1 : 0] = fma(a[j], qe.y, accx[j][XC > 1 ? 1 : 0]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) asm volatile("{ .reg .b64 st; mbarrier.arrive.release.cta.shared::cta.b64 st, [%0]; }" ::"r"(
                                        tt_smem(&empty[s])) : "memory");
    }
    // fixed-order sum of the two row halves through shared memory (the ring is drained: every
    // stage was consumed by all consumer warps before they reach this barrier)
    if constexpr (XC > 0) {   // the 4 lanes t hold disjoint rows of the same columns
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < XC; ++e) {
                accx[j][e] += __shfl_xor_sync(0xffffffffu, accx[j][e], 1);
                accx[j][e] += __shfl_xor_sync(0xffffffffu, accx[j][e], 2);
            }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kTtCW) : "memory");
    constexpr int kRed = 4 * NT * 2 + 4 * XC;
    double* red = As + (size_t)(threadIdx.x & 255) * kRed;
    if (half == 1) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                red[(j * NT + nt) * 2] = acc[j][nt][0];
                red[(j * NT + nt) * 2 + 1] = acc[j][nt][1];
            }
#pragma unroll
            for (int e = 0; e < XC; ++e) red[4 * NT * 2 + j * XC + e] = accx[j][e];
        }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kTtCW) : "memory");
    if (half == 1) return;
    // D[g][2t+e] of DMMA j: column l0 + 32 warp + g + 8j, class nt*8 + 2t + e
    double* out = D.partial + chunk * cols * C;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int c = cbase + 8 * j;
        if (c >= wcols) continue;
        const int64_t l = l0 + c;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int k = nt * 8 + 2 * t + e;
                if (k < C) out[l * C + k] = acc[j][nt][e] + red[(j * NT + nt) * 2 + e];
            }
        if constexpr (XC > 0)
            if (t == 0)
#pragma unroll
                for (int e = 0; e < XC; ++e)
                    if (8 + e < C) out[l * C + 8 + e] = accx[j][e] + red[4 * NT * 2 + j * XC + e];
    }
}

static bool gemv_t_tma_ok(int dtype, int C, const GemvTDesc* d, int nd) {
    static const bool on = [] { const char* e = getenv("BICADMM_GEMVTC_TMA"); return !(e && atoi(e) == 0); }();
    if (!on || dtype != BICADMM_F64 || (C & 1)) return false;
    for (int k = 0; k < nd; ++k)
        if ((d[k].cols & 1) || (d[k].lda & 1) ||
            (reinterpret_cast<uintptr_t>(d[k].A) & 15) || (reinterpret_cast<uintptr_t>(d[k].p) & 15) ||
            (d[k].delta && (reinterpret_cast<uintptr_t>(d[k].delta) & 15)))
            return false;
    return true;
}

int launch_gemv_t_c_dmma(int dtype, int C, GemvTDesc* d, int nd, cudaStream_t s) {
    if (C < 2 || C > 16) return BICADMM_ERR_INVALID;
    if (gemv_t_tma_ok(dtype, C, d, nd)) {
        static bool attr = false;
        if (!attr) {
            if (cudaFuncSetAttribute(k_gemv_t_dmma_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTtSmem) !=
                    cudaSuccess ||
                cudaFuncSetAttribute(k_gemv_t_dmma_tma<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTtSmem) !=
                    cudaSuccess ||
                cudaFuncSetAttribute(k_gemv_t_dmma_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTtSmem) !=
                    cudaSuccess)
                return BICADMM_ERR_CUDA;
            attr = true;
        }
        for (int base = 0; base < nd; base += kMaxDesc) {
            GemvTBatchD B;
            B.nd = nd - base < kMaxDesc ? nd - base : kMaxDesc;
            int64_t t = 0;
            for (int k = 0; k < B.nd; ++k) {
                B.d[k] = d[base + k];
                B.d[k].cta_begin = t;
                t += (int64_t)B.d[k].nstrips * B.d[k].nchunks;
            }
            B.total_ctas = t;
            if (t == 0) continue;
            if (C <= 8) k_gemv_t_dmma_tma<1><<<(unsigned)t, kTtThreads, kTtSmem, s>>>(B, C);
            else if (C <= 10 && gemv_c_mixed()) k_gemv_t_dmma_tma<1, 2><<<(unsigned)t, kTtThreads, kTtSmem, s>>>(B, C);
            else k_gemv_t_dmma_tma<2><<<(unsigned)t, kTtThreads, kTtSmem, s>>>(B, C);
            BIC_LAUNCHED();
        }
        return BICADMM_OK;
    }
    for (int base = 0; base < nd; base += kMaxDesc) {
        GemvTBatchD B;
        B.nd = nd - base < kMaxDesc ? nd - base : kMaxDesc;
        int64_t t = 0;
        for (int k = 0; k < B.nd; ++k) {
            B.d[k] = d[base + k];
            B.d[k].cta_begin = t;
            t += (int64_t)B.d[k].nstrips * B.d[k].nchunks;
        }
        B.total_ctas = t;
        if (t == 0) continue;
        if (t > 0x7fffffff) return BICADMM_ERR_INVALID;
        if (dtype == BICADMM_F64) {
            if (C <= 8) k_gemv_t_dmma<double, 1><<<(unsigned)t, kGtdThreads, 0, s>>>(B, C);
            else k_gemv_t_dmma<double, 2><<<(unsigned)t, kGtdThreads, 0, s>>>(B, C);
        } else {
            if (C <= 8) k_gemv_t_dmma<float, 1><<<(unsigned)t, kGtdThreads, 0, s>>>(B, C);
            else k_gemv_t_dmma<float, 2><<<(unsigned)t, kGtdThreads, 0, s>>>(B, C);
        }
        BIC_LAUNCHED();
    }
    return BICADMM_OK;
}

}  // namespace bic
