// k_fused.cu -- single-HBM-pass inner sweep, same algebra as
// Eqs. (22)-(24).
//
// The two-pass sweep streams A_ij twice: GEMV-T for r = rho_l A^T q + ... (a2) and
// GEMV for p = A x (a4).  But q_ij = p_ij + delta_i depends only on the row's own
// p and its per-sample prox (22)-(23), so sweep k's GEMV, prox and sweep k+1's
// GEMV-T partial products can share one read of each row:
//
//   phase A (HBM)  row r:  p_ij[r] = A_ij[r,:] x_ij (all local blocks j of node i),
//                          S = sum_j p_ij[r], abar = S/M, omega = prox(abar + nu),
//                          nu += abar - omega, delta = omega - abar - nu
//   phase B (L2)   chunk:  partial_j[chunk][l] = sum_{r in chunk} A_ij[r, l] (p_ij[r] + delta[r])
//
// One persistent kernel pulls tasks from a global queue ordered
//   A(0) A(1) B(0) A(2) B(1) ... A(last) B(last-1) B(last)
// so phase B re-reads a chunk (~16 MB) about one chunk after phase A streamed it
// from HBM, while it is still L2-resident (126 MB L2).  B(c) waits on a per-chunk
// completion counter of A(c) (tasks are dequeued in order by running CTAs, so
// the wait always terminates).  The next sweep's r = rho_l sum_chunks partial +
// rho_c (z - u) is the existing fixed-order chunk reduction.  Valid because q does
// not depend on z, u: partials computed at the end of an outer iteration serve the
// first sweep of the next.  All sums are fixed-order (bit-reproducible); integer
// atomics only schedule work.
#include <stdlib.h>
#include <cfloat>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace bic {

constexpr int kFThreads = 256;
constexpr int kFWarps = kFThreads / 32;
constexpr int kFStripK = 4;           // double2 slots per lane in a B task -> 256-column strip
constexpr int kFStrip = 32 * 2 * kFStripK;

__device__ __forceinline__ double f_sigmoid(double a) {
    if (a >= 0.0) return 1.0 / (1.0 + exp(-a));
    const double e = exp(a);
    return e / (1.0 + e);
}

__device__ double f_prox(int loss, int M, double rho, double b, double p) {
    const double Md = (double)M;
    if (loss == BICADMM_LS) return (2.0 * b + rho * p) / (2.0 * Md + rho);
    if (loss == BICADMM_HINGE) {
        const double pp = b * p;
        double y;
        if (Md * pp > 1.0) y = pp;
        else if (Md * (pp + 1.0 / rho) < 1.0) y = pp + 1.0 / rho;
        else y = 1.0 / Md;
        return b * y;
    }
    // logistic: safeguarded Newton on -b sigma(-b M w) + rho (w - p)
    double lo = p - 1.0 / rho, hi = p + 1.0 / rho, w = p;
    for (int it = 0; it < 60; ++it) {
        const double sg = f_sigmoid(-b * Md * w);
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

// dot of one row segment with x (FP64 or FP32 storage), whole warp, 4 loads in flight
template <typename T>
__device__ __forceinline__ double row_dot(const T* __restrict__ row, const double* __restrict__ x, int64_t n, int lane);

template <>
__device__ __forceinline__ double row_dot<double>(const double* __restrict__ row, const double* __restrict__ x,
                                                  int64_t n, int lane) {
    const double2* rv = reinterpret_cast<const double2*>(row);
    const double2* xv = reinterpret_cast<const double2*>(x);
    const int64_t nv = n >> 1;
    double acc = 0.0, acc2 = 0.0;
    int64_t v = lane;
    for (; v + 96 < nv; v += 128) {
        const double2 a0 = ld_stream(rv + v), a1 = ld_stream(rv + v + 32), a2 = ld_stream(rv + v + 64),
                      a3 = ld_stream(rv + v + 96);
        const double2 x0 = __ldg(xv + v), x1 = __ldg(xv + v + 32), x2 = __ldg(xv + v + 64), x3 = __ldg(xv + v + 96);
        acc = fma(a0.x, x0.x, acc); acc2 = fma(a0.y, x0.y, acc2);
        acc = fma(a1.x, x1.x, acc); acc2 = fma(a1.y, x1.y, acc2);
        acc = fma(a2.x, x2.x, acc); acc2 = fma(a2.y, x2.y, acc2);
        acc = fma(a3.x, x3.x, acc); acc2 = fma(a3.y, x3.y, acc2);
    }
    for (; v < nv; v += 32) {
        const double2 a0 = ld_stream(rv + v), x0 = __ldg(xv + v);
        acc = fma(a0.x, x0.x, acc); acc2 = fma(a0.y, x0.y, acc2);
    }
    if ((n & 1) && lane == 0) acc = fma(row[n - 1], __ldg(x + n - 1), acc);
    return warp_sum(acc + acc2);
}

template <>
__device__ __forceinline__ double row_dot<float>(const float* __restrict__ row, const double* __restrict__ x,
                                                 int64_t n, int lane) {
    const float4* rv = reinterpret_cast<const float4*>(row);
    const double2* xv = reinterpret_cast<const double2*>(x);
    const int64_t nv = n >> 2;
    double acc = 0.0, acc2 = 0.0;
    int64_t v = lane;
    for (; v + 32 < nv; v += 64) {
        const float4 a0 = ld_stream(rv + v), a1 = ld_stream(rv + v + 32);
        const double2 x0 = __ldg(xv + 2 * v), x1 = __ldg(xv + 2 * v + 1);
        const double2 y0 = __ldg(xv + 2 * (v + 32)), y1 = __ldg(xv + 2 * (v + 32) + 1);
        acc = fma((double)a0.x, x0.x, acc); acc2 = fma((double)a0.y, x0.y, acc2);
        acc = fma((double)a0.z, x1.x, acc); acc2 = fma((double)a0.w, x1.y, acc2);
        acc = fma((double)a1.x, y0.x, acc); acc2 = fma((double)a1.y, y0.y, acc2);
        acc = fma((double)a1.z, y1.x, acc); acc2 = fma((double)a1.w, y1.y, acc2);
    }
    for (; v < nv; v += 32) {
        const float4 a0 = ld_stream(rv + v);
        const double2 x0 = __ldg(xv + 2 * v), x1 = __ldg(xv + 2 * v + 1);
        acc = fma((double)a0.x, x0.x, acc); acc2 = fma((double)a0.y, x0.y, acc2);
        acc = fma((double)a0.z, x1.x, acc); acc2 = fma((double)a0.w, x1.y, acc2);
    }
    const int64_t tail = n - 4 * nv;
    if (lane < tail) acc = fma((double)row[4 * nv + lane], __ldg(x + 4 * nv + lane), acc);
    return warp_sum(acc + acc2);
}

template <typename T>
__device__ __forceinline__ void vfma_f(double* acc, const T* p, double q);
template <>
__device__ __forceinline__ void vfma_f<double>(double* acc, const double* p, double q) {
    acc[0] = fma(p[0], q, acc[0]);
    acc[1] = fma(p[1], q, acc[1]);
}
template <>
__device__ __forceinline__ void vfma_f<float>(double* acc, const float* p, double q) {
    acc[0] = fma((double)p[0], q, acc[0]);
    acc[1] = fma((double)p[1], q, acc[1]);
    acc[2] = fma((double)p[2], q, acc[2]);
    acc[3] = fma((double)p[3], q, acc[3]);
}

template <typename T>
__device__ void task_A(const FusedNode& nd, const FusedChunk& ch, int64_t u, int loss, int M, double rho, int lane,
                       int warp, double* sq_slot) {
    const int64_t r = ch.r0 + u * kFWarps + warp;
    double e2 = 0.0;
    if (r < ch.r1) {
        double S = 0.0;
        for (int j = 0; j < nd.nb; ++j) {
            const T* row = static_cast<const T*>(nd.A[j]) + r * nd.lda[j];
            const double pj = row_dot<T>(row, nd.x[j], nd.nj[j], lane);
            if (lane == 0) nd.p[j][r] = pj;
            S += pj;
        }
        if (lane == 0) {
            const double Md = (double)M;
            const double abar = S / Md;
            const double bl = (double)static_cast<const T*>(nd.b)[r];
            const double nu0 = nd.nu[r];
            const double om = f_prox(loss, M, rho, bl, abar + nu0);
            const double nu = nu0 + abar - om;
            nd.nu[r] = nu;
            nd.delta[r] = om - abar - nu;
            e2 = (abar - om) * (abar - om);
        }
    }
    if (sq_slot && lane == 0) sq_slot[warp] = e2;
}

template <typename T>
__device__ void task_B(const FusedNode& nd, const FusedChunk& ch, int64_t u, int lane, int warp, double* red) {
    constexpr int VN = sizeof(T) == 8 ? 2 : 4;
    constexpr int W = 32 * kFStripK * VN;
    // decode (block, strip)
    int j = 0;
    int64_t uu = u;
    while (j + 1 < nd.nb && uu >= nd.nstrips[j]) { uu -= nd.nstrips[j]; ++j; }
    const int64_t c_strip = uu * W;
    const int64_t cols = nd.nj[j];
    const T* A = static_cast<const T*>(nd.A[j]);
    const int64_t lda = nd.lda[j];
    const double* __restrict__ p = nd.p[j];
    double acc[kFStripK * VN];
#pragma unroll
    for (int k = 0; k < kFStripK * VN; ++k) acc[k] = 0.0;
    using V = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
    const bool full = c_strip + W <= cols;
    for (int64_t r = ch.r0 + warp; r < ch.r1; r += kFWarps) {
        const double q = __ldcg(p + r) + __ldcg(nd.delta + r);
        const T* row = A + r * lda + c_strip;
        if (full) {
            V a[kFStripK];
#pragma unroll
            for (int k = 0; k < kFStripK; ++k) a[k] = ld_stream(reinterpret_cast<const V*>(row) + lane + 32 * k);
#pragma unroll
            for (int k = 0; k < kFStripK; ++k) vfma_f<T>(acc + k * VN, reinterpret_cast<const T*>(&a[k]), q);
        } else {
#pragma unroll
            for (int k = 0; k < kFStripK; ++k) {
                const int64_t c = (int64_t)(32 * k + lane) * VN;
#pragma unroll
                for (int e = 0; e < VN; ++e)
                    if (c_strip + c + e < cols) acc[k * VN + e] = fma((double)row[c + e], q, acc[k * VN + e]);
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kFStripK; ++k)
#pragma unroll
        for (int e = 0; e < VN; ++e) red[warp * W + (32 * k + lane) * VN + e] = acc[k * VN + e];
    __syncthreads();
    double* out = nd.partial[j] + ch.chunk_in_node * cols;
    for (int c = threadIdx.x; c < W; c += kFThreads) {
        double s = 0.0;
#pragma unroll
        for (int ww = 0; ww < kFWarps; ++ww) s += red[ww * W + c];
        if (c_strip + c < cols) out[c_strip + c] = s;
    }
}

template <typename T>
__global__ void __launch_bounds__(kFThreads) k_fused_sweep(const FusedTables tb, int loss, int M, double rho) {
    __shared__ double red[kFWarps * kFStrip * (sizeof(T) == 8 ? 1 : 2)];
    __shared__ long long s_task;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (;;) {
        if (threadIdx.x == 0) s_task = (long long)atomicAdd(reinterpret_cast<unsigned long long*>(tb.task_counter), 1ull);
        __syncthreads();
        const int64_t t = s_task;
        __syncthreads();
        if (t >= tb.ntasks) break;
        int lo = 0, hi = tb.nseg - 1;          // last segment with start <= t
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (tb.segs[mid].t0 <= t) lo = mid; else hi = mid - 1;
        }
        const FusedSeg sg = tb.segs[lo];
        const FusedChunk ch = tb.chunks[sg.chunk];
        const FusedNode& nd = tb.nodes[ch.node];
        const int64_t u = t - sg.t0;
        if (!tb.active[ch.node]) continue;
        if (sg.type == 0) {
            double* slot = tb.sq_slots ? tb.sq_slots + (ch.a_slot0 + u) * kFWarps : nullptr;
            task_A<T>(nd, ch, u, loss, M, rho, lane, warp, slot);
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) {
                const int64_t rows = min((int64_t)kFWarps, ch.r1 - (ch.r0 + u * kFWarps));
                atomicAdd(tb.done + sg.chunk, (int)rows);
            }
        } else {
            if (threadIdx.x == 0) {
                const int need = (int)(ch.r1 - ch.r0);
                int spins = 0;
                while (atomicAdd(tb.done + sg.chunk, 0) < need) {
                    __nanosleep(200);
                    if (++spins > (1 << 26)) { asm volatile("trap;"); }
                }
                __threadfence();
            }
            __syncthreads();
            task_B<T>(nd, ch, u, lane, warp, red);
        }
    }
}

int fused_strip_width(int dtype) { return dtype == BICADMM_F64 ? kFStrip : 2 * kFStrip; }

int launch_fused_sweep(int dtype, const FusedTables& tb, int loss, int M, double rho, int grid, cudaStream_t s) {
    // reset the queue head and the per-chunk completion counters
    BIC_CUDA(cudaMemsetAsync(tb.task_counter, 0, sizeof(unsigned long long), s));
    BIC_CUDA(cudaMemsetAsync(tb.done, 0, sizeof(int) * (size_t)tb.nchunks, s));
    if (dtype == BICADMM_F64) k_fused_sweep<double><<<grid, kFThreads, 0, s>>>(tb, loss, M, rho);
    else k_fused_sweep<float><<<grid, kFThreads, 0, s>>>(tb, loss, M, rho);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

int fused_grid(int dtype, int sm_count) {
    int occ = 0;
    if (dtype == BICADMM_F64) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fused_sweep<double>, kFThreads, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fused_sweep<float>, kFThreads, 0);
    if (occ < 1) occ = 1;
    return occ * sm_count;
}

int fused_rows_per_task() { return kFWarps; }

}  // namespace bic
