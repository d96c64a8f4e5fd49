// k_fused2.cu -- single-HBM-pass inner sweep, one CTA per SM.
//
// Same algebra as the two-pass sweep (Eqs. (22)-(24)) for nodes whose feature
// block is ONE local block with n_j <= kF2Threads * E columns.  CTA c owns the
// contiguous row range [c R / G, (c+1) R / G) of all local nodes concatenated.
// Rows stream HBM -> shared memory with cp.async into a double buffer (the next
// row is in flight while the current one is used); thread t owns columns
// t + 512 e and keeps x and the A^T q accumulators for them in registers.  Per row:
//   p = A[r,:] x            (per-thread FMAs, warp shuffles, fixed-order CTA sum)
//   thread 0: omega = prox(p + nu), nu += p - omega, delta = omega - p - nu  ((22),(23); M = 1)
//   acc[col] += A[r,col] (p + delta)   (the next sweep's GEMV-T products, same smem row)
// so A is read from HBM exactly once per sweep, with no inter-CTA synchronisation.
// At a node boundary / range end the CTA writes acc to partial[cta][col]; the next
// sweep's r = rho_l sum_cta partial + rho_c (z - u) is the fixed-order reduction over
// the CTAs that touched the node (bit-reproducible).
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace bic {

constexpr int kF2Threads = 512;
constexpr int kF2Warps = kF2Threads / 32;

__device__ __forceinline__ double f2_sigmoid(double a) {
    if (a >= 0.0) return 1.0 / (1.0 + exp(-a));
    const double e = exp(a);
    return e / (1.0 + e);
}

__device__ double f2_prox(int loss, double rho, double b, double p) {
    // M = 1 (one local block per node on this path)
    if (loss == BICADMM_LS) return (2.0 * b + rho * p) / (2.0 + rho);
    if (loss == BICADMM_HINGE) {
        const double pp = b * p;
        double y;
        if (pp > 1.0) y = pp;
        else if (pp + 1.0 / rho < 1.0) y = pp + 1.0 / rho;
        else y = 1.0;
        return b * y;
    }
    double lo = p - 1.0 / rho, hi = p + 1.0 / rho, w = p;
    for (int it = 0; it < 60; ++it) {
        const double sg = f2_sigmoid(-b * w);
        const double g = -b * sg + rho * (w - p);
        if (g > 0.0) hi = w; else lo = w;
        const double gp = sg * (1.0 - sg) + rho;
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

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;"); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;"); }

// row (bytes = ncols * sizeof(T), 16-byte aligned start) -> smem buffer
template <typename T>
__device__ __forceinline__ void f2_issue(T* dst, const T* __restrict__ row, int64_t ncols) {
    const int64_t bytes = ncols * (int64_t)sizeof(T);
    const int64_t n16 = bytes >> 4;
    const char* src = reinterpret_cast<const char*>(row);
    char* d = reinterpret_cast<char*>(dst);
    for (int64_t k = threadIdx.x; k < n16; k += kF2Threads) cp_async16(d + 16 * k, src + 16 * k);
    const int64_t done = n16 << 4;
    for (int64_t k = done / 4 + threadIdx.x; k < bytes / 4; k += kF2Threads) cp_async4(d + 4 * k, src + 4 * k);
}

template <typename T, int E>
__global__ void __launch_bounds__(kF2Threads, 1) k_fused2(const Fused2Args a, int loss, double rho) {
    extern __shared__ __align__(16) unsigned char f2_smem[];
    T* buf[2] = {reinterpret_cast<T*>(f2_smem), reinterpret_cast<T*>(f2_smem) + a.max_cols_pad};
    __shared__ double red[kF2Warps];
    __shared__ double s_q;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t cta = blockIdx.x;
    const int64_t rb = cta * a.total_rows / gridDim.x, re = (cta + 1) * a.total_rows / gridDim.x;
    if (rb >= re) return;
    int nd = 0;
    while (nd + 1 < a.nn && rb >= a.row_off[nd + 1]) ++nd;
    double acc[E], xr[E];
    auto load_node = [&](int node) {
        const double* x = a.x[node];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int64_t c = threadIdx.x + (int64_t)kF2Threads * e;
            xr[e] = c < a.ncols[node] ? x[c] : 0.0;
            acc[e] = 0.0;
        }
    };
    load_node(nd);
    double e2 = 0.0;
    auto node_of = [&](int64_t r, int from) {
        int k = from;
        while (k + 1 < a.nn && r >= a.row_off[k + 1]) ++k;
        return k;
    };
    // prologue: row rb -> buf[0]
    f2_issue<T>(buf[0], static_cast<const T*>(a.A[nd]) + (rb - a.row_off[nd]) * a.lda[nd], a.ncols[nd]);
    cp_commit();
    for (int64_t r = rb; r < re; ++r) {
        const int cb = (int)((r - rb) & 1);
        if (r + 1 < re) {
            const int n2 = node_of(r + 1, nd);
            f2_issue<T>(buf[cb ^ 1], static_cast<const T*>(a.A[n2]) + (r + 1 - a.row_off[n2]) * a.lda[n2],
                        a.ncols[n2]);
        }
        cp_commit();
        cp_wait1();
        __syncthreads();
        const bool last = r + 1 == re;
        const bool cross = !last && nd + 1 < a.nn && r + 1 >= a.row_off[nd + 1];
        if (!a.active[nd]) {           // uniform per CTA: skip the row, keep the node's state
            if (cross) { ++nd; load_node(nd); }
            __syncthreads();
            continue;
        }
        const T* row = buf[cb];
        const int64_t ncols = a.ncols[nd];
        double dot = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int64_t c = threadIdx.x + (int64_t)kF2Threads * e;
            if (c < ncols) dot = fma((double)row[c], xr[e], dot);
        }
        dot = warp_sum(dot);
        if (lane == 0) red[warp] = dot;
        __syncthreads();
        if (threadIdx.x == 0) {
            double p = 0.0;
#pragma unroll
            for (int w = 0; w < kF2Warps; ++w) p += red[w];
            const int64_t rl = r - a.row_off[nd];
            const double bl = (double)static_cast<const T*>(a.b[nd])[rl];
            const double nu0 = a.nu[nd][rl];
            const double om = f2_prox(loss, rho, bl, p + nu0);
            const double nu = nu0 + p - om;
            const double dl = om - p - nu;
            a.p[nd][rl] = p;
            a.nu[nd][rl] = nu;
            a.delta[nd][rl] = dl;
            e2 += (p - om) * (p - om);
            s_q = p + dl;
        }
        __syncthreads();
        const double q = s_q;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int64_t c = threadIdx.x + (int64_t)kF2Threads * e;
            if (c < ncols) acc[e] = fma((double)row[c], q, acc[e]);
        }
        if (last || cross) {
            double* out = a.partial[nd] + (cta - a.cta_lo[nd]) * ncols;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int64_t c = threadIdx.x + (int64_t)kF2Threads * e;
                if (c < ncols) out[c] = acc[e];
            }
            if (threadIdx.x == 0 && a.sq_slots) a.sq_slots[a.slot0[nd] + (cta - a.cta_lo[nd])] = e2;
            e2 = 0.0;
            if (cross) {
                ++nd;
                load_node(nd);
            }
        }
        __syncthreads();   // buf[cb] is refilled by the next iteration's prefetch
    }
    cp_wait0();
}

int fused2_max_cols(int dtype) { (void)dtype; return kF2Threads * 20; }

template <typename T>
static int f2_launch(int E, const Fused2Args& a, int loss, double rho, int grid, cudaStream_t s) {
    const size_t smem = 2 * (size_t)a.max_cols_pad * sizeof(T);
#define F2_CASE(EE)                                                                                         \
    case EE: {                                                                                              \
        static bool set = false;                                                                            \
        if (!set) {                                                                                         \
            if (cudaFuncSetAttribute(k_fused2<T, EE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != \
                cudaSuccess)                                                                                \
                return BICADMM_ERR_CUDA;                                                                    \
            set = true;                                                                                     \
        }                                                                                                   \
        k_fused2<T, EE><<<grid, kF2Threads, smem, s>>>(a, loss, rho);                                       \
        break;                                                                                              \
    }
    switch (E) {
        F2_CASE(2) F2_CASE(4) F2_CASE(8) F2_CASE(12) F2_CASE(16) F2_CASE(20)
    default: return BICADMM_ERR_INVALID;
    }
#undef F2_CASE
    return BICADMM_OK;
}

int launch_fused2(int dtype, const Fused2Args& a, int loss, double rho, int grid, cudaStream_t s) {
    int64_t maxc = 0;
    for (int k = 0; k < a.nn; ++k) maxc = a.ncols[k] > maxc ? a.ncols[k] : maxc;
    const int64_t e = (maxc + kF2Threads - 1) / kF2Threads;
    const int E = e <= 2 ? 2 : e <= 4 ? 4 : e <= 8 ? 8 : e <= 12 ? 12 : e <= 16 ? 16 : e <= 20 ? 20 : -1;
    if (E < 0) return BICADMM_ERR_INVALID;
    if (2 * (size_t)a.max_cols_pad * (dtype == BICADMM_F64 ? 8 : 4) > 200 * 1024) return BICADMM_ERR_INVALID;
    int rc = dtype == BICADMM_F64 ? f2_launch<double>(E, a, loss, rho, grid, s) : f2_launch<float>(E, a, loss, rho, grid, s);
    if (rc) return rc;
    BIC_LAUNCHED();
    return BICADMM_OK;
}

}  // namespace bic
