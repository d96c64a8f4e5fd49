// k_fused3.cu -- warp-specialised single-HBM-read inner sweep.
//
// Same algebra as the two-pass sweep (Eqs. (22)-(24)) for nodes with one local
// block of n_j <= kF3Main*32*E columns.  One CTA per SM owns a contiguous row range
// (all local nodes concatenated).  14 "main" warps and 2 "prox" warps:
//
//   main, iteration k:  p_k partial dot  A[r_k,:] x          (A from HBM; x in smem)
//                       -> per-warp partials, mbarrier arrive (dot ready)
//                       acc[col] += A[r_{k-D}, col] q_{k-D}  (row re-read from L2:
//                       only D * G * row_bytes ~ 35 MB of new lines entered L2 since)
//   prox warp (r even / odd): wait dot ready, p = fixed-order sum of the partials,
//                       omega = prox(p + nu) (22), nu += p - omega (23),
//                       delta = omega - p - nu, q = p + delta -> smem, arrive (q ready)
//
// The serial per-sample prox (Newton with FP64 exp) is off the main warps' critical
// path: they wait for q_{k-D} only D rows later.  A is read from HBM once per sweep
// (the delayed re-read hits L2).  At node boundaries the CTA writes its partial
// products acc to partial[cta][col]; the next sweep's r is the fixed-order reduction
// over the CTAs that touched the node (bit-reproducible, no inter-CTA sync).
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace bic {

constexpr int kF3Main = 12;                 // main warps
constexpr int kF3ProxW = 4;                 // prox warps
constexpr int kF3Threads = 32 * (kF3Main + kF3ProxW);
constexpr int kF3MainT = 32 * kF3Main;      // 384 main threads
constexpr int kF3D = 3;                     // axpy delay in rows
constexpr int kF3Q = 8;                     // pipeline slots (> kF3D + prox lag)

__device__ __forceinline__ double f3_sigmoid(double a) {
    if (a >= 0.0) return 1.0 / (1.0 + exp(-a));
    const double e = exp(a);
    return e / (1.0 + e);
}

// w0: warm start (the previous sweep's omega of this sample); the root is the same.
__device__ double f3_prox(int loss, double rho, double b, double p, double w0) {
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
    double lo = p - 1.0 / rho, hi = p + 1.0 / rho;
    double w = (w0 > lo && w0 < hi) ? w0 : p;
    for (int it = 0; it < 60; ++it) {
        const double sg = f3_sigmoid(-b * w);
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

// ---- mbarrier helpers (shared::cta)
__device__ __forceinline__ void mb_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(count));
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(
        (unsigned)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{ .reg .pred P; WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra WAIT_%=; }" ::"r"(
            (unsigned)__cvta_generic_to_shared(b)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ double ldg_stream_d(const double* p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ldg_stream_d(const float* p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return (double)v;
}

template <typename T, int E>
__global__ void __launch_bounds__(kF3Threads, 1) k_fused3(const Fused2Args a, int loss, double rho) {
    extern __shared__ __align__(16) double xs[];          // x of the dot row's node (max_cols_pad doubles)
    __shared__ double dotp[kF3Q][kF3Main];
    __shared__ double qv[kF3Q];
    __shared__ __align__(8) uint64_t bar_dot[kF3Q], bar_q[kF3Q];
    __shared__ int x_node;                                 // node whose x is in xs
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t cta = blockIdx.x;
    const int64_t rb = cta * a.total_rows / gridDim.x, re = (cta + 1) * a.total_rows / gridDim.x;
    if (rb >= re) return;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kF3Q; ++s) { mb_init(&bar_dot[s], kF3Main); mb_init(&bar_q[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        x_node = -1;
    }
    auto node_of = [&](int64_t r, int from) {
        int k = from;
        while (k + 1 < a.nn && r >= a.row_off[k + 1]) ++k;
        return k;
    };
    // all threads load x of the first node
    int nd0 = node_of(rb, 0);
    for (int64_t c = threadIdx.x; c < a.ncols[nd0]; c += kF3Threads) xs[c] = a.x[nd0][c];
    __syncthreads();

    if (warp < kF3Main) {
        // ------------------------------------------------------------ main warps
        const int mt = threadIdx.x;                       // 0 .. kF3MainT-1
        int ndd = nd0, nda = nd0;                        // node of the dot row / of the axpy row
        double acc[E];
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = 0.0;
        auto flush = [&](int node) {
            const int64_t nc = a.ncols[node];
            double* out = a.partial[node] + (cta - a.cta_lo[node]) * nc;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int64_t c = mt + (int64_t)kF3MainT * e;
                if (c < nc) out[c] = acc[e];
                acc[e] = 0.0;
            }
        };
        for (int64_t k = rb; k < re + kF3D; ++k) {
            // ---- dot of row k
            if (k < re) {
                const int nn2 = node_of(k, ndd);
                if (nn2 != ndd) {
                    // x of the new node: main warps only (prox warps never read xs)
                    asm volatile("bar.sync 1, %0;" ::"n"(kF3MainT));
                    for (int64_t c = mt; c < a.ncols[nn2]; c += kF3MainT) xs[c] = a.x[nn2][c];
                    asm volatile("bar.sync 1, %0;" ::"n"(kF3MainT));
                    ndd = nn2;
                }
                const int s = (int)((k - rb) % kF3Q);
                double dot = 0.0;
                if (a.active[ndd]) {
                    const T* row = static_cast<const T*>(a.A[ndd]) + (k - a.row_off[ndd]) * a.lda[ndd];
                    const int64_t nc = a.ncols[ndd];
                    double v[E];            // all E loads in flight before the first FMA
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const int64_t c = mt + (int64_t)kF3MainT * e;
                        v[e] = c < nc ? (double)__ldg(row + c) : 0.0;
                    }
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const int64_t c = mt + (int64_t)kF3MainT * e;
                        if (c < nc) dot = fma(v[e], xs[c], dot);
                    }
                }
                dot = warp_sum(dot);
                if (lane == 0) {
                    dotp[s][warp] = dot;
                    mb_arrive(&bar_dot[s]);
                }
            }
            // ---- delayed axpy of row k - D
            const int64_t ra = k - kF3D;
            if (ra >= rb) {
                const int nn2 = node_of(ra, nda);
                if (nn2 != nda) {
                    if (a.active[nda]) flush(nda);
                    nda = nn2;
                }
                const int s = (int)((ra - rb) % kF3Q);
                const bool on = a.active[nda];
                double v[E];                // row re-read (L2) issued before waiting for q
                const T* row = static_cast<const T*>(a.A[nda]) + (ra - a.row_off[nda]) * a.lda[nda];
                const int64_t nc = a.ncols[nda];
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int64_t c = mt + (int64_t)kF3MainT * e;
                    v[e] = (on && c < nc) ? (double)__ldg(row + c) : 0.0;
                }
                mb_wait(&bar_q[s], (unsigned)(((ra - rb) / kF3Q) & 1));
                const double q = qv[s];
                if (on) {
#pragma unroll
                    for (int e = 0; e < E; ++e) acc[e] = fma(v[e], q, acc[e]);
                }
            }
        }
        if (a.active[nda]) flush(nda);
    } else if (lane == 0) {
        // ------------------------------------------------------------ prox warps (lane 0)
        const int pw = warp - kF3Main;
        int nd = nd0;
        for (int64_t r = rb + pw; r < re; r += kF3ProxW) {
            nd = node_of(r, nd);
            const int s = (int)((r - rb) % kF3Q);
            const int64_t rl = r - a.row_off[nd];
            // prefetchable loads (independent of the dot)
            const bool on = a.active[nd];
            double bl = 0.0, nu0 = 0.0, w0 = 0.0;
            if (on) {
                bl = (double)static_cast<const T*>(a.b[nd])[rl];
                nu0 = a.nu[nd][rl];
                w0 = a.delta[nd][rl] + a.p[nd][rl] + nu0;   // previous omega = delta + abar + nu
            }
            mb_wait(&bar_dot[s], (unsigned)(((r - rb) / kF3Q) & 1));
            double q = 0.0;
            if (on) {
                double p = 0.0;
#pragma unroll
                for (int w = 0; w < kF3Main; ++w) p += dotp[s][w];
                const double om = f3_prox(loss, rho, bl, p + nu0, w0);
                const double nu = nu0 + p - om;
                const double dl = om - p - nu;
                a.p[nd][rl] = p;
                a.nu[nd][rl] = nu;
                a.delta[nd][rl] = dl;
                if (a.e2row[nd]) a.e2row[nd][rl] = (p - om) * (p - om);
                q = p + dl;
            }
            qv[s] = q;
            mb_arrive(&bar_q[s]);
        }
    }
}

int fused3_max_cols(int dtype) { (void)dtype; return kF3MainT * 28; }

template <typename T>
static int f3_launch(int E, const Fused2Args& a, int loss, double rho, int grid, cudaStream_t s) {
    const size_t smem = (size_t)a.max_cols_pad * sizeof(double);
#define F3_CASE(EE)                                                                                          \
    case EE: {                                                                                               \
        static bool set = false;                                                                             \
        if (!set) {                                                                                          \
            if (cudaFuncSetAttribute(k_fused3<T, EE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != \
                cudaSuccess)                                                                                 \
                return BICADMM_ERR_CUDA;                                                                     \
            set = true;                                                                                      \
        }                                                                                                    \
        k_fused3<T, EE><<<grid, kF3Threads, smem, s>>>(a, loss, rho);                                        \
        break;                                                                                               \
    }
    switch (E) {
        F3_CASE(2) F3_CASE(4) F3_CASE(8) F3_CASE(12) F3_CASE(16) F3_CASE(24) F3_CASE(28)
    default: return BICADMM_ERR_INVALID;
    }
#undef F3_CASE
    return BICADMM_OK;
}

int launch_fused3(int dtype, const Fused2Args& a, int loss, double rho, int grid, cudaStream_t s) {
    int64_t maxc = 0;
    for (int k = 0; k < a.nn; ++k) maxc = a.ncols[k] > maxc ? a.ncols[k] : maxc;
    const int64_t e = (maxc + kF3MainT - 1) / kF3MainT;
    const int E = e <= 2 ? 2 : e <= 4 ? 4 : e <= 8 ? 8 : e <= 12 ? 12 : e <= 16 ? 16 : e <= 24 ? 24 : e <= 28 ? 28 : -1;
    if (E < 0 || (size_t)a.max_cols_pad * 8 > 200 * 1024) return BICADMM_ERR_INVALID;
    int rc = dtype == BICADMM_F64 ? f3_launch<double>(E, a, loss, rho, grid, s) : f3_launch<float>(E, a, loss, rho, grid, s);
    if (rc) return rc;
    BIC_LAUNCHED();
    return BICADMM_OK;
}

}  // namespace bic
