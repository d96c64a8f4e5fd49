#pragma once
// k_fused4.cuh -- single-HBM-read inner sweep on CTA pairs: the kernel
// template; instantiated per row-batch size R in k_fused4_r{1,2,4}.cu, launched from
// k_fused4.cu.
//
// Same algebra as the two-pass sweep (Eqs. (22)-(24)) for nodes with one local
// block.  A cluster of 2 CTAs (2 SMs) owns a contiguous row range; CTA h of the pair
// owns column half h of every row, so a ring of half-rows fits in shared memory even
// for wide rows (up to 210 KB: 5 x 40 KB at n = 10^4 FP64, 4 x 50 KB at 12,500, up to
// 32 slots for narrow rows):
//
//   producer warp : TMA bulk copy (cp.async.bulk, mbarrier complete_tx) of a half-row
//                   into the ring as soon as its slot is released
//   12 main warps : dot of half-row k with x (x half in registers) -> 12 partials,
//                   kept locally and sent to the peer CTA with st.async (mbarrier
//                   complete_tx on the peer's "dot" barrier: no cluster-scope fence);
//                   axpy acc[col] += A[k-D, col] q_{k-D} from the ring (no second read)
//   3 prox warps  : wait for the 24 partials of a row, p = fixed-order sum (identical
//                   in both CTAs), omega = prox(p + nu) (22), nu += p - omega (23),
//                   delta = omega - p - nu, q = p + delta; rank 0 stores p, nu, delta.
//
// Both CTAs compute the prox redundantly from bit-identical inputs, so the only
// cluster traffic per row is 12 doubles each way plus one 8-byte token from CTA 1 (it
// has read the row's p, nu, delta, which only CTA 0 overwrites).  Narrow rows run as
// 2, 3, 4 or 6 row groups of 12/g main warps (compiled per g).  A crosses HBM exactly
// once per sweep; partial products are written per (cluster, row group) and reduced in
// fixed order by the next sweep's Eq. (24) epilogue (bit-reproducible).
//
// Row batches: every role synchronises per batch of R consecutive rows of one node (one
// ring slot, one "full"/"empty"/"dot"/"q" barrier phase per batch), not per row.  The
// per-row cost of the kernel was almost entirely fixed synchronisation latency (mbarrier
// waits and arrives, the shuffle reduction, the cross-CTA publish: measured row period
// ~2,000-2,300 cycles per cluster at n = 2,500, 5,000 and 10,000 alike, tools/f4_trace.py),
// so a batch of R rows costs about as much as one row did.  R is chosen so that a slot
// (R half-rows) stays <= ~42 KB: R = 1 for FP64 n = 10^4 (40 KB half-rows: its bound is
// the TMA latency over the 5-slot ring), R = 2 for FP32 n = 10^4, R = 4 for narrow rows.
#include <cfloat>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace bic {

#ifndef BIC_F4_MAIN
#define BIC_F4_MAIN 12
#endif
constexpr int kF4Main = BIC_F4_MAIN;           // main warps per CTA
constexpr int kF4Prox = 3;                     // prox warps per CTA
constexpr int kF4Threads = 32 * (kF4Main + kF4Prox + 1);   // + 1 producer warp = 512
constexpr int kF4MainT = 32 * kF4Main;         // 384
#ifdef BIC_F4_CHECK
constexpr int kF4RingBytes = (kF4Main > 12 ? 202 : 208) * 1024;   // the check build's slot tags take 1.5 KB
#else
constexpr int kF4RingBytes = (kF4Main > 12 ? 204 : 210) * 1024;   // dynamic smem of the ring (static smem grows with kF4Main)
#endif
constexpr int kF4RingMax = 32;                 // ring depth in batches (runtime nring <= 32, by smem)
constexpr int kF4D = 2;                        // axpy delay (rows) when the axpy reads the smem ring
constexpr int kF4PF = 4;                       // prox input lookahead (rows of a prox worker)
// dot / q / token slots, indexed by row mod kF4Q.  A slot is reused kF4Q rows later; the
// peer CTA may run ahead of this CTA's prox warps by at most nring + ngrp (D + 1) rows (its
// producer is held by its ring, its main warps by the q of rows that need this CTA's dots),
// so f4_launch keeps nring + ngrp (D + 1) <= kF4Q (with 32 slots, n = 2000 FP64,
// 26 ring slots and 6 row groups exceeded it)
constexpr int kF4Q = 64;

// The logistic prox sits on every row's critical path, so its FP64
// pieces are latency-trimmed (tools/prox_latency2.cu: 2,220 -> 1,250 cycles per prox,
// results within 5e-16 of the libm version):
// exp: x = n ln2 + r (Cody-Waite, two-part ln2), |r| <= ln2/2, degree-11 Taylor evaluated by
// Estrin (depth 5; truncation < 2e-17 relative), 2^n by exponent construction (|x| < 700)
__device__ __forceinline__ double f4_exp(double x) {
    const double n = rint(x * 1.4426950408889634);
    double r = fma(n, -6.93147180369123816490e-01, x);
    r = fma(n, -1.90821492927058770002e-10, r);
    const double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
    const double c01 = fma(r, 1.0, 1.0), c23 = fma(r, 1.6666666666666666e-01, 0.5);
    const double c45 = fma(r, 8.333333333333333e-03, 4.1666666666666664e-02);
    const double c67 = fma(r, 1.984126984126984e-04, 1.388888888888889e-03);
    const double c89 = fma(r, 2.7557319223985893e-06, 2.48015873015873e-05);
    const double cab = fma(r, 2.505210838544172e-08, 2.755731922398589e-07);
    const double c03 = fma(r2, c23, c01), c47 = fma(r2, c67, c45), c8b = fma(r2, cab, c89);
    const double q = fma(r8, c8b, fma(r4, c47, c03));
    return q * __longlong_as_double(((long long)n + 1023) << 52);
}
// reciprocal: hardware approximation + two Newton refinements (~0.5 ulp)
__device__ __forceinline__ double f4_rcp(double a) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    double e = fma(-a, y, 1.0);
    y = fma(y, e, y);
    e = fma(-a, y, 1.0);
    return fma(y, e, y);
}
// sigma(t), overflow-safe: exp of -|t| only (|t| of a prox iterate is far below 700)
__device__ __forceinline__ double f4_sigmoid(double t) {
    const double e = f4_exp(-fabs(t));
    const double r = f4_rcp(1.0 + e);
    return t >= 0.0 ? r : e * r;
}

static __device__ double f4_prox(int loss, double rho, double b, double p, double w0) {
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
        const double sg = f4_sigmoid(-b * w);
        const double g = -b * sg + rho * (w - p);
        if (g > 0.0) hi = w; else lo = w;
        const double step = g * f4_rcp(sg * (1.0 - sg) + rho);
        // converged: quadratic convergence with |f''/2f'| <= 1/(8 rho) leaves an error below
        // 1e-19 |w| after a step <= 1e-9, so that step is accepted without another
        // evaluation (checked BEFORE the bracket safeguard, which would otherwise turn a
        // tiny step landing on the bracket into a bisection)
        if (fabs(step) <= 1e-9 * fmax(1.0, fabs(w))) { w -= step; break; }
        double wn = w - step;
        if (!(wn > lo && wn < hi)) wn = 0.5 * (lo + hi);
        w = wn;
    }
    return w;
}

// ---- PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned mapa(unsigned local, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
__device__ __forceinline__ void mb4_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mb4_arrive_local(uint64_t* b) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.release.cta.shared::cta.b64 st, [%0]; }" ::"r"(smem_u32(b))
                 : "memory");
}
__device__ __forceinline__ void mb4_arrive_remote(unsigned cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mb4_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// bounded waits: a protocol bug traps (error) instead of hanging the GPU
__device__ __forceinline__ bool mb4_try_cta(uint64_t* b, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{ .reg .pred P; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
        : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ bool mb4_try_cluster(uint64_t* b, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{ .reg .pred P; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
        : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
    return ok != 0;
}
// (a try_wait suspend-time hint of 1 or 20 us measured no better than plain polling)
__device__ __forceinline__ void mb4_wait_cta(uint64_t* b, unsigned parity) {
    for (unsigned it = 0; !mb4_try_cta(b, parity);)
        if (++it > (1u << 26)) asm volatile("trap;");
}
__device__ __forceinline__ void mb4_wait_cluster(uint64_t* b, unsigned parity) {
    for (long long it = 0; !mb4_try_cluster(b, parity); ++it)
        if (it > (1ll << 26)) asm volatile("trap;");
}
// asynchronous remote store that completes 8 bytes of the peer's mbarrier transaction
// count: no cluster-scope release fence (MEMBAR.GPU) per row, unlike st + remote arrive
__device__ __forceinline__ void st_async_f64(unsigned cluster_addr, double v, unsigned cluster_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(cluster_addr),
                 "d"(v), "r"(cluster_bar)
                 : "memory");
}
__device__ __forceinline__ void st_cluster_f64(unsigned cluster_addr, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(cluster_addr), "d"(v) : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// shared-memory vectors of the ring: 2 elements (float2 / double2).  Two, not four, FP32
// elements per vector: a half-row of n = 10^4 is 2,500 pairs over 384 lanes (at most 7 per
// lane, 14 elements, as with scalars); with float4 some warps carry 16 elements and the
// slowest warp sets the row period (measured 1.52 vs 1.30 ms per sweep at configs[1] FP32).
template <typename T> struct F4Vec;
template <> struct F4Vec<float> { using type = float2; };
template <> struct F4Vec<double> { using type = double2; };
__device__ __forceinline__ void f4_dot(const float2& v, const double* x, double& d) {
    d = fma((double)v.x, x[0], d);
    d = fma((double)v.y, x[1], d);
}
__device__ __forceinline__ void f4_dot(const double2& v, const double* x, double& d) {
    d = fma(v.x, x[0], d);
    d = fma(v.y, x[1], d);
}
__device__ __forceinline__ void f4_axpy(const float2& v, double q, double* acc) {
    acc[0] = fma((double)v.x, q, acc[0]);
    acc[1] = fma((double)v.y, q, acc[1]);
}
__device__ __forceinline__ void f4_axpy(const double2& v, double q, double* acc) {
    acc[0] = fma(v.x, q, acc[0]);
    acc[1] = fma(v.y, q, acc[1]);
}

// Debug timeline (variant builds only: tools/build_variant.sh ... -DBIC_F4_TRACE): clock64
// stamps of the first kF4TraceRows batches of cluster 0, both CTAs:
// [cta][batch][0 TMA issued, 1 dot start, 2 dot published (warp 0), 3 q wait done (warp 0,
// batch = the axpy batch), 4 slot released (warp 0), 5 dots complete (prox), 6 q published].
constexpr int kF4TraceRows = 1024;
#ifdef BIC_F4_TRACE
static __device__ long long* g_f4_trace = nullptr;   // one per translation unit (set by f4_trace_set)
#define F4_T(row, ev)                                                                       \
    do {                                                                                    \
        if (g_f4_trace && clu == 0 && (row) >= 0 && (row) < kF4TraceRows)                  \
            g_f4_trace[((int64_t)h * kF4TraceRows + (row)) * 8 + (ev)] = clock64();         \
    } while (0)
#else
#define F4_T(row, ev) \
    do {              \
    } while (0)
#endif

// One batch of rows: rows [r0, r0 + n) of node nd, n <= R; batches never span two nodes.
// Timing experiments only (tools/build_variant.sh ... -DBIC_F4_EXP=mask; results are wrong):
// 1 main warps skip the FMA blocks, 2 prox skips the prox (q = p), 4 main warps skip the q wait,
// 8 main warps skip the cross-CTA publish (the prox then waits for local dots only), 16 / 32
// fill qv and dotp with NaN / zero (and the ring with zero) at kernel start
#ifndef BIC_F4_EXP
#define BIC_F4_EXP 0
#endif


// Protocol check (variant builds only: tools/build_variant.sh ... -DBIC_F4_CHECK; compute-
// sanitizer is closed on this GPU pool): every row slot carries the global row index it
// holds -- written by each CTA's main warps for its own dots, sent to the peer with the dots
// (one more st.async per row, counted in the peer's expect_tx), and written by the prox warps
// next to q.  The prox warps check both dot tags of every row they reduce and the main warps
// the q tag of every row they accumulate; a slot reused too early or a barrier phase that
// completed for the wrong row shows up as a tag mismatch, counted in g_f4_errors
// (bicadmm_debug_f4_errors).
#ifdef BIC_F4_CHECK
static __device__ unsigned long long g_f4_errors = 0;
#define F4_CHECK_ON 1
#else
#define F4_CHECK_ON 0
#endif

struct F4Batch {
    int64_t r0;
    int n;
    int nd;
    int64_t nd_end;
};

// predicated shared-memory vector load (zero when the predicate is off)
template <typename V> __device__ __forceinline__ V f4_lds(unsigned addr, bool p);
template <> __device__ __forceinline__ float2 f4_lds<float2>(unsigned addr, bool p) {
    float2 v = make_float2(0.f, 0.f);
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q ld.shared.v2.f32 {%0, %1}, [%3]; }"
                 : "+f"(v.x), "+f"(v.y)
                 : "r"((int)p), "r"(addr));
    return v;
}
template <> __device__ __forceinline__ double2 f4_lds<double2>(unsigned addr, bool p) {
    double2 v = make_double2(0.0, 0.0);
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q ld.shared.v2.f64 {%0, %1}, [%3]; }"
                 : "+d"(v.x), "+d"(v.y)
                 : "r"((int)p), "r"(addr));
    return v;
}

// The axpy of batch b - D GR reads its rows from the batch's ring slot, held until then
// (measured alternatives -- an L2 re-read for the axpy, a register delay line -- were slower
// and are described in DESIGN.md section 6).
template <typename T, int E, int GR, int R>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kF4Threads, 1)
    k_fused4(const Fused2Args a, int loss, double rho, int nring, int dly) {
    const int D = dly;                   // axpy delay (in the group's own batches)
    constexpr int W = kF4Main / GR;      // warps of a row group
    constexpr int QB = kF4Q / R;         // batch slots of the dot / q barriers
    static_assert(kF4Q % R == 0 && (QB & (QB - 1)) == 0, "batch slots");
    extern __shared__ __align__(128) unsigned char f4_smem[];
    T* ring = reinterpret_cast<T*>(f4_smem);             // nring x R x half_pad elements
    __shared__ double dotp[kF4Q][2 * kF4Main];            // [row slot][cta * W + warp of the group]
    __shared__ double qv[kF4Q];
    __shared__ double tok[kF4Q];                          // CTA 1 -> CTA 0: row inputs read
#if F4_CHECK_ON
    __shared__ long long ctag[kF4Q], ptag[kF4Q], qtag[kF4Q];   // row index held by a slot (own / peer dots, q)
    for (int i = threadIdx.x; i < kF4Q; i += blockDim.x) ctag[i] = ptag[i] = qtag[i] = -1;
#endif
    __shared__ __align__(8) uint64_t bar_full[kF4RingMax], bar_empty[kF4RingMax], bar_dot[QB], bar_q[QB];
    const unsigned h = cluster_rank();                     // column half owned by this CTA
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t clu = blockIdx.x >> 1, nclu = gridDim.x >> 1;
    const int64_t rb = clu * a.total_rows / nclu, re = (clu + 1) * a.total_rows / nclu;
    const int64_t half_pad = ((a.max_cols_pad / 2 + 3) / 4) * 4 + 4;   // elements per half-row (>= ch)
    const int64_t slot_el = (int64_t)R * half_pad;                      // elements per ring slot
    // ring position (slot, phase of its w-th use) advanced incrementally: no division by nring
    struct RingPos {
        int s = 0;
        unsigned ph = 0;
        __device__ void adv(int n, int g) {   // g < n
            s += g;
            if (s >= n) { s -= n; ph ^= 1u; }
        }
    };
#if BIC_F4_EXP & 16
    for (int i = threadIdx.x; i < kF4Q; i += blockDim.x) qv[i] = __longlong_as_double(0x7ff4000000000000ll + 1);
    for (int i = threadIdx.x; i < kF4Q * 2 * kF4Main; i += blockDim.x) (&dotp[0][0])[i] = __longlong_as_double(0x7ff4000000000000ll + 2);
#endif
#if BIC_F4_EXP & 32
    for (int i = threadIdx.x; i < kF4Q; i += blockDim.x) qv[i] = 0.0;
    for (int i = threadIdx.x; i < kF4Q * 2 * kF4Main; i += blockDim.x) (&dotp[0][0])[i] = 0.0;
    for (int i = threadIdx.x; i < nring * (int)slot_el; i += blockDim.x) ring[i] = (T)0;
#endif
    if (threadIdx.x == 0) {
        for (int s = 0; s < nring; ++s) { mb4_init(&bar_full[s], 1); mb4_init(&bar_empty[s], W); }
        for (int s = 0; s < QB; ++s) { mb4_init(&bar_dot[s], W); mb4_init(&bar_q[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_sync_all();   // barriers of both CTAs initialised before any remote arrive
    if (rb >= re) { cluster_sync_all(); return; }
    auto node_of = [&](int64_t r, int from) {
        int k = from;
        while (k + 1 < a.nn && r >= a.row_off[k + 1]) ++k;
        return k;
    };
    // column split of node nd (ncols even, lda * sizeof(T) % 16 == 0): half 0 = [0, ch), half 1 = [ch, ncols),
    // ch % 4 == 0, so both halves start 16-byte aligned and hold whole 2-element vectors (TMA bulk copy)
    auto half_range = [&](int nd, int64_t& c0, int64_t& cn) {
        const int64_t nc = a.ncols[nd];
        const int64_t ch = ((nc / 2 + 3) / 4) * 4;
        c0 = h == 0 ? 0 : ch;
        cn = h == 0 ? ch : nc - ch;
    };
    auto nd_end_of = [&](int nd) { return nd + 1 < a.nn ? a.row_off[nd + 1] : INT64_MAX; };
    // the batch sequence of this cluster (identical in every role): R rows at a time, cut at
    // node boundaries and at the end of the cluster's row range
    auto first_batch = [&]() {
        F4Batch b;
        b.r0 = rb;
        b.nd = node_of(rb, 0);
        b.nd_end = nd_end_of(b.nd);
        b.n = (int)min((int64_t)R, min(b.nd_end, re) - rb);
        return b;
    };
    auto next_batch = [&](F4Batch& b) {
        b.r0 += b.n;
        if (b.r0 >= re) { b.n = 0; return; }
        if (b.r0 >= b.nd_end) {
            b.nd = node_of(b.r0, b.nd);
            b.nd_end = nd_end_of(b.nd);
        }
        b.n = (int)min((int64_t)R, min(b.nd_end, re) - b.r0);
    };

    if (warp == kF4Main + kF4Prox) {
        // ------------------------------------------------------------ producer (lane 0)
        if (lane == 0) {
            RingPos pw;
            int i = 0;
            for (F4Batch b = first_batch(); b.n > 0; next_batch(b), ++i, pw.adv(nring, 1)) {
                const int s = pw.s;
                if (i >= nring) mb4_wait_cta(&bar_empty[s], pw.ph ^ 1u);   // (w-1)-th release
                int64_t c0, cn;
                half_range(b.nd, c0, cn);
                // rounded up to a 16-byte multiple (FP32 half-rows of an odd number of pairs): the extra
                // elements are the row's own padding inside lda, never read by the main warps
                const unsigned bytes = (unsigned)(((cn * (int64_t)sizeof(T)) + 15) / 16 * 16);
                mb4_expect_tx(&bar_full[s], bytes * (unsigned)b.n);
                F4_T(i, 0);
                if (bytes)
                    for (int k = 0; k < b.n; ++k)
                        tma_bulk_g2s(ring + s * slot_el + k * half_pad,
                                     static_cast<const T*>(a.A[b.nd]) + (b.r0 + k - a.row_off[b.nd]) * a.lda[b.nd] + c0,
                                     bytes, &bar_full[s]);
            }
        }
    } else if (warp < kF4Main) {
        // ------------------------------------------------------------ main warps
        // GR groups of W warps; group gi owns batches gi, gi + GR, ... (GR = 1: all batches).
        // A lane owns the vectors v = mt + GT j (j < EV) of each half-row: VT = 2 elements
        // each, read from the ring slot with one 64-bit (FP32) or 128-bit (FP64) shared load.
        // Half-rows are whole vectors (launch_fused4), so a vector is either wholly inside the
        // node's half-row or wholly past it: the lane's valid vectors are the prefix j < jv.
        constexpr int VT = 2;
        constexpr int EV = E / VT;
        static_assert(E % VT == 0, "E must be a whole number of vectors");
        using V = typename F4Vec<T>::type;
        constexpr int GT = 32 * W;             // threads of a group (cover a half-row)
        const int gi = warp / W, wig = warp % W;
        const int mt = wig * 32 + lane;
        const unsigned peer = h ^ 1u;
        double xr[E], acc[E];
        int jv = 0, jva = 0, ndd = -1, nda = -1;
        auto valid_vectors = [&](int64_t cn) {   // j < result: vector mt + GT j lies inside [0, cn)
            const int64_t nv = cn / VT;
            return nv > mt ? (int)min((int64_t)EV, (nv - mt + GT - 1) / GT) : 0;
        };
        auto load_x = [&](int nd) {
            int64_t c0, cn;
            half_range(nd, c0, cn);
            jv = valid_vectors(cn);
#pragma unroll
            for (int j = 0; j < EV; ++j)
#pragma unroll
                for (int u = 0; u < VT; ++u) {
                    const int64_t c = (int64_t)VT * (mt + GT * j) + u;
                    xr[j * VT + u] = j < jv ? a.x[nd][c0 + c] : 0.0;
                }
        };
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = 0.0;
        int64_t ac0 = 0, acn = 0;
        auto flush = [&](int node) {   // partial row (cluster, group) of the node
            double* out = a.partial[node] + ((clu - a.cta_lo[node]) * GR + gi) * a.ncols[node] + ac0;
#pragma unroll
            for (int j = 0; j < EV; ++j)
#pragma unroll
                for (int u = 0; u < VT; ++u) {
                    if (j < jva) out[(int64_t)VT * (mt + GT * j) + u] = acc[j * VT + u];
                    acc[j * VT + u] = 0.0;
                }
        };
        RingPos pd, pa;   // ring slots of this group's batches (dot side, axpy side)
        pd.s = pa.s = gi;
        F4Batch bd = first_batch(), ba;
        for (int g = 0; g < gi; ++g) next_batch(bd);
        ba = bd;
        const int lag = D * GR;
        // One iteration = the dot of batch id (published to both CTAs' prox warps as soon as it is
        // done), then the axpy of batch id - lag once its q is ready.  Publishing before waiting
        // for q keeps lag + 1 batch periods between a dot and its axpy (computing the axpy first
        // measured 1.52 instead of 1.32 ms per sweep at configs[1] FP64).  Each block is straight
        // line: its shared loads are predicated (a vector past the half-row or a row past the
        // batch reads as zero), so the loads, widenings and FMAs of all j interleave.
        const unsigned rstride = (unsigned)(half_pad * sizeof(T));
        for (int id = gi;; id += GR) {
            const bool dodot = bd.n > 0;
            const int ia = id - lag;
            const bool doax = ia >= 0 && ba.n > 0;
            if (!dodot && !doax && ia >= 0) break;
            if (dodot) {
                if (bd.nd != ndd) {
                    ndd = bd.nd;
                    load_x(ndd);
                }
                const int s = pd.s;
                mb4_wait_cta(&bar_full[s], pd.ph);
                if (warp == 0 && lane == 0) F4_T(id, 1);
                pd.adv(nring, GR);
                const bool actd = a.active[ndd];
                const int nbd = bd.n;
                const unsigned sd = smem_u32(ring + s * slot_el) + (unsigned)(mt * sizeof(V));
                double d0[R], d1[R];
#pragma unroll
                for (int k = 0; k < R; ++k) d0[k] = d1[k] = 0.0;
#pragma unroll
                for (int j = 0; j < ((BIC_F4_EXP & 1) ? 0 : EV); ++j)
#pragma unroll
                    for (int k = 0; k < R; ++k) {
                        const V v = f4_lds<V>(sd + k * rstride + (unsigned)(GT * j * sizeof(V)), actd && j < jv && k < nbd);
                        f4_dot(v, &xr[j * VT], j & 1 ? d1[k] : d0[k]);
                    }
                double dot[R];
#pragma unroll
                for (int k = 0; k < R; ++k) dot[k] = d0[k] + d1[k];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                    for (int k = 0; k < R; ++k) dot[k] += __shfl_xor_sync(0xffffffffu, dot[k], o);
                if (lane == 0) {
                    const int qb = id & (QB - 1);
                    const int idx = (int)h * W + wig;
                    const unsigned pbar = mapa(smem_u32(&bar_dot[qb]), peer);
#pragma unroll
                    for (int k = 0; k < R; ++k)
                        if (k < nbd) {
                            double* dp = &dotp[qb * R + k][idx];
                            *dp = dot[k];
                            if (!(BIC_F4_EXP & 8)) st_async_f64(mapa(smem_u32(dp), peer), dot[k], pbar);
                        }
#if F4_CHECK_ON
                    if (wig == 0)
                        for (int k = 0; k < nbd; ++k) {   // own tag, and the row index to the peer's ptag
                            ctag[qb * R + k] = bd.r0 + k;
                            st_async_f64(mapa(smem_u32(&ptag[qb * R + k]), peer), __longlong_as_double(bd.r0 + k), pbar);
                        }
                    const unsigned ctx = 8u * (unsigned)nbd;
#else
                    const unsigned ctx = 0u;
#endif
                    // the peer group's W stores per row (+ on CTA 0 the peer's "inputs read" token per row)
                    if (wig == 0) mb4_expect_tx(&bar_dot[qb], (BIC_F4_EXP & 8) ? 0u : 8u * (unsigned)nbd * (W + (h == 0 ? 1 : 0)) + ctx);
                    else mb4_arrive_local(&bar_dot[qb]);
                    if (warp == 0) F4_T(id, 2);
                }
            }
            if (doax) {
                if (ba.nd != nda) {
                    if (nda >= 0 && a.active[nda]) flush(nda);
                    nda = ba.nd;
                    half_range(nda, ac0, acn);
                    jva = valid_vectors(acn);
                }
                const int qb = ia & (QB - 1);
                if (!(BIC_F4_EXP & 4)) mb4_wait_cta(&bar_q[qb], (unsigned)((ia / QB) & 1));
                if (warp == 0 && lane == 0) F4_T(ia, 3);
                const int nba = ba.n;
                double qq[R];
#pragma unroll
                for (int k = 0; k < R; ++k) qq[k] = k < nba ? qv[qb * R + k] : 0.0;
#if F4_CHECK_ON
                for (int k = 0; k < nba; ++k)
                    if (qtag[qb * R + k] != ba.r0 + k && lane == 0) atomicAdd(&g_f4_errors, 1ull);
#endif
                const int sa = pa.s;
                pa.adv(nring, GR);
                const bool acta = a.active[nda];
                const unsigned sx = smem_u32(ring + sa * slot_el) + (unsigned)(mt * sizeof(V));
#pragma unroll
                for (int j = 0; j < ((BIC_F4_EXP & 1) ? 0 : EV); ++j)
#pragma unroll
                    for (int k = 0; k < R; ++k) {
                        const V w = f4_lds<V>(sx + k * rstride + (unsigned)(GT * j * sizeof(V)), acta && j < jva && k < nba);
                        f4_axpy(w, qq[k], &acc[j * VT]);   // qq[k] = 0 past the batch: 0 * 0
                    }
                __syncwarp();   // every lane has read batch ia: release its slot to the producer
                if (lane == 0) mb4_arrive_local(&bar_empty[sa]);
                if (warp == 0 && lane == 0) F4_T(ia, 4);
            }
            for (int g = 0; g < GR; ++g) {
                if (dodot) next_batch(bd);
                if (doax) next_batch(ba);
            }
        }
        if (nda >= 0 && a.active[nda]) flush(nda);
    } else {
        // ------------------------------------------------------------ prox warps
        // Prox warp pw owns batches pw, pw + P, ... (P = kF4Prox); lane k < n handles row k of
        // the batch.  The per-sample inputs (b, nu, delta, p) are loaded kF4PF batches of the
        // warp ahead: under a saturated HBM a global load takes several microseconds, and
        // nothing else in the row's chain may wait on it.
        constexpr int P = kF4Prox;
        const int pw = warp - kF4Main;
        struct In { int nd; int64_t rl; bool on; double bl, nu0, w0; };
        auto fetch = [&](const F4Batch& b) {
            In v;
            v.on = false;
            v.nd = b.nd;
            v.rl = 0;
            v.bl = v.nu0 = v.w0 = 0.0;
            if (lane >= b.n) return v;
            v.rl = b.r0 + lane - a.row_off[b.nd];
            v.on = a.active[b.nd];
            if (v.on) {
                v.bl = (double)static_cast<const T*>(a.b[b.nd])[v.rl];
                v.nu0 = a.nu[b.nd][v.rl];
                v.w0 = a.delta[b.nd][v.rl] + a.p[b.nd][v.rl] + v.nu0;
            }
            return v;
        };
        // CTA 0 overwrites p, nu, delta of a row once it has both CTAs' dots; CTA 1 reads the
        // same entries.  CTA 1 therefore sends a token per row, data-dependent on its loaded
        // values, that completes 8 bytes of CTA 0's dot barrier for that row's batch: CTA 0
        // cannot write a row before CTA 1 has read it.  The tokens of batch i + P are sent
        // while batch i is processed, from inputs loaded kF4PF - 1 warp batches earlier.
        auto token = [&](int i, const F4Batch& b, const In& v) {
            if (!(BIC_F4_EXP & 8) && h == 1 && lane < b.n) {
                const int qb = i & (QB - 1);
                st_async_f64(mapa(smem_u32(&tok[qb * R + lane]), 0u), v.on ? v.w0 + v.bl : 0.0,
                             mapa(smem_u32(&bar_dot[qb]), 0u));
            }
        };
        auto adv = [&](F4Batch& b, int k) { for (int g = 0; g < k; ++g) next_batch(b); };
        static_assert(kF4PF == 4, "the prox lookahead is a 4-deep register rotation");
        F4Batch c0 = first_batch();
        adv(c0, pw);
        F4Batch c1 = c0, c2, c3;
        adv(c1, P);
        c2 = c1;
        adv(c2, P);
        c3 = c2;
        adv(c3, P);
        In b0 = fetch(c0), b1 = fetch(c1), b2 = fetch(c2), b3 = fetch(c3);
        int i = pw;
        // one row per batch: lane 0 alone runs the loop (no idle lanes polling the barriers)
        if (R == 1 && lane != 0) c0.n = 0;
        if (c0.n > 0) token(i, c0, b0);
        for (; c0.n > 0; i += P) {
            if (c1.n > 0) token(i + P, c1, b1);
            F4Batch c4 = c3;
            adv(c4, P);
            const In nb = fetch(c4);
            const int qb = i & (QB - 1);
            // the peer's dots arrive by st.async complete_tx on this CTA's barrier: observing the
            // phase (CTA-scope acquire, as for TMA) makes them visible; no cluster-scope acquire
            mb4_wait_cta(&bar_dot[qb], (unsigned)((i / QB) & 1));
            if (lane == 0) F4_T(i, 5);
#if F4_CHECK_ON
            if (lane < c0.n) {
                const int q = qb * R + lane;
                const long long want = c0.r0 + lane;
                if (ctag[q] != want || (!(BIC_F4_EXP & 8) && ptag[q] != want)) atomicAdd(&g_f4_errors, 1ull);
            }
#endif
            if (lane < c0.n) {
                const int q = qb * R + lane;
                double qq = 0.0;
                if (b0.on) {
                    // fixed-order sum of the 2W partials (four interleaved chains, then pairwise):
                    // identical in both CTAs
                    double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                    for (int w = 0; w < 2 * W; ++w) s4[w & 3] += dotp[q][w];
                    const double p = (s4[0] + s4[1]) + (s4[2] + s4[3]);
                    const double om = (BIC_F4_EXP & 2) ? p : f4_prox(loss, rho, b0.bl, p + b0.nu0, b0.w0);
                    const double nu = b0.nu0 + p - om;
                    const double dl = om - p - nu;
                    if (h == 0) {
                        a.p[b0.nd][b0.rl] = p;
                        a.nu[b0.nd][b0.rl] = nu;
                        a.delta[b0.nd][b0.rl] = dl;
                        if (a.e2row[b0.nd]) a.e2row[b0.nd][b0.rl] = (p - om) * (p - om);
                    }
                    qq = p + dl;
                }
                qv[q] = qq;
#if F4_CHECK_ON
                qtag[q] = c0.r0 + lane;
#endif
            }
            if (R > 1) __syncwarp();
            if (lane == 0) {
                mb4_arrive_local(&bar_q[qb]);
                F4_T(i, 6);
            }
            c0 = c1;
            c1 = c2;
            c2 = c3;
            c3 = c4;
            b0 = b1;
            b1 = b2;
            b2 = b3;
            b3 = nb;
        }
    }
    cluster_sync_all();   // no CTA exits while its peer may still write into its smem
}

// Launch one compiled instance (per-lane vector count EV in {1, 2, 4, 6, 7, 8, 9}).
template <typename T, int GR, int R>
int f4_launch_inst(int EV, const Fused2Args& a, int loss, double rho, int nring, int dly, size_t smem, int grid,
                   cudaStream_t s) {
    constexpr int VT = 2;
#define F4_CASE(EE)                                                                                        \
    case EE: {                                                                                             \
        static bool set = false;                                                                           \
        if (!set) {                                                                                        \
            if (cudaFuncSetAttribute(k_fused4<T, EE * VT, GR, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                     kF4RingBytes + 2048) != cudaSuccess)                                  \
                return BICADMM_ERR_CUDA;                                                                   \
            set = true;                                                                                    \
        }                                                                                                  \
        k_fused4<T, EE * VT, GR, R><<<grid, kF4Threads, smem, s>>>(a, loss, rho, nring, dly);              \
        break;                                                                                             \
    }
    switch (EV) {
        F4_CASE(1) F4_CASE(2) F4_CASE(4) F4_CASE(6) F4_CASE(7) F4_CASE(8) F4_CASE(9)
    default: return BICADMM_ERR_INVALID;
    }
#undef F4_CASE
    return cudaPeekAtLastError() == cudaSuccess ? BICADMM_OK : BICADMM_ERR_CUDA;
}

// per-R entry points (k_fused4_r{1,2,4}.cu)
int f4_launch_r1(int dtype, int GR, int EV, const Fused2Args& a, int loss, double rho, int nring, int dly, size_t smem,
                 int grid, cudaStream_t s);
int f4_launch_r2(int dtype, int GR, int EV, const Fused2Args& a, int loss, double rho, int nring, int dly, size_t smem,
                 int grid, cudaStream_t s);
int f4_launch_r4(int dtype, int GR, int EV, const Fused2Args& a, int loss, double rho, int nring, int dly, size_t smem,
                 int grid, cudaStream_t s);
int f4_errors_r1(unsigned long long* out);
int f4_errors_r2(unsigned long long* out);
int f4_errors_r4(unsigned long long* out);
int f4_trace_set_r1(void* p);
int f4_trace_set_r2(void* p);
int f4_trace_set_r4(void* p);

}  // namespace bic
