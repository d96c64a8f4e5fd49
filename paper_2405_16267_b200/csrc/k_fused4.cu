// k_fused4.cu -- single-HBM-read inner sweep on CTA pairs.
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
#include <cfloat>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace bic {

constexpr int kF4Main = 12;                    // main warps per CTA
constexpr int kF4Prox = 3;                     // prox warps per CTA
constexpr int kF4Threads = 32 * (kF4Main + kF4Prox + 1);   // + 1 producer warp = 512
constexpr int kF4MainT = 32 * kF4Main;         // 384
constexpr int kF4RingMax = 32;                 // half-row ring depth (runtime nring <= 32 = kF4Q, by smem)
constexpr int kF4D = 2;                        // axpy delay (rows) when the axpy reads the smem ring
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

__device__ double f4_prox(int loss, double rho, double b, double p, double w0) {
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

// The axpy of row k - D reads the row from its smem ring slot, held until then (measured
// alternatives -- an L2 re-read for the axpy, a register delay line -- were slower and are
// described in DESIGN.md section 6).
template <typename T, int E, int GR>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kF4Threads, 1)
    k_fused4(const Fused2Args a, int loss, double rho, int nring, int dly, int ngrp) {
    const int D = dly;   // axpy delay (rows; in a group's own rows when ngrp > 1)
    // row groups: the 12 main warps form ngrp groups of W warps; group gi owns the
    // rows rb + gi, rb + gi + ngrp, ...  For narrow rows this overlaps the per-row latency
    // chain of ngrp rows.  Every row's dot has W partials per CTA.
    ngrp = GR;                           // GR groups of W = 12 / GR warps, fixed at compile time
    const int W = kF4Main / ngrp;
    extern __shared__ __align__(128) unsigned char f4_smem[];
    T* ring = reinterpret_cast<T*>(f4_smem);             // nring x half_pad elements
    __shared__ double dotp[kF4Q][2 * kF4Main];            // [slot][cta * 12 + warp]
    __shared__ double qv[kF4Q];
    __shared__ double tok[kF4Q];                          // CTA 1 -> CTA 0: row inputs read
    __shared__ __align__(8) uint64_t bar_full[kF4RingMax], bar_empty[kF4RingMax], bar_dot[kF4Q], bar_q[kF4Q];
    const unsigned h = cluster_rank();                     // column half owned by this CTA
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t clu = blockIdx.x >> 1, nclu = gridDim.x >> 1;
    const int64_t rb = clu * a.total_rows / nclu, re = (clu + 1) * a.total_rows / nclu;
    const int64_t half_pad = ((a.max_cols_pad / 2 + 3) / 4) * 4 + 4;   // elements per ring slot (>= ch)
    // ring position (slot, phase of its w-th use) advanced incrementally: no division by nring
    struct RingPos {
        int s = 0;
        unsigned ph = 0;
        __device__ void next(int n) { if (++s == n) { s = 0; ph ^= 1u; } }
        __device__ void adv(int n, int g) {   // g < n
            if (GR == 1) { next(n); return; }
            s += g;
            if (s >= n) { s -= n; ph ^= 1u; }
        }
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < nring; ++s) { mb4_init(&bar_full[s], 1); mb4_init(&bar_empty[s], W); }
        for (int s = 0; s < kF4Q; ++s) { mb4_init(&bar_dot[s], W); mb4_init(&bar_q[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_sync_all();   // barriers of both CTAs initialised before any remote arrive
    if (rb >= re) { cluster_sync_all(); return; }
    auto node_of = [&](int64_t r, int from) {
        int k = from;
        while (k + 1 < a.nn && r >= a.row_off[k + 1]) ++k;
        return k;
    };
    // column split of node nd (ncols * sizeof(T) % 16 == 0): half 0 = [0, ch), half 1 = [ch, ncols), ch % 4 == 0,
    // so both halves start 16-byte aligned and are whole 16-byte multiples (TMA bulk copy)
    auto half_range = [&](int nd, int64_t& c0, int64_t& cn) {
        const int64_t nc = a.ncols[nd];
        const int64_t ch = ((nc / 2 + 3) / 4) * 4;
        c0 = h == 0 ? 0 : ch;
        cn = h == 0 ? ch : nc - ch;
    };
    const int nd0 = node_of(rb, 0);
    // rows are visited in increasing order at every call site: keep the current node's end
    // row in a register instead of re-scanning row_off (parameter space) for every row
    struct NodeCur {
        int nd;
        int64_t end;
    };
    auto cur_init = [&](int nd) { return NodeCur{nd, nd + 1 < a.nn ? a.row_off[nd + 1] : INT64_MAX}; };
    auto cur_adv = [&](NodeCur& c, int64_t r) {   // true when r starts another node
        if (r < c.end) return false;
        c = cur_init(node_of(r, c.nd));
        return true;
    };

    if (warp == kF4Main + kF4Prox) {
        // ------------------------------------------------------------ producer (lane 0)
        if (lane == 0) {
            NodeCur nc = cur_init(nd0);
            RingPos pw;
            for (int64_t r = rb; r < re; ++r, pw.next(nring)) {
                cur_adv(nc, r);
                const int nd = nc.nd;
                const int s = pw.s;
                if (r - rb >= nring) mb4_wait_cta(&bar_empty[s], pw.ph ^ 1u);   // (w-1)-th release
                int64_t c0, cn;
                half_range(nd, c0, cn);
                const unsigned bytes = (unsigned)(cn * (int64_t)sizeof(T));
                mb4_expect_tx(&bar_full[s], bytes);
                if (bytes)
                    tma_bulk_g2s(ring + s * half_pad,
                                 static_cast<const T*>(a.A[nd]) + (r - a.row_off[nd]) * a.lda[nd] + c0, bytes,
                                 &bar_full[s]);
            }
        }
    } else if (GR != 1 && warp < kF4Main) {
        // ------------------------------------------------------------ main warps (row groups)
        const int gi = warp / W, wig = warp % W;
        const int GT = 32 * W;                 // threads of a group (cover a half-row)
        const int mt = wig * 32 + lane;
        const unsigned peer = h ^ 1u;
        int ndd = nd0, nda = nd0;
        int64_t ndd_end = cur_init(nd0).end, nda_end = ndd_end;
        double xr[E], acc[E];
        int64_t hc0, hcn;
        auto load_x = [&](int nd) {
            half_range(nd, hc0, hcn);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int64_t c = mt + (int64_t)GT * e;
                xr[e] = c < hcn ? a.x[nd][hc0 + c] : 0.0;
            }
        };
        load_x(ndd);
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = 0.0;
        int64_t ac0, acn;
        half_range(nda, ac0, acn);
        auto flush = [&](int node) {   // partial row (cluster, group) of the node
            double* out = a.partial[node] + ((clu - a.cta_lo[node]) * ngrp + gi) * a.ncols[node] + ac0;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int64_t c = mt + (int64_t)GT * e;
                if (c < acn) out[c] = acc[e];
                acc[e] = 0.0;
            }
        };
        RingPos pd, pa;   // ring slots of this group's rows (dot side, axpy side)
        pd.s = pa.s = gi;
        const int64_t lag = (int64_t)D * ngrp;
        for (int64_t k = rb + gi; k < re + lag; k += ngrp) {
            if (k < re) {
                if (k >= ndd_end) {
                    ndd = node_of(k, ndd);
                    ndd_end = cur_init(ndd).end;
                    load_x(ndd);
                }
                const int s = pd.s;
                mb4_wait_cta(&bar_full[s], pd.ph);
                pd.adv(nring, ngrp);
                const T* row = ring + s * half_pad;
                double dot = 0.0;
                if (a.active[ndd]) {
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const int64_t c = mt + (int64_t)GT * e;
                        if (c < hcn) dot = fma((double)row[c], xr[e], dot);
                    }
                }
                dot = warp_sum(dot);
                if (lane == 0) {
                    const int q = (int)((k - rb) % kF4Q);
                    const int idx = (int)h * W + wig;
                    dotp[q][idx] = dot;
                    st_async_f64(mapa(smem_u32(&dotp[q][idx]), peer), dot, mapa(smem_u32(&bar_dot[q]), peer));
                    // the peer group's W stores (+ on CTA 0 the peer's "inputs read" token)
                    if (wig == 0) mb4_expect_tx(&bar_dot[q], 8u * (W + (h == 0 ? 1 : 0)));
                    else mb4_arrive_local(&bar_dot[q]);
                }
            }
            const int64_t ra = k - lag;
            if (ra >= rb) {
                if (ra >= nda_end) {
                    if (a.active[nda]) flush(nda);
                    nda = node_of(ra, nda);
                    nda_end = cur_init(nda).end;
                    half_range(nda, ac0, acn);
                }
                const int q = (int)((ra - rb) % kF4Q);
                mb4_wait_cta(&bar_q[q], (unsigned)(((ra - rb) / kF4Q) & 1));
                const double qq = qv[q];
                const int s = pa.s;
                pa.adv(nring, ngrp);
                const T* row = ring + s * half_pad;
                if (a.active[nda]) {
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const int64_t c = mt + (int64_t)GT * e;
                        if (c < acn) acc[e] = fma((double)row[c], qq, acc[e]);
                    }
                }
                __syncwarp();
                if (lane == 0) mb4_arrive_local(&bar_empty[s]);
            }
        }
        if (a.active[nda]) flush(nda);
    } else if (GR == 1 && warp < kF4Main) {
        // ------------------------------------------------------------ main warps (one group)
        const int mt = threadIdx.x;
        const unsigned peer = h ^ 1u;
        int ndd = nd0, nda = nd0;
        int64_t ndd_end = cur_init(nd0).end, nda_end = ndd_end;
        double xr[E], acc[E];
        int64_t hc0, hcn;
        auto load_x = [&](int nd) {
            half_range(nd, hc0, hcn);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int64_t c = mt + (int64_t)kF4MainT * e;
                xr[e] = c < hcn ? a.x[nd][hc0 + c] : 0.0;
            }
        };
        load_x(ndd);
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = 0.0;
        int64_t ac0, acn;
        half_range(nda, ac0, acn);
        auto flush = [&](int node) {
            double* out = a.partial[node] + (clu - a.cta_lo[node]) * a.ncols[node] + ac0;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int64_t c = mt + (int64_t)kF4MainT * e;
                if (c < acn) out[c] = acc[e];
                acc[e] = 0.0;
            }
        };
        RingPos pd, pa;
        for (int64_t k = rb; k < re + D; ++k) {
            if (k < re) {
                if (k >= ndd_end) {
                    ndd = node_of(k, ndd);
                    ndd_end = cur_init(ndd).end;
                    load_x(ndd);
                }
                const int s = pd.s;
                mb4_wait_cta(&bar_full[s], pd.ph);
                pd.next(nring);
                const T* row = ring + s * half_pad;
                double dot = 0.0;
                if (a.active[ndd]) {
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const int64_t c = mt + (int64_t)kF4MainT * e;
                        if (c < hcn) dot = fma((double)row[c], xr[e], dot);
                    }
                }
                dot = warp_sum(dot);
                if (lane == 0) {
                    const int q = (int)((k - rb) % kF4Q);
                    const int idx = (int)h * kF4Main + warp;
                    dotp[q][idx] = dot;
                    st_async_f64(mapa(smem_u32(&dotp[q][idx]), peer), dot, mapa(smem_u32(&bar_dot[q]), peer));
                    // the peer's 12 stores (+ on CTA 0 the peer's "inputs read" token)
                    if (warp == 0) mb4_expect_tx(&bar_dot[q], 8u * (kF4Main + (h == 0 ? 1 : 0)));
                    else mb4_arrive_local(&bar_dot[q]);
                }
            }
            const int64_t ra = k - D;
            if (ra >= rb) {
                if (ra >= nda_end) {
                    if (a.active[nda]) flush(nda);
                    nda = node_of(ra, nda);
                    nda_end = cur_init(nda).end;
                    half_range(nda, ac0, acn);
                }
                const int q = (int)((ra - rb) % kF4Q);
                const bool on = a.active[nda];
                    mb4_wait_cta(&bar_q[q], (unsigned)(((ra - rb) / kF4Q) & 1));
                    const double qq = qv[q];
                    const int s = pa.s;
                    pa.next(nring);
                    const T* row = ring + s * half_pad;
                    if (on) {
#pragma unroll
                        for (int e = 0; e < E; ++e) {
                            const int64_t c = mt + (int64_t)kF4MainT * e;
                            if (c < acn) acc[e] = fma((double)row[c], qq, acc[e]);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mb4_arrive_local(&bar_empty[s]);
            }
        }
        if (a.active[nda]) flush(nda);
    } else if (lane == 0) {
        // ------------------------------------------------------------ prox warps (lane 0)
        // The per-sample inputs (b, nu, delta, p) of a warp's next row are loaded while it
        // waits for the current row's dots (their global-load latency is ~1 us, several row
        // periods when rows are narrow).
        const int pw = warp - kF4Main;
        int nd = nd0;
        struct In { int nd; int64_t rl; bool on; double bl, nu0, w0; };
        NodeCur pc = cur_init(nd0);
        auto fetch = [&](int64_t r, int from) {
            (void)from;
            In v;
            cur_adv(pc, r);
            v.nd = pc.nd;
            v.rl = r - a.row_off[v.nd];
            v.on = a.active[v.nd];
            v.bl = v.nu0 = v.w0 = 0.0;
            if (v.on) {
                v.bl = (double)static_cast<const T*>(a.b[v.nd])[v.rl];
                v.nu0 = a.nu[v.nd][v.rl];
                v.w0 = a.delta[v.nd][v.rl] + a.p[v.nd][v.rl] + v.nu0;
            }
            return v;
        };
        // CTA 0 overwrites p, nu, delta of a row once it has both CTAs' dots; CTA 1 reads the
        // same entries.  CTA 1 therefore sends a token, data-dependent on its loaded values, that
        // completes 8 bytes of CTA 0's dot barrier for that row: CTA 0 cannot write a row before
        // CTA 1 has read it.
        auto token = [&](int64_t r, const In& v) {
            if (h == 1) {
                const int qt = (int)((r - rb) % kF4Q);
                st_async_f64(mapa(smem_u32(&tok[qt]), 0u), v.on ? v.w0 + v.bl : 0.0, mapa(smem_u32(&bar_dot[qt]), 0u));
            }
        };
        In cur = fetch(rb + pw < re ? rb + pw : rb, nd);
        if (rb + pw < re) token(rb + pw, cur);
        for (int64_t r = rb + pw; r < re; r += kF4Prox) {
            In nxt = cur;
            if (r + kF4Prox < re) {
                nxt = fetch(r + kF4Prox, cur.nd);
                token(r + kF4Prox, nxt);
            }
            const int q = (int)((r - rb) % kF4Q);
            // the peer's dots arrive by st.async complete_tx on this CTA's barrier: observing the
            // phase (CTA-scope acquire, as for TMA) makes them visible; no cluster-scope acquire
            mb4_wait_cta(&bar_dot[q], (unsigned)(((r - rb) / kF4Q) & 1));
            double qq = 0.0;
            if (cur.on) {
                double p = 0.0;
#pragma unroll
                for (int w = 0; w < 2 * W; ++w) p += dotp[q][w];
                const double om = f4_prox(loss, rho, cur.bl, p + cur.nu0, cur.w0);
                const double nu = cur.nu0 + p - om;
                const double dl = om - p - nu;
                if (h == 0) {
                    a.p[cur.nd][cur.rl] = p;
                    a.nu[cur.nd][cur.rl] = nu;
                    a.delta[cur.nd][cur.rl] = dl;
                    if (a.e2row[cur.nd]) a.e2row[cur.nd][cur.rl] = (p - om) * (p - om);
                }
                qq = p + dl;
            }
            qv[q] = qq;
            mb4_arrive_local(&bar_q[q]);
            cur = nxt;
        }
        (void)nd;
    }
    cluster_sync_all();   // no CTA exits while its peer may still write into its smem
}

int fused4_max_cols(int dtype) { (void)dtype; return 2 * kF4MainT * 17; }

static size_t f4_slot_bytes(const Fused2Args& a, size_t es) { return (size_t)(((a.max_cols_pad / 2 + 3) / 4) * 4 + 4) * es; }
static int f4_ring(const Fused2Args& a, size_t es) {
    const char* e = getenv("BICADMM_F4_RING");
    int r = (int)((210 * 1024) / f4_slot_bytes(a, es));
    if (e) r = atoi(e) < r ? atoi(e) : r;
    return r > kF4RingMax ? kF4RingMax : r;
}

// Row groups for narrow rows: the largest ngrp in {6, 4, 3, 2} whose W = 12/ngrp warps
// still cover a half-row with <= 17 elements per thread (every group count is compiled
// with W fixed: no spills up to E = 17; BICADMM_F4_GROUPS overrides).  Measured: n = 4000
// FP64 (Table-1 rows) 3 groups 1.87 ms per sweep vs 2 groups 2.05 ms (2.44 ms with the
// runtime-W kernel); C5 shard (n_j = 6,250) 2 groups 17.7 ms vs 1 group 23.9 ms.
int fused4_groups(int dtype, int64_t max_cols) {
    (void)dtype;
    const int64_t half = (max_cols + 1) / 2 + 2;
    int g = 1;
    const int cand[4] = {6, 4, 3, 2};
    for (int k = 0; k < 4; ++k)
        if (half <= (int64_t)32 * (kF4Main / cand[k]) * 17) { g = cand[k]; break; }
    if (const char* e = getenv("BICADMM_F4_GROUPS")) {
        const int v = atoi(e);
        if ((v == 1 || v == 2 || v == 3 || v == 4 || v == 6) && half <= (int64_t)32 * (kF4Main / v) * 17) g = v;
    }
    return g;
}

// axpy delay D (in the group's own rows; the ring holds about ngrp (D + 1) rows):
// one group: D = 2 (measured best at C2 FP64, 5 slots; BICADMM_F4_D overrides) but at
// most nring - 3, so 2 slots keep loading (C3 shard, 4 slots of 50 KB: D = 1 runs at
// 6.15 TB/s, D = 2 at 5.87).  Always ngrp * D <= nring - 2.
static int f4_delay(int nring, int ngrp) {
    static int d = [] { const char* e = getenv("BICADMM_F4_D"); return e ? (atoi(e) < 1 ? 1 : atoi(e)) : 0; }();
    // ngrp > 1: D = 1 (a group's next row comes ngrp rows later, so the prox chain already
    // has ngrp row periods), which keeps the most slots loading
    int v = d ? d : (ngrp == 1 ? kF4D : 1);
    if (v < 1) v = 1;
    while (v > 1 && ngrp * v > nring - 2) --v;
    if (!d && ngrp == 1 && v > nring - 3) v = nring - 3 < 1 ? 1 : nring - 3;
    return v;
}

template <typename T, int GR>
static int f4_launch(int E, int ngrp, const Fused2Args& a, int loss, double rho, int grid, cudaStream_t s) {
    int nring = f4_ring(a, sizeof(T));
    if (nring < 4 || ngrp >= nring - 1) return BICADMM_ERR_INVALID;
    while (nring > 4 && nring + ngrp * (f4_delay(nring, ngrp) + 1) > kF4Q) --nring;   // slot reuse bound
    if (nring + ngrp * (f4_delay(nring, ngrp) + 1) > kF4Q) return BICADMM_ERR_INVALID;
    const size_t smem = (size_t)nring * f4_slot_bytes(a, sizeof(T));
#define F4_CASE(EE)                                                                                            \
    case EE: {                                                                                                 \
        static bool set = false;                                                                               \
        if (!set) {                                                                                            \
            if (cudaFuncSetAttribute(k_fused4<T, EE, GR>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                     212 * 1024) != cudaSuccess)                                               \
                return BICADMM_ERR_CUDA;                                                                       \
            set = true;                                                                                        \
        }                                                                                                      \
        k_fused4<T, EE, GR><<<grid, kF4Threads, smem, s>>>(a, loss, rho, nring, f4_delay(nring, ngrp), ngrp); \
        break;                                                                                                 \
    }
    switch (E) {
        F4_CASE(2) F4_CASE(4) F4_CASE(8) F4_CASE(12) F4_CASE(14) F4_CASE(16) F4_CASE(17)
    default: return BICADMM_ERR_INVALID;
    }
#undef F4_CASE
    return BICADMM_OK;
}

int launch_fused4(int dtype, const Fused2Args& a, int loss, double rho, int grid, cudaStream_t s) {
    int64_t maxc = 0;
    for (int k = 0; k < a.nn; ++k) maxc = a.ncols[k] > maxc ? a.ncols[k] : maxc;
    const int64_t half = (maxc + 1) / 2 + 2;
    const int ngrp = fused4_groups(dtype, maxc);
    const int64_t gt = 32 * (kF4Main / ngrp);
    const int64_t e = (half + gt - 1) / gt;
    const int E = e <= 2 ? 2 : e <= 4 ? 4 : e <= 8 ? 8 : e <= 12 ? 12 : e <= 14 ? 14 : e <= 16 ? 16 : e <= 17 ? 17 : -1;
    if (E < 0 || f4_ring(a, dtype == BICADMM_F64 ? 8 : 4) < 4 || (grid & 1)) return BICADMM_ERR_INVALID;
    // TMA bulk copies: both half-rows start 16-byte aligned (ch % 4 == 0, lda * size % 16 == 0)
    // and are whole 16-byte multiples
    const int64_t es = dtype == BICADMM_F64 ? 8 : 4;
    for (int k = 0; k < a.nn; ++k) if ((a.ncols[k] * es) % 16 || (a.lda[k] * es) % 16) return BICADMM_ERR_INVALID;
    int rc;
#define F4_GROUPS(TT)                                                                  \
    switch (ngrp) {                                                                    \
    case 1: rc = f4_launch<TT, 1>(E, 1, a, loss, rho, grid, s); break;                 \
    case 2: rc = f4_launch<TT, 2>(E, 2, a, loss, rho, grid, s); break;                 \
    case 3: rc = f4_launch<TT, 3>(E, 3, a, loss, rho, grid, s); break;                 \
    case 4: rc = f4_launch<TT, 4>(E, 4, a, loss, rho, grid, s); break;                 \
    case 6: rc = f4_launch<TT, 6>(E, 6, a, loss, rho, grid, s); break;                 \
    default: rc = BICADMM_ERR_INVALID;                                                 \
    }
    if (dtype == BICADMM_F64) { F4_GROUPS(double) } else { F4_GROUPS(float) }
#undef F4_GROUPS
    if (rc) return rc;
    BIC_LAUNCHED();
    return BICADMM_OK;
}

}  // namespace bic
