// k_outer.cu -- the global (consensus) step of Bi-cADMM, replicated on every rank
// (Algorithm 1 "Global Updates").
//
//   Collect  : wbar = (1/N) sum_i (x_i + u_i)                       (DESIGN R1)
//   (7b)     : (z, t) = argmin_{||z||_1 <= t} (N rho_c/2)||z - wbar||^2 + (rho_b/2)(s'z - t + v)^2
//              exact: z_l = sgn(w_l) max(|w_l| - tau d_l, 0), d_l = 1 - s_l sgn(w_l),
//              tau the root of N rho_c tau = rho_b (psi(tau) - v), psi(tau) = sum d_l |z_l(tau)|
//              (DESIGN R3).  Root: 16-way multisection on the IEEE bit
//              patterns of tau to isolate the active set, then the exact segment formula.
//   (13)     : s = clamp((t - v)/Mcap, -1, 1) sgn(z) 1_T, T = top-kappa |z| (ties -> lower
//              index; DESIGN R4).  Device radix select on the uint64 bit patterns of |z|.
//   (14)     : g = z's - t, v += g                                  (DESIGN R5)
//   (9)      : u_ij += x_ij - z_j
//   (15)     : p_r = sum_i ||x_i - z||, d_r = sqrt(N) rho_c ||z - z_prev||, b_r = |g|
// The global step is O(n) and latency-bound; it runs in single-CTA kernels with
// fixed-order block reductions so every rank computes bit-identical z, s, v.
#include "common.cuh"
#include "kernels.h"

namespace bic {

constexpr int kOuterThreads = 1024;
// short vectors (configs[0]: n = 50) run the same kernels with 8 warps: the step is a chain of
// block barriers and cross-warp reductions whose cost grows with the warp count
constexpr int kOuterThreadsSmall = 256;
constexpr int64_t kOuterSmall = 8192;
constexpr int kProbes = 15;  // interior probes per multisection pass (16-way)

__device__ __forceinline__ uint64_t dkey(double a) { return (uint64_t)__double_as_longlong(a); }
__device__ __forceinline__ double kdbl(uint64_t k) { return __longlong_as_double((long long)k); }

// ------------------------------------------------------------------ (7b)
template <int NT>
__global__ void __launch_bounds__(NT) k_zt(int64_t len, int N, double rho_c, double rho_b,
                                                     double* __restrict__ wsum, const double* __restrict__ s,
                                                     double* __restrict__ wbar, double* __restrict__ z,
                                                     double* __restrict__ z_prev, OuterScalars* sc, WsumIn cw) {
    __shared__ double scratch[32];
    __shared__ double probe_red[32][kProbes + 1];
    __shared__ int probe_cnt[32][kProbes + 1];
    __shared__ uint64_t s_lo, s_hi;
    __shared__ int s_clo, s_chi, s_done;
    const double v = sc->v;
    const double Nd = (double)N, Nrc = Nd * rho_c;
    double psi0 = 0.0, sw = 0.0, bmax = 0.0;
    for (int64_t l = threadIdx.x; l < len; l += NT) {
        double ws;
        if (cw.x_all) {   // Collect fused in (single rank, short vectors): k_wsum's sum, same order
            ws = 0.0;
            for (int i = 0; i < cw.nl; ++i) ws += cw.x_all[(int64_t)i * cw.stride + l] + cw.u_all[(int64_t)i * cw.stride + l];
            wsum[l] = ws;
        } else {
            ws = wsum[l];
        }
        const double w = ws / Nd;
        wbar[l] = w;
        z_prev[l] = z[l];
        const double d = 1.0 - s[l] * sgn(w);
        psi0 += d * fabs(w);
        sw += s[l] * w;
        if (d > 0.0 && w != 0.0) bmax = fmax(bmax, fabs(w) / d);
    }
    psi0 = block_sum(psi0, scratch);
    sw = block_sum(sw, scratch);
    bmax = block_max(bmax, scratch);

    double tau = 0.0;
    const bool case1 = psi0 <= v;
    if (!case1) {
        // f(tau) = N rho_c tau - rho_b (psi(tau) - v): increasing; f(0) < 0.
        // f(bmax) = N rho_c bmax + rho_b v (psi(bmax) = 0).
        double Asum, Bsum;
        if (Nrc * bmax + rho_b * v <= 0.0) {
            Asum = 0.0; Bsum = 0.0;   // every shrinkable coordinate is zero
        } else {
            // early exit: the closed form below depends only on the active set
            // {l : |w_l|/d_l > tau}; once the bracket holds no breakpoint |w_l|/d_l
            // (count(lo) == count(hi), the count is monotone in tau) that set is fixed,
            // so stopping there gives bit-for-bit the same tau as narrowing to one ulp.
            int c0 = 0;
            for (int64_t l = threadIdx.x; l < len; l += NT) {
                const double w = wbar[l];
                const double dl = 1.0 - s[l] * sgn(w);
                c0 += (dl > 0.0 && w != 0.0 && fabs(w) / dl > 0.0);
            }
            c0 = (int)block_sum((double)c0, scratch);
            if (threadIdx.x == 0) { s_lo = 0; s_hi = dkey(bmax); s_clo = c0; s_chi = 0; s_done = 0; }
            __syncthreads();
            const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
            for (int pass = 0; pass < 40; ++pass) {
                const uint64_t lo = s_lo, hi = s_hi;
                if (hi - lo <= 1 || s_done) break;
                const uint64_t d = hi - lo;
                double tp[kProbes], acc[kProbes];
                int cn[kProbes];
#pragma unroll
                for (int p = 0; p < kProbes; ++p) {
                    const uint64_t kp = lo + (d / 16) * (uint64_t)(p + 1) + ((d % 16) * (uint64_t)(p + 1)) / 16;
                    tp[p] = kdbl(kp);
                    acc[p] = 0.0;
                    cn[p] = 0;
                }
                for (int64_t l = threadIdx.x; l < len; l += NT) {
                    const double w = wbar[l];
                    const double dl = 1.0 - s[l] * sgn(w);
                    if (dl > 0.0) {
                        const double aw = fabs(w);
                        const double bl = w != 0.0 ? aw / dl : -1.0;
#pragma unroll
                        for (int p = 0; p < kProbes; ++p) {
                            acc[p] += dl * fmax(aw - tp[p] * dl, 0.0);
                            cn[p] += bl > tp[p];
                        }
                    }
                }
#pragma unroll
                for (int p = 0; p < kProbes; ++p) {
                    const double t = warp_sum(acc[p]);
                    const int c = __reduce_add_sync(0xffffffffu, cn[p]);
                    if (lane == 0) { probe_red[wid][p] = t; probe_cnt[wid][p] = c; }
                }
                __syncthreads();
                if (wid == 0) {
                    // lane p < kProbes sums probe p over the warps (ascending warp order, as a
                    // serial loop would); the new bracket is [probe best, first probe above it]
                    const int p = lane;
                    const uint64_t kp = lo + (d / 16) * (uint64_t)(p + 1) + ((d % 16) * (uint64_t)(p + 1)) / 16;
                    double psi = 0.0;
                    int cp = 0;
                    if (p < kProbes)
                        for (int ww = 0; ww < NT / 32; ++ww) {
                            psi += probe_red[ww][p];
                            cp += probe_cnt[ww][p];
                        }
                    const bool neg = p < kProbes && Nrc * kdbl(kp) - rho_b * (psi - v) <= 0.0;
                    const unsigned bneg = __ballot_sync(0xffffffffu, neg);
                    const int best = bneg ? 31 - __clz((int)bneg) : -1;   // largest probe with f <= 0
                    const uint64_t nlo = best >= 0 ? (uint64_t)__shfl_sync(0xffffffffu, (long long)kp, best) : lo;
                    const int clo = best >= 0 ? __shfl_sync(0xffffffffu, cp, best) : s_clo;
                    const unsigned bup = __ballot_sync(0xffffffffu, p < kProbes && p > best && kp < hi && kp > nlo);
                    const int up = bup ? __ffs((int)bup) - 1 : -1;
                    const uint64_t nhi = up >= 0 ? (uint64_t)__shfl_sync(0xffffffffu, (long long)kp, up) : hi;
                    const int chi = up >= 0 ? __shfl_sync(0xffffffffu, cp, up) : s_chi;
                    if (lane == 0) {
                        s_lo = nlo; s_hi = nhi; s_clo = clo; s_chi = chi;
                        s_done = clo == chi;
                    }
                }
                __syncthreads();
            }
            const double tlo = kdbl(s_lo);
            double a = 0.0, b = 0.0;
            for (int64_t l = threadIdx.x; l < len; l += NT) {
                const double w = wbar[l];
                const double dl = 1.0 - s[l] * sgn(w);
                if (dl > 0.0 && w != 0.0 && fabs(w) / dl > tlo) { a += dl * fabs(w); b += dl * dl; }
            }
            Asum = block_sum(a, scratch);
            Bsum = block_sum(b, scratch);
        }
        tau = rho_b * (Asum - v) / (Nrc + rho_b * Bsum);
    }
    double l1 = 0.0, dz2 = 0.0;
    for (int64_t l = threadIdx.x; l < len; l += NT) {
        const double w = wbar[l];
        double zl;
        if (case1) zl = w;
        else {
            const double dl = 1.0 - s[l] * sgn(w);
            zl = sgn(w) * fmax(fabs(w) - tau * dl, 0.0);
        }
        z[l] = zl;
        l1 += fabs(zl);
        const double e = zl - z_prev[l];
        dz2 += e * e;
    }
    l1 = block_sum(l1, scratch);
    dz2 = block_sum(dz2, scratch);
    if (threadIdx.x == 0) {
        sc->t = case1 ? sw + v : l1;
        sc->tau = tau;
        sc->dz2 = dz2;
        sc->psi0 = psi0;
    }
}

int launch_zt(int64_t len, int N, double rho_c, double rho_b, double* wsum, const double* s, double* wbar,
              double* z, double* z_prev, OuterScalars* sc, cudaStream_t st, WsumIn cw) {
    if (len <= kOuterSmall) k_zt<kOuterThreadsSmall><<<1, kOuterThreadsSmall, 0, st>>>(len, N, rho_c, rho_b, wsum, s, wbar, z, z_prev, sc, cw);
    else k_zt<kOuterThreads><<<1, kOuterThreads, 0, st>>>(len, N, rho_c, rho_b, wsum, s, wbar, z, z_prev, sc, cw);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

// ------------------------------------------------------------------ top-kappa selection
// Radix select (8 passes x 8 bits, MSB first) of the kk-th largest key among keys
// of |z|; returns threshold key K and the number `take` of elements with key == K
// that belong to T (lowest indices first).  If nonzero_only, zero keys never count.
struct TopK { uint64_t K; int64_t take; int64_t kk; };

template <int NT>
__device__ TopK radix_topk(int64_t len, int64_t kk, const double* __restrict__ z, bool nonzero_only) {
    __shared__ int hist[256];
    __shared__ uint64_t s_prefix;
    __shared__ int64_t s_rem, s_nz;
    TopK r;
    if (nonzero_only) {
        int cnt = 0;
        for (int64_t l = threadIdx.x; l < len; l += NT) cnt += z[l] != 0.0;
        if (threadIdx.x == 0) s_nz = 0;
        __syncthreads();
        atomicAdd(reinterpret_cast<unsigned long long*>(&s_nz), (unsigned long long)cnt);
        __syncthreads();
        if (kk > s_nz) kk = s_nz;
    }
    r.kk = kk;
    if (kk <= 0) { r.K = ~0ull; r.take = 0; return r; }
    if (threadIdx.x == 0) { s_prefix = 0; s_rem = kk; }
    __syncthreads();
    uint64_t mask = 0;
    for (int pass = 0; pass < 8; ++pass) {
        const int shift = 56 - 8 * pass;
        for (int b = threadIdx.x; b < 256; b += NT) hist[b] = 0;
        __syncthreads();
        const uint64_t prefix = s_prefix;
        for (int64_t l = threadIdx.x; l < len; l += NT) {
            const uint64_t key = dkey(fabs(z[l]));
            if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            // the bin holding the rem-th largest key: lane k owns bins 255 - 8k .. 248 - 8k, an
            // inclusive scan of the lane counts from the top finds the lane, which then walks
            // its 8 bins (the same choice as a serial walk down from bin 255)
            const int lane = threadIdx.x;
            const int64_t rem = s_rem;
            int hb[8], loc = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) { hb[k] = hist[255 - 8 * lane - k]; loc += hb[k]; }
            int inc = loc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            const int exc = inc - loc;
            const bool mine = exc < rem && rem <= inc;
            if (mine) {
                int64_t cum = exc;
                int sel = 0;
                int64_t r2 = rem;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (cum + hb[k] >= rem) { sel = 255 - 8 * lane - k; r2 = rem - cum; break; }
                    cum += hb[k];
                }
                s_prefix = prefix | ((uint64_t)sel << shift);
                s_rem = r2;
            }
            // (no bin reaches rem -- not reachable with kk <= len -- leaves prefix and rem as they are)
        }
        mask |= (uint64_t)255 << shift;
        __syncthreads();
    }
    r.K = s_prefix;
    r.take = s_rem;
    __syncthreads();
    return r;
}

// Visit elements of T in ascending index order, contiguous range per thread.
// f(l, rank_in_T_for_this_thread_ordering) is called for members.
template <int NT, typename F>
__device__ void for_members(int64_t len, const double* __restrict__ z, const TopK& tk, bool nonzero_only,
                            int64_t* scan_scratch, F f) {
    const int64_t per = (len + NT - 1) / NT;
    const int64_t l0 = threadIdx.x * per, l1 = l0 + per < len ? l0 + per : len;
    int64_t eq = 0, mem = 0;
    for (int64_t l = l0; l < l1; ++l) {
        const uint64_t key = dkey(fabs(z[l]));
        if (nonzero_only && key == 0) continue;
        if (key == tk.K) ++eq;
    }
    int64_t total;
    const int64_t eq_before = block_exclusive_scan(eq, scan_scratch, &total);
    // members in this thread's range = (#key > K) + min(max(take - eq_before, 0), eq)
    for (int64_t l = l0; l < l1; ++l) {
        const uint64_t key = dkey(fabs(z[l]));
        if (nonzero_only && key == 0) continue;
        if (key > tk.K && tk.kk > 0) ++mem;
    }
    int64_t take_here = tk.take - eq_before;
    if (take_here < 0) take_here = 0;
    if (take_here > eq) take_here = eq;
    mem += take_here;
    int64_t mem_total;
    const int64_t mem_before = block_exclusive_scan(mem, scan_scratch, &mem_total);
    int64_t seen_eq = 0, pos = mem_before;
    for (int64_t l = l0; l < l1; ++l) {
        const uint64_t key = dkey(fabs(z[l]));
        if (nonzero_only && key == 0) continue;
        bool in = false;
        if (tk.kk > 0) {
            if (key > tk.K) in = true;
            else if (key == tk.K) { in = seen_eq < take_here; ++seen_eq; }
        }
        if (in) f(l, pos++);
    }
}

template <int NT>
__global__ void __launch_bounds__(NT) k_s_update(int64_t len, int64_t kappa, const double* __restrict__ z,
                                                           double* __restrict__ s, OuterScalars* sc) {
    __shared__ double scratch[32];
    __shared__ int64_t scan_scratch[32];
    const double t = sc->t, v = sc->v;
    const int64_t kk = kappa < len ? kappa : len;
    const TopK tk = radix_topk<NT>(len, kk, z, false);
    for (int64_t l = threadIdx.x; l < len; l += NT) s[l] = 0.0;
    __syncthreads();
    double mc = 0.0;
    for_members<NT>(len, z, tk, false, scan_scratch, [&](int64_t l, int64_t) { mc += fabs(z[l]); });
    const double mcap = block_sum(mc, scratch);
    const double scale = mcap > 0.0 ? fmin(fmax((t - v) / mcap, -1.0), 1.0) : 0.0;
    if (mcap > 0.0)
        for_members<NT>(len, z, tk, false, scan_scratch, [&](int64_t l, int64_t) { s[l] = scale * sgn(z[l]); });
    __syncthreads();
    double zs = 0.0;
    for (int64_t l = threadIdx.x; l < len; l += NT) zs += z[l] * s[l];
    zs = block_sum(zs, scratch);
    if (threadIdx.x == 0) {
        const double g = zs - t;
        sc->mcap = mcap;
        sc->g = g;
        sc->v = v + g;
    }
}

// len <= 256 (configs[0]): one element per thread; T = the elements whose rank under
// (|z| descending, index ascending) is below kappa -- the same set as the radix select with
// its ties-to-lower-index rule (DESIGN R4), found with one barrier instead of 8 select passes
constexpr int kRankThreads = 256;
__device__ __forceinline__ bool rank_member(int64_t len, int64_t kk, const double* __restrict__ z, bool nonzero_only,
                                            uint64_t* keys) {
    const int l = threadIdx.x;
    const uint64_t key = l < len ? dkey(fabs(z[l])) : 0ull;
    keys[l] = key;
    __syncthreads();
    if (l >= len || kk <= 0 || (nonzero_only && key == 0)) return false;
    int64_t rank = 0;
    for (int k = 0; k < len; ++k) {
        const uint64_t o = keys[k];
        rank += o > key || (o == key && k < l);
    }
    return rank < kk;
}

__global__ void __launch_bounds__(kRankThreads) k_s_update_rank(int64_t len, int64_t kappa, const double* __restrict__ z,
                                                               double* __restrict__ s, OuterScalars* sc) {
    __shared__ double scratch[32];
    __shared__ uint64_t keys[kRankThreads];
    const double t = sc->t, v = sc->v;
    const int64_t kk = kappa < len ? kappa : len;
    const int l = threadIdx.x;
    const bool in = rank_member(len, kk, z, false, keys);
    const double zl = l < len ? z[l] : 0.0;
    const double mcap = block_sum(in ? fabs(zl) : 0.0, scratch);
    const double scale = mcap > 0.0 ? fmin(fmax((t - v) / mcap, -1.0), 1.0) : 0.0;
    const double sl = in && mcap > 0.0 ? scale * sgn(zl) : 0.0;
    if (l < len) s[l] = sl;
    const double zs = block_sum(zl * sl, scratch);
    if (threadIdx.x == 0) {
        const double g = zs - t;
        sc->mcap = mcap;
        sc->g = g;
        sc->v = v + g;
    }
}

__global__ void __launch_bounds__(kRankThreads) k_support_rank(int64_t len, int64_t kappa, const double* __restrict__ z,
                                                              int64_t* __restrict__ support, int64_t* count) {
    __shared__ uint64_t keys[kRankThreads];
    __shared__ int64_t scan_scratch[32];
    const int64_t kk = kappa < len ? kappa : len;
    const bool in = rank_member(len, kk, z, true, keys);
    int64_t total;
    const int64_t pos = block_exclusive_scan((int64_t)in, scan_scratch, &total);   // ascending index order
    if (in) support[pos] = threadIdx.x;
    if (threadIdx.x == 0) *count = total;
}

int launch_s_update(int64_t len, int64_t kappa, const double* z, double* s, OuterScalars* sc, cudaStream_t st) {
    if (len <= kRankThreads) k_s_update_rank<<<1, kRankThreads, 0, st>>>(len, kappa, z, s, sc);
    else if (len <= kOuterSmall) k_s_update<kOuterThreadsSmall><<<1, kOuterThreadsSmall, 0, st>>>(len, kappa, z, s, sc);
    else k_s_update<kOuterThreads><<<1, kOuterThreads, 0, st>>>(len, kappa, z, s, sc);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

template <int NT>
__global__ void __launch_bounds__(NT) k_support(int64_t len, int64_t kappa, const double* __restrict__ z,
                                                          int64_t* __restrict__ support, int64_t* count) {
    __shared__ int64_t scan_scratch[32];
    const int64_t kk = kappa < len ? kappa : len;
    const TopK tk = radix_topk<NT>(len, kk, z, true);
    for_members<NT>(len, z, tk, true, scan_scratch, [&](int64_t l, int64_t pos) { support[pos] = l; });
    if (threadIdx.x == 0) *count = tk.kk;
}

int launch_support(int64_t len, int64_t kappa, const double* z, int64_t* support, int64_t* count, cudaStream_t st) {
    if (len <= kRankThreads) k_support_rank<<<1, kRankThreads, 0, st>>>(len, kappa, z, support, count);
    else if (len <= kOuterSmall) k_support<kOuterThreadsSmall><<<1, kOuterThreadsSmall, 0, st>>>(len, kappa, z, support, count);
    else k_support<kOuterThreads><<<1, kOuterThreads, 0, st>>>(len, kappa, z, support, count);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

// ------------------------------------------------------------------ Collect / (9) / (15)
__global__ void k_wsum(int64_t len, int64_t stride, const double* __restrict__ x_all,
                       const double* __restrict__ u_all, int nl, double* __restrict__ wsum) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= len) return;
    double acc = 0.0;
    for (int i = 0; i < nl; ++i) acc += x_all[(int64_t)i * stride + l] + u_all[(int64_t)i * stride + l];
    wsum[l] = acc;
}

int launch_wsum(int64_t len, int64_t stride, const double* x_all, const double* u_all, int nl, double* wsum,
                cudaStream_t s) {
    k_wsum<<<(unsigned)((len + 255) / 256), 256, 0, s>>>(len, stride, x_all, u_all, nl, wsum);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

struct UBatch {
    BlockVec b[kMaxDesc];
    int nb;
};
constexpr int kUPer = 4;  // elements per thread

// mode 0: u_ij += x_ij - z_j, partials of ||x_ij - z_j||^2   (Eq. (9) + Eq. (15) p_r)
// mode 1: partials of ||x_ij - u_ij||^2 with u := x_old            (inner tol criterion)
__global__ void __launch_bounds__(kUThreads) k_u_update(const __grid_constant__ UBatch B, const double* __restrict__ z,
                                                        double* __restrict__ partial, int64_t partial_base, int mode) {
    __shared__ double scratch[32];
    const int64_t cta = blockIdx.x;
    int bi = 0;
    while (bi + 1 < B.nb && cta >= B.b[bi + 1].cta_begin) ++bi;
    const BlockVec& V = B.b[bi];
    const int64_t e0 = (cta - V.cta_begin) * (kUThreads * kUPer);
    double sq = 0.0;
#pragma unroll
    for (int k = 0; k < kUPer; ++k) {
        const int64_t e = e0 + threadIdx.x + k * kUThreads;
        if (e < V.len) {
            const double x = V.x[e];
            if (mode == 0) {
                const double d = x - z[V.c0 + e];
                V.u[e] += d;
                sq += d * d;
            } else {
                const double d = x - V.u[e];
                sq += d * d;
            }
        }
    }
    sq = block_sum(sq, scratch);
    if (threadIdx.x == 0) partial[partial_base + cta] = sq;
}

int launch_u_update(BlockVec* bv, int nb, const double* z, double* partial, cudaStream_t s, int mode) {
    int64_t base = 0;
    for (int b0 = 0; b0 < nb; b0 += kMaxDesc) {
        UBatch B;
        B.nb = nb - b0 < kMaxDesc ? nb - b0 : kMaxDesc;
        int64_t t = 0;
        for (int k = 0; k < B.nb; ++k) {
            B.b[k] = bv[b0 + k];
            B.b[k].cta_begin = t;
            bv[b0 + k].cta_begin = base + t;   // record global partial offsets for node_sq
            t += (B.b[k].len + kUThreads * kUPer - 1) / (kUThreads * kUPer);
        }
        if (t > 0) {
            k_u_update<<<(unsigned)t, kUThreads, 0, s>>>(B, z, partial, base, mode);
            BIC_LAUNCHED();
        }
        base += t;
    }
    return BICADMM_OK;
}

// out[node[k]] = sum of parts[k][0..count[k]) (fixed order) for each listed node
struct SegArgs {
    const double* ptr[kMaxDesc];
    int64_t count[kMaxDesc];
    int32_t node[kMaxDesc];
    int n;
};
__global__ void k_seg_sums(const __grid_constant__ SegArgs A, double* __restrict__ out) {
    for (int k = threadIdx.x; k < A.n; k += blockDim.x) {
        double s = 0.0;
        for (int64_t e = 0; e < A.count[k]; ++e) s += A.ptr[k][e];
        out[A.node[k]] = s;
    }
}

int launch_seg_sums(const double* const* ptr, const int64_t* count, const int32_t* node, int n, double* out,
                    cudaStream_t s) {
    for (int b0 = 0; b0 < n; b0 += kMaxDesc) {
        SegArgs A;
        A.n = n - b0 < kMaxDesc ? n - b0 : kMaxDesc;
        for (int k = 0; k < A.n; ++k) { A.ptr[k] = ptr[b0 + k]; A.count[k] = count[b0 + k]; A.node[k] = node[b0 + k]; }
        k_seg_sums<<<1, 64, 0, s>>>(A, out);
        BIC_LAUNCHED();
    }
    return BICADMM_OK;
}

struct NodeSqArgs {
    int64_t begin[kMaxDesc * 4], count[kMaxDesc * 4];
    int32_t node[kMaxDesc * 4];
    int nb;
};

__device__ __forceinline__ void residuals_body(int N, double sqrtN_rho_c, const double* node_sq, OuterScalars* sc) {
    double pr = 0.0;
    for (int i = 0; i < N; ++i) pr += sqrt(node_sq[i]);
    sc->p_r = pr;
    sc->d_r = sqrtN_rho_c * sqrt(sc->dz2);
    sc->b_r = fabs(sc->g);
}

// res != nullptr (single rank: no AllReduce of node_sq in between): the residuals (15) are
// computed here too, by thread 0 after the block barrier (one launch instead of two)
__global__ void k_node_sq(const __grid_constant__ NodeSqArgs A, const double* __restrict__ partial, int N,
                          double* __restrict__ node_sq, OuterScalars* res, double sqrtN_rho_c) {
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        double acc = 0.0;
        for (int b = 0; b < A.nb; ++b)
            if (A.node[b] == i)
                for (int64_t k = 0; k < A.count[b]; ++k) acc += partial[A.begin[b] + k];
        node_sq[i] = acc;
    }
    if (res) {
        __syncthreads();
        if (threadIdx.x == 0) residuals_body(N, sqrtN_rho_c, node_sq, res);
    }
}

int launch_node_sq(const BlockVec* bv, int nb, const double* partial, int N, double* node_sq, cudaStream_t s,
                   OuterScalars* res, double sqrtN_rho_c) {
    if (nb > kMaxDesc * 4) return BICADMM_ERR_PLACEMENT;
    NodeSqArgs A;
    A.nb = nb;
    for (int b = 0; b < nb; ++b) {
        A.begin[b] = bv[b].cta_begin;
        A.count[b] = (bv[b].len + kUThreads * kUPer - 1) / (kUThreads * kUPer);
        A.node[b] = bv[b].node;
    }
    k_node_sq<<<1, 64, 0, s>>>(A, partial, N, node_sq, res, sqrtN_rho_c);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

__global__ void k_residuals(int N, double sqrtN_rho_c, const double* __restrict__ node_sq, OuterScalars* sc) {
    if (threadIdx.x == 0) residuals_body(N, sqrtN_rho_c, node_sq, sc);
}

int launch_residuals(int N, double sqrtN_rho_c, const double* node_sq, OuterScalars* sc, cudaStream_t s) {
    k_residuals<<<1, 32, 0, s>>>(N, sqrtN_rho_c, node_sq, sc);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

}  // namespace bic
