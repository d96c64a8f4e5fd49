// k_gram_tc.cu -- FP64-accurate Gram G = A^T A on the 5th-generation tensor cores
// (Ozaki-scheme emulation on tcgen05 kind::i8).
//
// sm_100a has no FP64 tcgen05 kind; the FP64 DMMA path (k_factor.cu) runs near its
// ~40 TFLOP/s peak.  Here every column l of A is scaled by 2^-e_l (|A[:,l]| 128 < 127 2^e_l)
// and split into S balanced digits by round-to-nearest,
//     A[r,l] 2^-e_l = sum_{s=1..S} d_s[r,l] 2^-7s + eps,  d_1 in [-127, 127], d_s in [-64, 64],
//     |eps| <= 2^-(7S+1)
// (S = 7: 50 bits below the column maximum, for FP64 and FP32 data alike), so that
//     G[i,j] = 2^(e_i+e_j) sum_{s+t <= S+1} 2^-7(s+t) (D_s^T D_t)[i,j]     (+ dropped terms)
// Round-to-nearest digits carry no sign bias (truncated digits all share the sign of the
// entry, so the dropped products of a diagonal entry G_ii would add up coherently: that
// costs ~1e-13 at S = 7); the dropped terms (s + t >= S + 2) and eps are zero-mean.
// Each D_s^T D_t is an exact int8 x int8 -> int32 product on tcgen05.mma kind::i8; the
// products of equal weight w = s + t accumulate in one TMEM accumulator (7 accumulators of
// 128 x 64 int32 = TMEM columns 0..447), flushed to FP64 registers every 16,384 rows
// (int32 headroom: 7 products x 127^2 x 16,384 < 2^31).  The weighted sum over w is formed
// in FP64 in a fixed order (deterministic), scaled, and written as alpha G + diag I (lower
// triangle).  Measured error <= ~2e-14 of sqrt(G_ii G_jj) (tests/test_gpu_ops.py).
// (A-in-TMEM operands were measured and rejected: tools/tc_i8_rate.cu -- at N = 64 a
// tcgen05.mma takes ~45 cycles with A in TMEM vs 48 from shared memory, and the
// tcgen05.cp + slot-reuse waits cost more than that saves.)
//
// Pipeline per CTA (one 128 x 64 tile of G, lower triangle of tiles):
//   warp 5    : one thread issues the bulk copies (cp.async.bulk, one contiguous 4 KB / 2 KB
//               block per digit tile: the digits are stored pre-swizzled, SWIZZLE_32B) of
//               the S slices of 32 rows x (128 + 64) columns into a 5-stage ring
//   warp 4    : one thread issues S(S+1)/2 tcgen05.mma (M 128, N 64, K 32) per stage,
//               commits to the stage's "empty" barrier and, per 16,384-row round, to
//               "acc_full"
//   warps 0-3 : the TMEM epilogue (tcgen05.ld of the 7 accumulators per round)
// The slices are produced once per block by k_oz_split (column-major int8, zero padded).
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace bic {

constexpr int kOzBM = 128, kOzBK = 32;               // tile M (columns i), K (rows per stage)
constexpr int kOzSMax = 7;                            // digits S; weights 2 .. S + 1
constexpr int kOzRoundStages = 16384 / kOzBK;         // stages per int32 accumulation round
constexpr int kOzRowChunk = 32768;                    // rows of A split per launch pair

__device__ __forceinline__ uint32_t oz_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// column exponent: 128 |A[:,l]| 2^-e < 127, so the first round-to-nearest digit fits int8
__device__ __forceinline__ int oz_exp(double mx) { return mx > 0.0 ? ilogb(mx * (128.0 / 127.0)) + 1 : 0; }

// ----------------------------------------------------------------------------- exponents
// Operand element (l, r) = src[l * sl + r * sr]: l indexes the MMA operand rows (columns of
// A for a Gram, rows of the left factor, columns of the right factor), r the summed index.
// mx[l] = max_r |(l, r)| as order-preserving int64 bits (atomicMax: exact, deterministic)
template <typename T>
__global__ void k_oz_absmax(const T* __restrict__ src, int64_t sl, int64_t sr, int64_t L, int64_t R,
                            int64_t r_per, unsigned long long* __restrict__ mx) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= L) return;
    const int64_t r0 = (int64_t)blockIdx.y * r_per, r1 = r0 + r_per < R ? r0 + r_per : R;
    double m = 0.0;
    for (int64_t r = r0; r < r1; ++r) m = fmax(m, fabs((double)src[l * sl + r * sr]));
    atomicMax(mx + l, (unsigned long long)__double_as_longlong(m));
}

// Operand rows contiguous (sr == 1): one warp per row, coalesced, shuffle max
template <typename T>
__global__ void k_oz_absmax_rows(const T* __restrict__ src, int64_t sl, int64_t L, int64_t R,
                                 unsigned long long* __restrict__ mx) {
    const int64_t l = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (l >= L) return;
    const int lane = threadIdx.x & 31;
    double m = 0.0;
    for (int64_t r = lane; r < R; r += 32) m = fmax(m, fabs((double)src[l * sl + r]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) mx[l] = (unsigned long long)__double_as_longlong(m);
}

// ----------------------------------------------------------------------------- split
// Thread = (operand row l, 32 summed indices): digits written K-chunk major,
// out[s][r / 32][l][r % 32] (32 bytes per digit per thread; adjacent rows l adjacent, so the
// stores coalesce and a tile of rows is one contiguous block); the two 16-byte halves of a
// row piece are stored in the SWIZZLE_32B order of the UMMA descriptor (chunk ^= bit 2 of
// the row), so a plain bulk copy lands in the layout the MMA reads.  r >= rows, l >= L: 0.
template <typename T>
__global__ void k_oz_split(const T* __restrict__ src, int64_t sl, int64_t sr, int64_t L, int64_t r_begin,
                           int64_t rows, const unsigned long long* __restrict__ mx, int8_t* __restrict__ out,
                           int64_t Lp, int64_t Kp) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t rg = (int64_t)blockIdx.y * 32;   // summed-index group within this chunk
    if (l >= Lp || rg >= Kp) return;
    const int e = l < L ? oz_exp(__longlong_as_double((long long)mx[l])) : 0;
    uint32_t pk[kOzSMax][8];
#pragma unroll
    for (int s = 0; s < kOzSMax; ++s)
#pragma unroll
        for (int q = 0; q < 8; ++q) pk[s][q] = 0u;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        const int64_t r = rg + k;
        double a = 0.0;
        if (l < L && r < rows) a = scalbn((double)src[l * sl + (r_begin + r) * sr], -e);
#pragma unroll
        for (int s = 0; s < kOzSMax; ++s) {
            const double t = a * 128.0;               // exact
            const double d = rint(t);                 // |d| <= 127 (s = 1), <= 64 (s > 1)
            a = t - d;                                // exact, |a| <= 1/2
            const uint32_t byte = (uint32_t)(uint8_t)(int8_t)(int)d;
            pk[s][k >> 2] |= byte << (8 * (k & 3));
        }
    }
#pragma unroll
    for (int s = 0; s < kOzSMax; ++s) {
        uint4* dst = reinterpret_cast<uint4*>(out + (((int64_t)s * (Kp / 32) + rg / 32) * Lp + l) * 32);
        const int sw = (int)((l >> 2) & 1);   // SWIZZLE_32B: 16-byte chunk ^= bit 2 of the row
        dst[sw] = make_uint4(pk[s][0], pk[s][1], pk[s][2], pk[s][3]);
        dst[sw ^ 1] = make_uint4(pk[s][4], pk[s][5], pk[s][6], pk[s][7]);
    }
}

// sr == 1 (operand rows contiguous): the CTA's 128 rows x 32 summed indices are staged
// through shared memory by coalesced row reads (row stride 33 doubles: conflict-free), then
// digitised as above.
template <typename T>
__global__ void __launch_bounds__(128) k_oz_split_rows(const T* __restrict__ src, int64_t sl, int64_t L, int64_t r_begin,
                                                       int64_t rows, const unsigned long long* __restrict__ mx,
                                                       int8_t* __restrict__ out, int64_t Lp, int64_t Kp) {
    __shared__ double tile[128][33];
    const int64_t l0 = (int64_t)blockIdx.x * 128;
    const int64_t rg = (int64_t)blockIdx.y * 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int q = warp; q < 128; q += 4) {
        const int64_t l = l0 + q, r = rg + lane;
        tile[q][lane] = (l < L && r < rows) ? (double)src[l * sl + r_begin + r] : 0.0;
    }
    __syncthreads();
    const int64_t l = l0 + threadIdx.x;
    if (l >= Lp || rg >= Kp) return;
    const int e = l < L ? oz_exp(__longlong_as_double((long long)mx[l])) : 0;
    uint32_t pk[kOzSMax][8];
#pragma unroll
    for (int s = 0; s < kOzSMax; ++s)
#pragma unroll
        for (int q = 0; q < 8; ++q) pk[s][q] = 0u;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        double a = scalbn(tile[threadIdx.x][k], -e);
#pragma unroll
        for (int s = 0; s < kOzSMax; ++s) {
            const double t = a * 128.0;
            const double d = rint(t);
            a = t - d;
            const uint32_t byte = (uint32_t)(uint8_t)(int8_t)(int)d;
            pk[s][k >> 2] |= byte << (8 * (k & 3));
        }
    }
#pragma unroll
    for (int s = 0; s < kOzSMax; ++s) {
        uint4* dst = reinterpret_cast<uint4*>(out + (((int64_t)s * (Kp / 32) + rg / 32) * Lp + l) * 32);
        const int sw = (int)((l >> 2) & 1);   // SWIZZLE_32B: 16-byte chunk ^= bit 2 of the row
        dst[sw] = make_uint4(pk[s][0], pk[s][1], pk[s][2], pk[s][3]);
        dst[sw ^ 1] = make_uint4(pk[s][4], pk[s][5], pk[s][6], pk[s][7]);
    }
}

// ----------------------------------------------------------------------------- GEMM
// Operands by bulk copy (pre-swizzled SWIZZLE_32B: one K = 32-byte row per column,
// 8-column atoms of 256 B), 4-stage ring, tcgen05.mma (M 128, N 128, K 32) per slice pair.
__device__ __forceinline__ uint64_t oz_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                    // LBO (unused for swizzled K-major layouts)
    d |= (uint64_t)(256 >> 4) << 32;           // SBO: 8 columns x 32 B
    d |= (uint64_t)1 << 46;                    // descriptor version 1 (sm_100)
    d |= (uint64_t)6 << 61;                    // SWIZZLE_32B
    return d;
}
__device__ __forceinline__ void oz_mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t ok = 0;
    for (long long it = 0; !ok; ++it) {
        asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                     : "=r"(ok) : "r"(oz_smem(b)), "r"(parity) : "memory");
        if (it > (1ll << 28)) asm volatile("trap;");
    }
}
// long waits (the epilogue waits a whole accumulation round): back off with nanosleep so
// the spinning warps do not take issue slots from the MMA and TMA threads
__device__ __forceinline__ void oz_mbar_wait_sleep(uint64_t* b, uint32_t parity) {
    uint32_t ok = 0;
    for (long long it = 0; !ok; ++it) {
        asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                     : "=r"(ok) : "r"(oz_smem(b)), "r"(parity) : "memory");
        if (!ok) __nanosleep(2000);
        if (it > (1ll << 26)) asm volatile("trap;");
    }
}
// plain bulk copy global -> shared (one contiguous block), completing on an mbarrier
__device__ __forceinline__ void oz_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(oz_smem(dst)), "l"(src), "r"(bytes), "r"(oz_smem(bar)) : "memory");
}
__device__ __forceinline__ void oz_mbar_arrive(uint64_t* b) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(oz_smem(b)) : "memory");
}
struct OzArgs {
    int64_t M, N;            // true sizes of C (rows i: A-operand rows; columns j: B-operand rows)
    int64_t Mp, Np, Kp;      // padded A / B operand rows, padded summed index of this chunk
    int64_t ntj;             // column tiles (rectangular tile set)
    int lower;               // tiles meeting the lower triangle only (M == N); entries j <= i
    int mirror;              // also write C[j][i] for the written i > j
    int k_lo, k_hi;          // zero structure of the operands (launch_gemm_tc), absolute indices
    int64_t K, r_begin;      // total summed length; this chunk starts at r_begin
    const unsigned long long *amax, *bmax;   // per-row maxima of the A / B operands
    const int8_t *da, *db;   // digits, [S][Kp / 32][Lp][32 bytes], 32-byte rows pre-swizzled
    double alpha, beta, diag;
    double* C;
    int64_t ldc;
};

// ----------------------------------------------------------------------------- N = 128, two passes
// (An earlier N = 64 single-pass variant was slower: at N = 64 a tcgen05.mma kind::i8 costs
// ~48 cycles instead of 32, tools/tc_i8_rate.cu; N = 128 runs at the full rate.)  Seven 128 x 128 int32
// accumulators do not fit the 512 TMEM columns, so each tile streams its summed range
// twice: pass 0 the weights 2..5 (digits 1..4, 10 products, 4 accumulators = 512
// columns), pass 1 the weights 6..8 (all digits, 18 products, 3 accumulators).  The FP64
// result is the same sum in another fixed order.  8 epilogue warps (lane quarter w & 3,
// column half w >> 2), 1 MMA warp, 1 TMA warp.
constexpr int kOz2BN = 128;
constexpr int kOz2Stages = 4;
constexpr int kOz2Threads = 320;
constexpr size_t kOz2Slice = (size_t)kOz2BN * kOzBK;                     // 4 KB per digit tile
constexpr size_t kOz2StageBytes = (size_t)kOzSMax * 2 * kOz2Slice;      // 56 KB

__device__ __forceinline__ void oz_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}

__device__ __forceinline__ constexpr int oz2_nslice(int pass) { return pass == 0 ? 4 : kOzSMax; }

__global__ void __launch_bounds__(kOz2Threads, 1)
    k_oz_mm128(const __grid_constant__ OzArgs a) {
    extern __shared__ __align__(1024) uint8_t oz_sm_raw[];
    uint8_t* oz_sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(oz_sm_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[kOz2Stages], empty[kOz2Stages], acc_full, acc_empty;
    __shared__ uint32_t tmem_base;
    int64_t bi, bj;
    if (a.lower) {   // 128 x 128 tiles with bj <= bi
        int64_t t = blockIdx.x;
        bi = 0;
        while (t >= bi + 1) { t -= bi + 1; ++bi; }
        bj = t;
    } else {
        bi = (int64_t)blockIdx.x / a.ntj;
        bj = (int64_t)blockIdx.x % a.ntj;
    }
    const int64_t i0 = bi * kOzBM, j0 = bj * kOz2BN;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    int64_t klo = 0, khi = a.K;
    if (a.k_lo == 1) klo = i0;
    if (a.k_lo == 2) klo = j0;
    if (a.k_lo == 3) klo = i0 > j0 ? i0 : j0;
    if (a.k_hi == 1 && i0 + kOzBM < khi) khi = i0 + kOzBM;
    if (a.k_hi == 2 && j0 + kOz2BN < khi) khi = j0 + kOz2BN;
    klo = (klo > a.r_begin ? klo : a.r_begin) - a.r_begin;
    khi = (khi < a.r_begin + a.Kp ? khi : a.r_begin + a.Kp) - a.r_begin;
    const int st0 = (int)(klo / kOzBK);
    const int st1 = khi > klo ? (int)((khi + kOzBK - 1) / kOzBK) : st0;
    const int nstage = st1 - st0;
    const int nround = (nstage + kOzRoundStages - 1) / kOzRoundStages;   // per pass
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(oz_smem(&tmem_base)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int s = 0; s < kOz2Stages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(oz_smem(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(oz_smem(&empty[s])));
        }
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(oz_smem(&acc_full)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(oz_smem(&acc_empty)), "r"(256));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base;

    if (warp == 9) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            int q = 0;   // stage counter over both passes
            for (int pass = 0; pass < 2; ++pass) {
                const int ns = oz2_nslice(pass);
                for (int st = 0; st < nstage; ++st, ++q) {
                    const int sb = q % kOz2Stages;
                    if (q >= kOz2Stages) oz_mbar_wait(&empty[sb], (uint32_t)((q / kOz2Stages - 1) & 1));
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(oz_smem(&full[sb])),
                                 "r"((uint32_t)(ns * 2 * kOz2Slice)) : "memory");
                    uint8_t* base = oz_sm + (size_t)sb * kOz2StageBytes;
                    const int64_t kc = st0 + st, KC = a.Kp / kOzBK;
                    for (int s = 0; s < ns; ++s) {
                        const int64_t ra = (s * KC + kc) * a.Mp + i0, rbb = (s * KC + kc) * a.Np + j0;
                        oz_bulk(base + (size_t)s * kOz2Slice, a.da + ra * kOzBK, (uint32_t)kOz2Slice, &full[sb]);
                        oz_bulk(base + (size_t)(kOzSMax + s) * kOz2Slice, a.db + rbb * kOzBK, (uint32_t)kOz2Slice, &full[sb]);
                    }
                }
            }
        }
    } else if (warp == 8) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            // idesc: S32 accumulate, s8 x s8, K-major A and B, N = 128, M = 128
            const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kOz2BN >> 3) << 17) |
                                   ((uint32_t)(kOzBM >> 4) << 24);
            const uint32_t smem0 = oz_smem(oz_sm);
            int q = 0, rglob = 0;
            for (int pass = 0; pass < 2; ++pass) {
                const int wlo = pass == 0 ? 2 : 6, whi = pass == 0 ? 5 : kOzSMax + 1;
                int st = 0;
                for (int rd = 0; rd < nround; ++rd, ++rglob) {
                    if (rglob > 0) oz_mbar_wait(&acc_empty, (uint32_t)((rglob - 1) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const int st_end = (rd + 1) * kOzRoundStages < nstage ? (rd + 1) * kOzRoundStages : nstage;
                    const int st_begin = st;
                    for (; st < st_end; ++st, ++q) {
                        const int sb = q % kOz2Stages;
                        oz_mbar_wait(&full[sb], (uint32_t)((q / kOz2Stages) & 1));
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        const uint64_t dS = oz_desc(smem0 + (uint32_t)(sb * kOz2StageBytes));
                        const uint32_t first = st == st_begin ? 1u : 0u;
#pragma unroll
                        for (int sa = 1; sa <= kOzSMax; ++sa)
#pragma unroll
                            for (int sbk = 1; sbk <= kOzSMax; ++sbk) {
                                const int w = sa + sbk;
                                if (w < wlo || w > whi) continue;
                                const uint32_t dt = tmem + (uint32_t)((w - wlo) * kOz2BN);
                                const uint64_t da = dS + (uint64_t)(((sa - 1) * kOz2Slice) >> 4);
                                const uint64_t db = dS + (uint64_t)(((kOzSMax + sbk - 1) * kOz2Slice) >> 4);
                                // the first product of each weight in a round overwrites its accumulator
                                const uint32_t accum = (sa == 1) ? (first ^ 1u) : 1u;
                                asm volatile(
                                    "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }" ::"r"(dt),
                                    "l"(da), "l"(db), "r"(idesc), "r"(accum));
                            }
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                            oz_smem(&empty[sb])));
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                        oz_smem(&acc_full)));
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue (warps 0-7)
        const int quarter = warp & 3, half = warp >> 2;
        double acc[64];
#pragma unroll
        for (int c = 0; c < 64; ++c) acc[c] = 0.0;
        int rglob = 0;
        for (int pass = 0; pass < 2; ++pass) {
            const int wlo = pass == 0 ? 2 : 6, whi = pass == 0 ? 5 : kOzSMax + 1;
            for (int rd = 0; rd < nround; ++rd, ++rglob) {
                oz_mbar_wait_sleep(&acc_full, (uint32_t)(rglob & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t lane_addr = tmem + ((uint32_t)(32 * quarter) << 16) + (uint32_t)(64 * half);
                for (int w = wlo; w <= whi; ++w) {   // fixed order
                    const double sc = ldexp(1.0, -7 * w);
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        uint32_t v[32];
                        oz_ld32(lane_addr + (uint32_t)((w - wlo) * kOz2BN + 32 * hh), v);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                        for (int c = 0; c < 32; ++c) acc[32 * hh + c] = fma((double)(int32_t)v[c], sc, acc[32 * hh + c]);
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                oz_mbar_arrive(&acc_empty);
            }
        }
        const int64_t i = i0 + 32 * quarter + lane;
        if (i < a.M) {
            const int ei = oz_exp(__longlong_as_double((long long)a.amax[i]));
            double* crow = a.C + i * a.ldc;
#pragma unroll
            for (int c = 0; c < 64; ++c) {
                const int64_t j = j0 + 64 * half + c;
                if (j >= a.N || (a.lower && j > i)) continue;
                const int ej = oz_exp(__longlong_as_double((long long)a.bmax[j]));
                double v = a.alpha * ldexp(acc[c], ei + ej);
                if (a.beta != 0.0) v += a.beta * crow[j];
                if (i == j) v += a.diag;
                crow[j] = v;
                if (a.mirror && j < i) a.C[j * a.ldc + i] = v;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ----------------------------------------------------------------------------- host
static int64_t oz_rup(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// scratch: A digits [S][Mp][Kp] (+ B digits [S][Np][Kp] unless B is A) + row maxima
size_t gemm_tc_scratch_bytes(int64_t M, int64_t N, int64_t K, bool same) {
    const int64_t Mp = oz_rup(M, kOzBM), Np = oz_rup(N, kOzBM);
    const int64_t Kp = oz_rup(K < kOzRowChunk ? K : kOzRowChunk, kOzBK);
    size_t b = (size_t)oz_rup((int64_t)kOzSMax * Mp * Kp, 256);
    if (!same) b += (size_t)oz_rup((int64_t)kOzSMax * Np * Kp, 256);
    return b + sizeof(unsigned long long) * (size_t)(Mp + (same ? 0 : Np)) + 1024;
}

size_t gram_tc_scratch_bytes(int dtype, int64_t m, int64_t nj) {
    (void)dtype;
    return gemm_tc_scratch_bytes(nj, nj, m, true);
}

bool gram_tc_enabled() {
    static const bool on = [] { const char* e = getenv("BICADMM_GRAM_TC"); return !(e && atoi(e) == 0); }();
    return on;
}

template <typename T>
static void oz_operand(const void* src, int64_t sl, int64_t sr, int64_t L, int64_t R, unsigned long long* mx,
                       cudaStream_t s) {
    if (sr == 1 && sl != 1) {
        k_oz_absmax_rows<T><<<(unsigned)((L + 7) / 8), 256, 0, s>>>(static_cast<const T*>(src), sl, L, R, mx);
        return;
    }
    const int64_t r_per = L >= 16384 ? 2048 : 256;   // enough CTAs for narrow operands
    dim3 g((unsigned)((L + 255) / 256), (unsigned)((R + r_per - 1) / r_per));
    k_oz_absmax<T><<<g, 256, 0, s>>>(static_cast<const T*>(src), sl, sr, L, R, r_per, mx);
}
template <typename T>
static void oz_digits(const void* src, int64_t sl, int64_t sr, int64_t L, int64_t r_begin, int64_t rows,
                      const unsigned long long* mx, int8_t* out, int64_t Lp, int64_t Kp, cudaStream_t s) {
    dim3 g((unsigned)((Lp + 127) / 128), (unsigned)(Kp / 32));
    if (sr == 1 && sl != 1)
        k_oz_split_rows<T><<<g, 128, 0, s>>>(static_cast<const T*>(src), sl, L, r_begin, rows, mx, out, Lp, Kp);
    else
        k_oz_split<T><<<g, 128, 0, s>>>(static_cast<const T*>(src), sl, sr, L, r_begin, rows, mx, out, Lp, Kp);
}

int launch_gemm_tc(const OzGemm& g, void* scratch, size_t scratch_bytes, cudaStream_t s) {
    if (g.M <= 0 || g.N <= 0) return BICADMM_OK;
    if (g.lower && g.M != g.N) return BICADMM_ERR_INVALID;
    if (scratch_bytes < gemm_tc_scratch_bytes(g.M, g.N, g.K, g.same)) return BICADMM_ERR_INVALID;
    const int64_t Mp = oz_rup(g.M, kOzBM), Np = g.same ? Mp : oz_rup(g.N, kOzBM);
    const int64_t Kmax = g.K < kOzRowChunk ? g.K : kOzRowChunk;
    const int64_t Kp_max = oz_rup(Kmax > 0 ? Kmax : 1, kOzBK);
    char* base = static_cast<char*>(scratch);
    int8_t* da = reinterpret_cast<int8_t*>(base);
    size_t off = (size_t)oz_rup((int64_t)kOzSMax * Mp * Kp_max, 256);
    int8_t* db = da;
    if (!g.same) {
        db = reinterpret_cast<int8_t*>(base + off);
        off += (size_t)oz_rup((int64_t)kOzSMax * Np * Kp_max, 256);
    }
    unsigned long long* amax = reinterpret_cast<unsigned long long*>(base + off);
    unsigned long long* bmax = g.same ? amax : amax + Mp;
    static bool attr = false;
    const size_t smem = kOz2Stages * kOz2StageBytes + 1024;   // + alignment slack
    if (!attr) {
        BIC_CUDA(cudaFuncSetAttribute(k_oz_mm128, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(kOz2Stages * kOz2StageBytes + 1024)));
        attr = true;
    }
    // per-row scales of both operands over the whole summed range
    BIC_CUDA(cudaMemsetAsync(amax, 0, sizeof(unsigned long long) * (size_t)(Mp + (g.same ? 0 : Np)), s));
    if (g.K > 0) {
        if (g.dtype == BICADMM_F64) oz_operand<double>(g.A, g.a_sl, g.a_sr, g.M, g.K, amax, s);
        else oz_operand<float>(g.A, g.a_sl, g.a_sr, g.M, g.K, amax, s);
        BIC_LAUNCHED();
        if (!g.same) {
            if (g.dtype == BICADMM_F64) oz_operand<double>(g.B, g.b_sl, g.b_sr, g.N, g.K, bmax, s);
            else oz_operand<float>(g.B, g.b_sl, g.b_sr, g.N, g.K, bmax, s);
            BIC_LAUNCHED();
        }
    }
    const int64_t ntb = Mp / kOzBM;
    const int64_t ntj = oz_rup(g.N, kOz2BN) / kOz2BN;
    // lower: sum over bi of (bi + 1) 128-wide column tiles
    const int64_t tiles = g.lower ? ntb * (ntb + 1) / 2 : ntb * ntj;
    for (int64_t r_begin = 0; r_begin < (g.K > 0 ? g.K : 1); r_begin += kOzRowChunk) {
        const int64_t rows = g.K - r_begin < kOzRowChunk ? g.K - r_begin : kOzRowChunk;
        const int64_t Kp = oz_rup(rows > 0 ? rows : 1, kOzBK);
        if (rows > 0) {
            if (g.dtype == BICADMM_F64) oz_digits<double>(g.A, g.a_sl, g.a_sr, g.M, r_begin, rows, amax, da, Mp, Kp, s);
            else oz_digits<float>(g.A, g.a_sl, g.a_sr, g.M, r_begin, rows, amax, da, Mp, Kp, s);
            BIC_LAUNCHED();
            if (!g.same) {
                if (g.dtype == BICADMM_F64) oz_digits<double>(g.B, g.b_sl, g.b_sr, g.N, r_begin, rows, bmax, db, Np, Kp, s);
                else oz_digits<float>(g.B, g.b_sl, g.b_sr, g.N, r_begin, rows, bmax, db, Np, Kp, s);
                BIC_LAUNCHED();
            }
        }
        OzArgs oa{};
        oa.M = g.M; oa.N = g.N; oa.Mp = Mp; oa.Np = Np; oa.Kp = rows > 0 ? Kp : 0; oa.ntj = ntj;
        oa.lower = g.lower; oa.mirror = g.mirror; oa.k_lo = g.k_lo; oa.k_hi = g.k_hi;
        oa.K = g.K; oa.r_begin = r_begin; oa.amax = amax; oa.bmax = bmax; oa.da = da; oa.db = db;
        oa.alpha = g.alpha; oa.beta = r_begin > 0 ? 1.0 : g.beta; oa.diag = r_begin > 0 ? 0.0 : g.diag;
        oa.C = g.C; oa.ldc = g.ldc;
        k_oz_mm128<<<(unsigned)tiles, kOz2Threads, smem, s>>>(oa);
        BIC_LAUNCHED();
    }
    return BICADMM_OK;
}

int launch_gram_tc(int dtype, int64_t m, int64_t nj, const void* A, int64_t lda, double alpha, double diag, double* G,
                   int64_t ldg, void* scratch, size_t scratch_bytes, cudaStream_t s) {
    if (m <= 0 || nj <= 0) return BICADMM_OK;
    OzGemm g{};
    g.M = nj; g.N = nj; g.K = m;
    g.A = A; g.a_sl = 1; g.a_sr = lda;     // operand row l = column l of A, summed over rows
    g.B = A; g.b_sl = 1; g.b_sr = lda;
    g.same = true; g.dtype = dtype;
    g.alpha = alpha; g.beta = 0.0; g.diag = diag; g.C = G; g.ldc = ldg;
    g.lower = 1;
    return launch_gemm_tc(g, scratch, scratch_bytes, s);
}

}  // namespace bic
