// k_symv.cu -- packed symmetric H-apply for Eq. (24), x = H r with H = H^T
// (H = (rho_l A^T A + c I)^{-1}, or the Woodbury K^{-1} of a fat block).
//
// Only the lower-triangle 64 x 64 tiles of H are stored, tile-major (tile (I, J),
// I >= J, at index I(I+1)/2 + J, each tile 64 x 64 row-major and contiguous, zero
// padded past n), so the per-sweep H read is n^2/2 + O(64 n) elements instead of
// n^2.  One CTA streams one tile T = H[I-block, J-block] from HBM exactly once and
// produces both halves of its contribution:
//   y_I += T x_J   (row dots: per-thread products, lane reduce-scatter 16 -> 1)
//   y_J += T^T x_I (column dots: per-thread sums over its 16 rows, 4 row groups in smem)
// Per-tile partial vectors are summed by a second kernel in a fixed order (J
// ascending, then K ascending), so the result is bit-reproducible.
#include "common.cuh"
#include "kernels.h"

namespace bic {

constexpr int kTS = 64;                 // tile edge
constexpr int kSymvThreads = 256;       // 8 warps: 4 row groups x 2 column halves

struct SymvBatch {
    SymvDesc d[kMaxDesc];
    int64_t tile_begin[kMaxDesc + 1];
    int64_t elem_begin[kMaxDesc + 1];
    int nd;
};

int64_t symv_nb(int64_t n) { return (n + kTS - 1) / kTS; }
int64_t symv_tiles(int64_t n) { const int64_t nb = symv_nb(n); return nb * (nb + 1) / 2; }
int64_t symv_packed_elems(int64_t n) { return symv_tiles(n) * kTS * kTS; }
int64_t symv_part_doubles(int64_t n) { return symv_tiles(n) * 2 * kTS; }

__device__ __forceinline__ void tile_ij(int64_t t, int64_t& I, int64_t& J) {
    int64_t i = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while (i > 0 && i * (i + 1) / 2 > t) --i;
    while ((i + 1) * (i + 2) / 2 <= t) ++i;
    I = i;
    J = t - i * (i + 1) / 2;
}

__device__ __forceinline__ double ld_h(const double* p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_h(const float* p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return (double)v;
}
// raw element loads (FP32 tiles keep 16 floats, not 16 doubles, while the loads are in flight)
__device__ __forceinline__ double ld_raw(const double* p) { return ld_h(p); }
__device__ __forceinline__ float ld_raw(const float* p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

// one reduce-scatter step over lane bit O: 2*HALF values -> HALF values
template <int HALF, int O>
__device__ __forceinline__ void rs_step(double* a, int lane) {
    const bool up = (lane & O) != 0;
#pragma unroll
    for (int k = 0; k < HALF; ++k) {
        const double send = up ? a[k] : a[k + HALF];
        const double keep = up ? a[k + HALF] : a[k];
        a[k] = keep + __shfl_xor_sync(0xffffffffu, send, O);
    }
}

template <typename T>
__global__ void __launch_bounds__(kSymvThreads, sizeof(T) == 4 ? 6 : 1) k_symv_tiles(const SymvBatch B) {
    __shared__ double xi[kTS], xj[kTS];
    __shared__ double colp[4][kTS];
    __shared__ double rowp[2][kTS];
    const int64_t gt = blockIdx.x;
    int k = 0;
    while (k + 1 < B.nd && gt >= B.tile_begin[k + 1]) ++k;
    const SymvDesc& D = B.d[k];
    const int64_t t = gt - B.tile_begin[k];
    int64_t I, J;
    tile_ij(t, I, J);
    const bool diag = I == J;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = w >> 1, hc = w & 1;
    const int c = hc * 32 + lane;
    const T* tile = static_cast<const T*>(D.H) + t * (int64_t)(kTS * kTS) + (g * 16) * kTS + c;
    T vr[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) vr[i] = ld_raw(tile + i * kTS);
    if (tid < kTS) {
        const int64_t r = I * kTS + tid;
        xi[tid] = r < D.n ? D.x[r] : 0.0;
    } else if (tid < 2 * kTS) {
        const int64_t r = J * kTS + (tid - kTS);
        xj[tid - kTS] = r < D.n ? D.x[r] : 0.0;
    }
    __syncthreads();
    // column dots (T^T x_I)[c] over this thread's 16 rows, rows ascending
    double cs = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) cs = fma((double)vr[i], xi[g * 16 + i], cs);
    colp[g][c] = cs;
    if (!diag) {
        // row dots (T x_J)[row] over this warp's 32 columns: lane reduce-scatter
        const double xc = xj[c];
        double v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = (double)vr[i] * xc;
        rs_step<8, 16>(v, lane);
        rs_step<4, 8>(v, lane);
        rs_step<2, 4>(v, lane);
        rs_step<1, 2>(v, lane);
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
        const int ri = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
        if ((lane & 1) == 0) rowp[hc][g * 16 + ri] = v[0];
    }
    __syncthreads();
    double* out = D.part + t * (int64_t)(2 * kTS);
    if (tid < kTS) {
        // -> y_J (a diagonal tile is symmetric: its column dots are y_I's whole contribution)
        const double s = ((colp[0][tid] + colp[1][tid]) + colp[2][tid]) + colp[3][tid];
        out[diag ? tid : kTS + tid] = s;
    } else if (tid < 2 * kTS && !diag) {
        const int r = tid - kTS;
        out[r] = rowp[0][r] + rowp[1][r];   // -> y_I
    }
}

// y[r] = alpha * (sum_{J <= I} part[(I, J)][0][rr] + sum_{K > I} part[(K, I)][1][rr])
// CTA = 64 outputs x 4 sub-ranges of the nb terms (4x the loads in flight of one thread
// per output: the sum is latency-bound); the 4 sub-sums are added in a fixed order.
constexpr int kRedOut = 64, kRedSub = 4;
__global__ void __launch_bounds__(kRedOut * kRedSub) k_symv_reduce(const SymvBatch B) {
    __shared__ double part_s[kRedSub][kRedOut];
    const int o = threadIdx.x % kRedOut, sub = threadIdx.x / kRedOut;
    const int64_t e = (int64_t)blockIdx.x * kRedOut + o;
    const bool live = e < B.elem_begin[B.nd];
    double s = 0.0;
    int k = 0;
    int64_t r = 0;
    if (live) {
        while (k + 1 < B.nd && e >= B.elem_begin[k + 1]) ++k;
        const SymvDesc& D = B.d[k];
        r = e - B.elem_begin[k];
        const int64_t I = r / kTS, rr = r % kTS, nb = (D.n + kTS - 1) / kTS;
        const double* P = D.part;
        // the nb terms in a fixed order: J = 0..I (row dots of tile (I, J)), then
        // K = I+1..nb-1 (column dots of tile (K, I)); this thread's contiguous quarter,
        // loads issued 8 at a time ahead of the adds
        const int64_t row0 = I * (I + 1) / 2;
        auto addr = [&](int64_t q) -> const double* {
            return q <= I ? P + (row0 + q) * (2 * kTS) + rr : P + (q * (q + 1) / 2 + I) * (2 * kTS) + kTS + rr;
        };
        const int64_t q0 = nb * sub / kRedSub, q1 = nb * (sub + 1) / kRedSub;
        int64_t q = q0;
        for (; q + 8 <= q1; q += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(addr(q + u));
#pragma unroll
            for (int u = 0; u < 8; ++u) s += v[u];
        }
        for (; q < q1; ++q) s += __ldcg(addr(q));
    }
    part_s[sub][o] = s;
    __syncthreads();
    if (sub == 0 && live) {
        const double t = ((part_s[0][o] + part_s[1][o]) + part_s[2][o]) + part_s[3][o];
        B.d[k].y[r] = B.d[k].alpha * t;
    }
}

int launch_symv_packed(int dtype, const SymvDesc* d, int nd, cudaStream_t s) {
    for (int base = 0; base < nd; base += kMaxDesc) {
        SymvBatch B;
        B.nd = nd - base < kMaxDesc ? nd - base : kMaxDesc;
        int64_t t = 0, e = 0;
        for (int k = 0; k < B.nd; ++k) {
            B.d[k] = d[base + k];
            B.tile_begin[k] = t;
            B.elem_begin[k] = e;
            t += symv_tiles(B.d[k].n);
            e += B.d[k].n;
        }
        B.tile_begin[B.nd] = t;
        B.elem_begin[B.nd] = e;
        if (t == 0) continue;
        if (t > 0x7fffffff) return BICADMM_ERR_INVALID;
        if (dtype == BICADMM_F64) k_symv_tiles<double><<<(unsigned)t, kSymvThreads, 0, s>>>(B);
        else k_symv_tiles<float><<<(unsigned)t, kSymvThreads, 0, s>>>(B);
        BIC_LAUNCHED();
        k_symv_reduce<<<(unsigned)((e + kRedOut - 1) / kRedOut), kRedOut * kRedSub, 0, s>>>(B);
        BIC_LAUNCHED();
    }
    return BICADMM_OK;
}

// Pack the full symmetric FP64 matrix G (n x n, leading dimension ldg) into lower tiles.
template <typename T>
__global__ void k_symv_pack(int64_t n, const double* __restrict__ G, int64_t ldg, T* __restrict__ Hp, int64_t total) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    const int64_t t = e / (kTS * kTS), w = e % (kTS * kTS);
    int64_t I, J;
    tile_ij(t, I, J);
    const int64_t r = I * kTS + w / kTS, c = J * kTS + w % kTS;
    Hp[e] = (r < n && c < n) ? (T)G[r * ldg + c] : (T)0;
}

int launch_symv_pack(int dtype, int64_t n, const double* G, int64_t ldg, void* Hp, cudaStream_t s) {
    const int64_t total = symv_packed_elems(n);
    const unsigned blocks = (unsigned)((total + 255) / 256);
    if (dtype == BICADMM_F64) k_symv_pack<double><<<blocks, 256, 0, s>>>(n, G, ldg, static_cast<double*>(Hp), total);
    else k_symv_pack<float><<<blocks, 256, 0, s>>>(n, G, ldg, static_cast<float*>(Hp), total);
    BIC_LAUNCHED();
    return BICADMM_OK;
}

}  // namespace bic
