// Probe: tcgen05.cp.128x256b (smem -> TMEM) of a K-major int8 A tile, then
// tcgen05.mma kind::i8 with A from TMEM and B from smem (M=128, N=64, K=32), both smem
// tiles in the SWIZZLE_32B K-major layout (32-byte rows, 16-byte chunk index ^= row bit 2).
// Also: two K chunks accumulated, the second A copied into a different TMEM slot after
// the first MMA was committed (the slot-rotation pattern tried for the Ozaki kernel).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/tc_i8_ts_test.cu -o tools/tc_i8_ts_test
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 64, K = 64;   // two K=32 chunks

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int sw32(int row, int kb) {   // byte offset of (row, kb) in a 32-byte-row SWIZZLE_32B tile
    const int o = row * 32 + kb;
    return o ^ (((o >> 7) & 1) << 4);
}
__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(256 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)6 << 61;
    return d;
}
__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t par) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                     : "=r"(ok) : "r"(smem_u32(b)), "r"(par) : "memory");
}

__global__ void k_tc(const int8_t* __restrict__ A, const int8_t* __restrict__ B, int32_t* __restrict__ D, int mode) {
    // A[M][K], B[N][K] row-major (K fastest); smem: per K chunk c, A tile 128 x 32 B, B tile 64 x 32 B
    __shared__ __align__(1024) int8_t sa[2][M * 32];
    __shared__ __align__(1024) int8_t sb[2][N * 32];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int c = 0; c < 2; ++c) {
        for (int e = tid; e < M * 32; e += blockDim.x) { const int r = e / 32, kb = e % 32; sa[c][sw32(r, kb)] = A[r * K + c * 32 + kb]; }
        for (int e = tid; e < N * 32; e += blockDim.x) { const int r = e / 32, kb = e % 32; sb[c][sw32(r, kb)] = B[r * K + c * 32 + kb]; }
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base;
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    if (tid == 0) {
        for (int c = 0; c < 2; ++c) {
            const uint32_t aslot = tmem + 448 + 8 * (mode == 0 ? c : 0);   // mode 1: same slot, reused after a wait
            if (mode == 1 && c == 1) {
                wait_bar(&bar[0], 0);   // MMA of chunk 0 done -> the slot may be overwritten
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            }
            asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(aslot), "l"(desc_sw32(smem_u32(sa[c]))));
            const uint64_t db = desc_sw32(smem_u32(sb[c]));
            const uint32_t acc = c > 0;
            asm volatile(
                "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p; }" ::"r"(tmem),
                "r"(aslot), "l"(db), "r"(idesc), "r"(acc));
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[c])));
        }
    }
    if (tid < 128) {
        wait_bar(&bar[1], 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        uint32_t v[8];
        const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16);
        for (int c0 = 0; c0 < N; c0 += 8) {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                         : "r"(taddr + c0));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int q = 0; q < 8; ++q) D[(32 * warp + lane) * N + c0 + q] = (int32_t)v[q];
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
    std::vector<int8_t> A(M * K), B(N * K);
    srand(7);
    for (auto& a : A) a = (int8_t)(rand() % 255 - 127);
    for (auto& b : B) b = (int8_t)(rand() % 255 - 127);
    int8_t *dA, *dB;
    int32_t* dD;
    cudaMalloc(&dA, A.size()); cudaMalloc(&dB, B.size()); cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(dD, 0, M * N * 4);
        k_tc<<<1, 128>>>(dA, dB, dD, mode);
        cudaError_t e = cudaDeviceSynchronize();
        printf("mode %d kernel: %s\n", mode, cudaGetErrorString(e));
        std::vector<int32_t> D(M * N);
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        long long maxerr = 0;
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
                long long ref = 0;
                for (int k = 0; k < K; ++k) ref += (int)A[i * K + k] * (int)B[j * K + k];
                const long long err = llabs(ref - D[i * N + j]);
                if (err) ++bad;
                if (err > maxerr) maxerr = err;
            }
        printf("mode %d: mismatches %d of %d, max abs err %lld; D[0][0] = %d\n", mode, bad, M * N, maxerr, D[0]);
    }
    return 0;
}
