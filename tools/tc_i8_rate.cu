// Rates of tcgen05 kind::i8 building blocks on one SM (cycles per stage of 28 MMAs
// M=128 N=64 K=32, the S = 7 Ozaki stage), operands already in smem / TMEM:
//   mode 0: A and B from smem (SS)
//   mode 1: A from TMEM (fixed slot), B from smem (TS), no copies
//   mode 2: TS with one tcgen05.cp 128x256b per slice group (7 per stage), single slot per
//           group rotating over 8 slots, no waits
//   mode 3: as 2 with the commit/wait slot protocol of an A-in-TMEM Ozaki kernel (measured, not adopted)
//   mode 4: 7 tcgen05.cp per stage only
//   mode 5: all 7 cps of a stage first (slots 0..6 / 7..13 alternating; N=56 layout), then 28 MMAs
//   mode 6: SS with N = 128 (4 accumulators), mode 7: SS with N = 256 (2 accumulators)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/tc_i8_rate.cu -o tools/tc_i8_rate
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
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
__device__ __forceinline__ void commit(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b)));
}

template <int MODE>
__global__ void k_rate(int iters, long long* out) {
    extern __shared__ __align__(1024) int8_t sm[];
    __shared__ __align__(8) uint64_t bar[9];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int e = tid; e < 7 * 128 * 32 + 3 * 256 * 32; e += blockDim.x) sm[e] = (int8_t)(e * 7);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0)
        for (int s = 0; s < 9; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base;
    constexpr int NN = MODE == 5 ? 56 : MODE == 6 ? 128 : MODE == 7 ? 256 : 64;
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t s0 = smem_u32(sm);
    const uint64_t dA0 = desc_sw32(s0), dB0 = desc_sw32(s0 + 7 * 128 * 32);
    if (tid == 0) {
        const long long t0 = clock64();
        uint32_t grp = 0;
        for (int it = 0; it < iters; ++it) {
            if (MODE >= 6) {
#pragma unroll
                for (int q = 0; q < 28; ++q) {
                    const uint32_t dt = tmem + (uint32_t)((q % (512 / NN)) * NN);
                    const uint64_t da = dA0 + (uint64_t)(((q % 7) * 4096) >> 4);
                    const uint64_t db = desc_sw32(s0 + 7 * 128 * 32 - 7 * 128 * 32 + 4096 * 7 + 0) + (uint64_t)((((q % 3) * NN * 32)) >> 4);
                    asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(dt), "l"(da), "l"(db),
                                 "r"(idesc));
                }
                continue;
            }
            if (MODE == 5) {
                const uint32_t base = tmem + 7 * NN + 56 * (it & 1);
#pragma unroll
                for (int sa = 1; sa <= 7; ++sa)
                    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(base + 8 * (sa - 1)),
                                 "l"(dA0 + (uint64_t)(((sa - 1) * 4096) >> 4)));
#pragma unroll
                for (int sa = 1; sa <= 7; ++sa)
#pragma unroll
                    for (int sb = 1; sb <= 7; ++sb) {
                        if (sa + sb > 8) continue;
                        const uint32_t dt = tmem + (uint32_t)((sa + sb - 2) * NN);
                        const uint64_t db = dB0 + (uint64_t)(((sb - 1) * 2048) >> 4);
                        asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 1;" ::"r"(dt),
                                     "r"(base + 8 * (sa - 1)), "l"(db), "r"(idesc));
                    }
                continue;
            }
#pragma unroll
            for (int sa = 1; sa <= 7; ++sa) {
                const uint32_t slot = grp & 7;
                const uint32_t ta = tmem + 448 + 8 * slot;
                if (MODE == 3 && grp >= 8) {
                    wait_bar(&bar[slot], ((grp >> 3) - 1) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                }
                if (MODE >= 2)
                    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(ta), "l"(dA0 + (uint64_t)(((sa - 1) * 4096) >> 4)));
                if (MODE != 4) {
#pragma unroll
                    for (int sb = 1; sb <= 7; ++sb) {
                        if (sa + sb > 8) continue;
                        const uint32_t dt = tmem + (uint32_t)((sa + sb - 2) * 64);
                        const uint64_t db = dB0 + (uint64_t)(((sb - 1) * 2048) >> 4);
                        if (MODE == 0) {
                            const uint64_t da = dA0 + (uint64_t)(((sa - 1) * 4096) >> 4);
                            asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(dt), "l"(da), "l"(db),
                                         "r"(idesc));
                        } else {
                            const uint32_t tA = MODE == 1 ? tmem + 448 : ta;
                            asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 1;" ::"r"(dt), "r"(tA), "l"(db),
                                         "r"(idesc));
                        }
                    }
                }
                if (MODE == 3) commit(&bar[slot]);
                ++grp;
            }
        }
        commit(&bar[8]);
        wait_bar(&bar[8], 0);
        const long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int MODE>
void run(long long* d, int iters) {
    const int smem = 7 * 128 * 32 + 3 * 256 * 32 + 1024;
    cudaFuncSetAttribute(k_rate<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_rate<MODE><<<148, 128, smem>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("mode %d: %s, %.1f cycles per stage (28 MMAs), %.1f per MMA\n", MODE, cudaGetErrorString(e),
           (double)mx / iters, (double)mx / iters / 28);
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    const int iters = 2000;
    run<0>(d, iters);
    run<1>(d, iters);
    run<2>(d, iters);
    run<3>(d, iters);
    run<4>(d, iters);
    run<6>(d, iters);
    run<7>(d, iters);
    return 0;
}
