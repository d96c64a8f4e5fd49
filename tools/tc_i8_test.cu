// Probe: one tcgen05.mma kind::i8 tile (M=128, N=64, K=64) from K-major, no-swizzle
// ("interleaved") shared-memory operands into TMEM, read back with tcgen05.ld.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/tc_i8_test.cu -o tools/tc_i8_test
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 64, K = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major interleaved layout: core matrix = 8 rows x 16 bytes (128 B contiguous);
// element (row, kb) at (row/8)*SBO + (kb/16)*LBO + (row%8)*16 + kb%16
__device__ __forceinline__ int il_off(int row, int kb, int lbo, int sbo) {
    return (row >> 3) * sbo + (kb >> 4) * lbo + (row & 7) * 16 + (kb & 15);
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;   // version 1 (sm100)
    // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
    return d;
}

__global__ void k_tc(const int8_t* __restrict__ A, const int8_t* __restrict__ B, int32_t* __restrict__ D) {
    __shared__ __align__(1024) int8_t sa[M * K];
    __shared__ __align__(1024) int8_t sb[N * K];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int LBO = 128, SBO_A = (K / 16) * 128, SBO_B = (K / 16) * 128;
    for (int e = tid; e < M * K; e += blockDim.x) { const int r = e / K, kb = e % K; sa[il_off(r, kb, LBO, SBO_A)] = A[e]; }
    for (int e = tid; e < N * K; e += blockDim.x) { const int r = e / K, kb = e % K; sb[il_off(r, kb, LBO, SBO_B)] = B[e]; }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    }
    // make the generic-proxy smem writes visible to the async (tensor) proxy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base;
    if (tid == 0) {
        // instruction descriptor: c_format S32 (2) @ [4,6), a_format s8 (1) @ [7,10), b_format s8 (1) @ [10,13),
        // a/b K-major (0), n_dim = N >> 3 @ [17,23), m_dim = M >> 4 @ [24,29)
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        for (int ks = 0; ks < K / 32; ++ks) {
            const uint64_t da = make_desc(smem_u32(sa) + ks * 2 * LBO, LBO, SBO_A);
            const uint64_t db = make_desc(smem_u32(sb) + ks * 2 * LBO, LBO, SBO_B);
            const uint32_t acc = ks > 0;
            asm volatile(
                "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }" ::"r"(tmem),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
    }
    // wait for the MMAs
    {
        uint32_t ok = 0;
        while (!ok) {
            asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                         : "=r"(ok) : "r"(smem_u32(&mbar)), "r"(0u) : "memory");
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // each warp reads its 32 lanes (rows), 64 columns
    uint32_t v[64];
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,"
        "%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]),
          "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]), "=r"(v[39]),
          "=r"(v[40]), "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]),
          "=r"(v[48]), "=r"(v[49]), "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]),
          "=r"(v[56]), "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int row = 32 * warp + lane;
    for (int c = 0; c < 64; ++c) D[row * N + c] = (int32_t)v[c];
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
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
    cudaMemset(dD, 0, M * N * 4);
    k_tc<<<1, 128>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
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
    printf("mismatches %d of %d, max abs err %lld; D[0][0] = %d\n", bad, M * N, maxerr, D[0]);
    return 0;
}
