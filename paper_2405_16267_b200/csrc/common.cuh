// common.cuh -- shared device helpers of libbicadmm (B200 / sm_100a).
// Deterministic reductions only: every sum below has a fixed order that does
// not depend on scheduling, so replicated state is bit-identical across runs
// and ranks.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <atomic>

#include "../../include/bicadmm.h"

namespace bic {

constexpr int kWarp = 32;
constexpr int kMaxDesc = 64;   // descriptors per batched launch

// Library-wide launch counter (the bench's gpu_launches evidence).
extern std::atomic<int64_t> g_launches;
inline void count_launch(int64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

#define BIC_CUDA(expr)                                            \
    do {                                                          \
        cudaError_t _e = (expr);                                  \
        if (_e != cudaSuccess) return BICADMM_ERR_CUDA;           \
    } while (0)

#define BIC_LAUNCHED()                                            \
    do {                                                          \
        ::bic::count_launch();                                    \
        cudaError_t _e = cudaPeekAtLastError();                   \
        if (_e != cudaSuccess) return BICADMM_ERR_CUDA;           \
    } while (0)

// Record a timing event on stream s; inside a stream capture it becomes an event-record
// node of the graph (so phase timings survive graph replay).
inline cudaError_t record_event(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &st);
    return st == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
                                               : cudaEventRecord(e, s);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double2 ld_stream(const double2* p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                 : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ float4 ld_stream(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}

__device__ __forceinline__ double sgn(double a) { return a > 0.0 ? 1.0 : (a < 0.0 ? -1.0 : 0.0); }

// Block-wide sum in a fixed tree order (warp shuffle tree, then warp 0 over
// the per-warp results in warp order).  All threads get the result.
// scratch: >= 32 doubles of shared memory.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double t = lane < nw ? scratch[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) scratch[0] = t;
    }
    __syncthreads();
    double r = scratch[0];
    __syncthreads();
    return r;
}

__device__ __forceinline__ double block_max(double v, double* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double t = lane < nw ? scratch[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
        if (lane == 0) scratch[0] = t;
    }
    __syncthreads();
    double r = scratch[0];
    __syncthreads();
    return r;
}

// Exclusive scan of one int64 per thread over the block (thread order).
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* scratch, int64_t* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) scratch[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int64_t w = lane < nw ? scratch[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        scratch[lane] = w;  // inclusive per-warp prefix
    }
    __syncthreads();
    int64_t base = wid > 0 ? scratch[wid - 1] : 0;
    if (total) *total = scratch[nw - 1];
    __syncthreads();
    return base + x - v;
}

}  // namespace bic
