// fp64_rate.cu -- FP64 pipe throughput on this GPU: DMMA (mma.sync m8n8k4 f64) vs DFMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_rate tools/fp64_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dmma(double* out, int iters) {
    double d[8][2];
    double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
    for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
    if (s == 12345.0) out[0] = s;
}

__global__ void k_dfma(double* out, int iters) {
    double d[16];
    double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
    for (int i = 0; i < 16; ++i) d[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) d[i] = fma(d[i], b, a);
    }
    double s = 0;
    for (int i = 0; i < 16; ++i) s += d[i];
    if (s == 12345.0) out[0] = s;
}

// DMMA and DFMA interleaved: do they share a pipe?
__global__ void k_mix(double* out, int iters) {
    double d[4][2], f[16];
    double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
    for (int i = 0; i < 4; ++i) d[i][0] = d[i][1] = 0.0;
    for (int i = 0; i < 16; ++i) f[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
#pragma unroll
        for (int i = 0; i < 16; ++i) f[i] = fma(f[i], b, a);
    }
    double s = 0;
    for (int i = 0; i < 4; ++i) s += d[i][0] + d[i][1];
    for (int i = 0; i < 16; ++i) s += f[i];
    if (s == 12345.0) out[0] = s;
}

int main() {
    double* o;
    cudaMalloc(&o, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int threads : {128, 256, 512, 1024}) {
        const int iters = 4096, blocks = sms * 2;
        k_dmma<<<blocks, threads>>>(o, 16);
        cudaEventRecord(e0);
        k_dmma<<<blocks, threads>>>(o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 256 * 8 * (double)iters * blocks * (threads / 32);
        printf("DMMA threads/CTA %4d: %.1f TFLOP/s\n", threads, fl / ms / 1e9);
        k_dfma<<<blocks, threads>>>(o, 16);
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        fl = 2.0 * 16 * (double)iters * blocks * threads;
        printf("DFMA threads/CTA %4d: %.1f TFLOP/s\n", threads, fl / ms / 1e9);
    }
    {
        const int iters = 4096, blocks = sms * 2, threads = 512;
        k_mix<<<blocks, threads>>>(o, 16);
        cudaEventRecord(e0);
        k_mix<<<blocks, threads>>>(o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fl_mma = 2.0 * 256 * 4 * (double)iters * blocks * (threads / 32);
        const double fl_fma = 2.0 * 16 * (double)iters * blocks * threads;
        printf("mixed: DMMA %.1f + DFMA %.1f = %.1f TFLOP/s (4 DMMA : 16 DFMA per warp iteration)\n",
               fl_mma / ms / 1e9, fl_fma / ms / 1e9, (fl_mma + fl_fma) / ms / 1e9);
    }
    return 0;
}
