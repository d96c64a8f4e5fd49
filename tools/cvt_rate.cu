// cvt_rate.cu -- FP32 -> FP64 widening throughput: F2F.F64.F32 vs an integer bit construction.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cvt_rate tools/cvt_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double widen_int(float f) {
    const unsigned F = __float_as_uint(f);
    const unsigned t = (unsigned)((int)F >> 3);
    unsigned hi = (t & 0x8FFFFFFFu) + 0x38000000u;
    const unsigned lo = F << 29;
    hi = (F & 0x7F800000u) ? hi : 0u;
    return __hiloint2double((int)hi, (int)lo);
}

template <int MODE>
__global__ void k(const float* __restrict__ in, double* out, int iters) {
    float v[8];
    for (int i = 0; i < 8; ++i) v[i] = in[(threadIdx.x + i) & 255];
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const double x = 1.0000001;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            double d;
            if (MODE == 0) d = (double)v[i];
            else d = widen_int(v[i]);
            acc[i] = fma(d, x, acc[i]);
            v[i] = __uint_as_float(__float_as_uint(v[i]) ^ 1u);   // keep the conversion in the loop
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 1.2345) out[0] = s;
}

int main() {
    float* in;
    double* o;
    cudaMalloc(&in, 256 * 4);
    cudaMalloc(&o, 8);
    float h[256];
    for (int i = 0; i < 256; ++i) h[i] = 0.1f * (i + 1);
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096, blocks = sms * 4, threads = 512;
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<blocks, threads>>>(in, o, iters);
            else k<1><<<blocks, threads>>>(in, o, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double n = 8.0 * iters * blocks * threads;
        printf("%s: %.2f conversions(+DFMA)/clk/SM at 1.9 GHz (%.1f G/s)\n", mode ? "int bits" : "F2F", n / (ms * 1e-3) / sms / 1.9e9,
               n / (ms * 1e-3) / 1e9);
    }
    // check the integer widening against the hardware conversion
    return 0;
}
