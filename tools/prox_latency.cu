// Single-thread latency of the per-sample logistic prox (Eq. (22)) as used on the
// fused sweep's critical path.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/prox_latency.cu
#include <cstdio>
#include <cfloat>
#include <cmath>
__device__ __forceinline__ double sig(double a) {
    if (a >= 0.0) return 1.0 / (1.0 + exp(-a));
    const double e = exp(a);
    return e / (1.0 + e);
}
__device__ double prox(double rho, double b, double p, double w0, int* its) {
    double lo = p - 1.0 / rho, hi = p + 1.0 / rho;
    double w = (w0 > lo && w0 < hi) ? w0 : p;
    int it = 0;
    for (; it < 60; ++it) {
        const double sg = sig(-b * w);
        const double g = -b * sg + rho * (w - p);
        if (g > 0.0) hi = w; else lo = w;
        const double gp = sg * (1.0 - sg) + rho;
        const double step = g / gp;
        if (fabs(step) <= 4.0 * DBL_EPSILON * fmax(1.0, fabs(w))) { w -= step; break; }
        double wn = w - step;
        if (!(wn > lo && wn < hi)) wn = 0.5 * (lo + hi);
        w = wn;
    }
    *its += it + 1;
    return w;
}
__global__ void k(const double* p, const double* w0, double* out, long long* cyc, int* its, int n, int warm) {
    long long t0 = clock64();
    double acc = 0;
    for (int i = 0; i < n; ++i) acc += prox(4.0, (i & 1) ? 1.0 : -1.0, p[i], warm ? w0[i] : 1e300, its);
    long long t1 = clock64();
    out[0] = acc;
    cyc[0] = t1 - t0;
}
__global__ void kexp(const double* p, double* out, long long* cyc, int n) {
    long long t0 = clock64();
    double acc = 0;
    for (int i = 0; i < n; ++i) acc += exp(p[i] + acc * 1e-300);
    long long t1 = clock64();
    out[0] = acc; cyc[0] = t1 - t0;
}
__global__ void kdiv(const double* p, double* out, long long* cyc, int n) {
    long long t0 = clock64();
    double acc = 1;
    for (int i = 0; i < n; ++i) acc = 1.0 / (p[i] + acc);
    long long t1 = clock64();
    out[0] = acc; cyc[0] = t1 - t0;
}
int main() {
    const int n = 1000;
    double *p, *w0, *out; long long* cyc; int* its;
    cudaMallocManaged(&p, n * 8); cudaMallocManaged(&w0, n * 8); cudaMallocManaged(&out, 8);
    cudaMallocManaged(&cyc, 8); cudaMallocManaged(&its, 4);
    for (int i = 0; i < n; ++i) { p[i] = 0.3 * sin(i * 0.7); }
    // warm start: the converged root perturbed by ~1e-3 relative (consecutive ADMM sweeps)
    *its = 0; k<<<1, 1>>>(p, w0, w0, cyc, its, n, 0); cudaDeviceSynchronize();
    for (int i = 0; i < n; ++i) {}
    for (int pass = 0; pass < 2; ++pass) {
        *its = 0;
        k<<<1, 1>>>(p, w0, out, cyc, its, n, pass);
        cudaDeviceSynchronize();
        printf("%s start: %.0f cycles/prox, %.2f Newton its/prox\n", pass ? "warm" : "cold", (double)*cyc / n, (double)*its / n);
    }
    kexp<<<1, 1>>>(p, out, cyc, n); cudaDeviceSynchronize();
    printf("exp: %.0f cycles (dependent chain)\n", (double)*cyc / n);
    kdiv<<<1, 1>>>(p, out, cyc, n); cudaDeviceSynchronize();
    printf("div: %.0f cycles (dependent chain)\n", (double)*cyc / n);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("sm clock attr %d kHz\n", clk);
    return 0;
}
