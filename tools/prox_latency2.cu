// Latency and accuracy of logistic-prox variants on the fused sweep's critical path:
//   ref : FP64 safeguarded Newton to the ulp (k_fused4 today)
//   mix : FP32 safeguarded Newton to ~1e-6, then ONE FP64 Newton step with the exact FP64
//         residual and the FP32 derivative (quasi-Newton: error ~1e-7 x 1e-7)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/prox_latency2.cu -o tools/prox_latency2
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ __forceinline__ double sig(double a) {
    if (a >= 0.0) return 1.0 / (1.0 + exp(-a));
    const double e = exp(a);
    return e / (1.0 + e);
}
__device__ double prox_ref(double rho, double b, double p, double w0) {
    double lo = p - 1.0 / rho, hi = p + 1.0 / rho;
    double w = (w0 > lo && w0 < hi) ? w0 : p;
    for (int it = 0; it < 60; ++it) {
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
    return w;
}
__device__ double prox_mix(double rho, double b, double p, double w0) {
    const double lo = p - 1.0 / rho, hi = p + 1.0 / rho;
    double w = (w0 > lo && w0 < hi) ? w0 : p;
    const float bf = (float)b, rf = (float)rho;
    // FP32 iterate on the offset y = w - p (well scaled even when |p| is large)
    float y = (float)(w - p), ylo = -1.0f / rf, yhi = 1.0f / rf;
    const float pf = (float)p;
    float gpf = rf;
    for (int it = 0; it < 30; ++it) {
        const float e = __expf(bf * (pf + y));                 // sigma(-b w) = 1 / (1 + e)
        const float sg = __frcp_rn(1.0f + e);
        const float g = -bf * sg + rf * y;
        if (g > 0.0f) yhi = y; else ylo = y;
        gpf = sg * (1.0f - sg) + rf;
        const float step = __fdividef(g, gpf);
        float yn = y - step;
        if (!(yn > ylo && yn < yhi)) yn = 0.5f * (ylo + yhi);
        const bool done = fabsf(yn - y) <= 2e-7f * fmaxf(fabsf(yn), 1e-30f) || yn == y;
        y = yn;
        if (done) break;
    }
    w = p + (double)y;
    // one FP64 step: exact residual, FP32 derivative
    const double sg = sig(-b * w);
    const double g = -b * sg + rho * (w - p);
    const double wn = w - g * (1.0 / (double)gpf);
    return (wn > lo && wn < hi) ? wn : w;
}
// fast FP64 exp: x = n ln2 + r (Cody-Waite, two-part ln2), |r| <= ln2/2, degree-11 Taylor
// (remainder < 2e-17 relative), 2^n by exponent construction; valid for |x| < 700
__device__ __forceinline__ double exp_fast(double x) {
    const double n = rint(x * 1.4426950408889634);
    double r = fma(n, -6.93147180369123816490e-01, x);
    r = fma(n, -1.90821492927058770002e-10, r);
    // Estrin evaluation of sum_{k<=11} r^k / k! (depth 5 instead of 11)
    const double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
    const double c01 = fma(r, 1.0, 1.0), c23 = fma(r, 1.6666666666666666e-01, 0.5);
    const double c45 = fma(r, 8.333333333333333e-03, 4.1666666666666664e-02);
    const double c67 = fma(r, 1.984126984126984e-04, 1.388888888888889e-03);
    const double c89 = fma(r, 2.7557319223985893e-06, 2.48015873015873e-05);
    const double cab = fma(r, 2.505210838544172e-08, 2.755731922398589e-07);
    const double c03 = fma(r2, c23, c01), c47 = fma(r2, c67, c45), c8b = fma(r2, cab, c89);
    const double q = fma(r8, c8b, fma(r4, c47, c03));
    const long long ni = (long long)n;
    return q * __longlong_as_double((ni + 1023) << 52);
}
// reciprocal: hardware approximation + two Newton refinements (~0.5 ulp)
__device__ __forceinline__ double rcp_fast(double a) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    double e = fma(-a, y, 1.0);
    y = fma(y, e, y);
    e = fma(-a, y, 1.0);
    return fma(y, e, y);
}
__device__ double prox_fast(double rho, double b, double p, double w0) {
    double lo = p - 1.0 / rho, hi = p + 1.0 / rho;
    double w = (w0 > lo && w0 < hi) ? w0 : p;
    for (int it = 0; it < 60; ++it) {
        const double t = -b * w;                                   // sigma(t) = sigma(-b w)
        const double e = exp_fast(-fabs(t));
        const double r = rcp_fast(1.0 + e);
        const double sg = t >= 0.0 ? r : e * r;
        const double g = -b * sg + rho * (w - p);
        if (g > 0.0) hi = w; else lo = w;
        const double step = g * rcp_fast(sg * (1.0 - sg) + rho);
        // quadratic convergence with |f''/2f'| <= 1/(8 rho): after a step <= 1e-9 the error
        // is below 1e-19 |w|, so the step is accepted without another evaluation
        if (fabs(step) <= 1e-9 * fmax(1.0, fabs(w))) { w -= step; break; }
        double wn = w - step;
        if (!(wn > lo && wn < hi)) wn = 0.5 * (lo + hi);
        w = wn;
    }
    return w;
}
__global__ void k(int variant, const double* p, const double* w0, const double* bb, double* out, long long* cyc, int n) {
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        const double w = variant == 2 ? prox_fast(4.0, bb[i], p[i], w0[i])
                         : variant ? prox_mix(4.0, bb[i], p[i], w0[i]) : prox_ref(4.0, bb[i], p[i], w0[i]);
        out[i] = w;
    }
    long long t1 = clock64();
    cyc[0] = t1 - t0;
}
int main() {
    const int n = 20000;
    std::vector<double> p(n), w0(n), b(n);
    srand(1);
    for (int i = 0; i < n; ++i) {
        double u = (rand() + 1.0) / (RAND_MAX + 2.0), v = (rand() + 1.0) / (RAND_MAX + 2.0);
        p[i] = 3.0 * sqrt(-2 * log(u)) * cos(2 * M_PI * v) + (i % 97 == 0 ? 40.0 : 0.0);
        b[i] = (i & 1) ? 1.0 : -1.0;
        w0[i] = p[i] + 0.1 * (rand() / (double)RAND_MAX - 0.5);   // warm start near the root
    }
    double *dp, *dw, *db, *o0, *o1;
    long long* dc;
    cudaMalloc(&dp, n * 8); cudaMalloc(&dw, n * 8); cudaMalloc(&db, n * 8); cudaMalloc(&o0, n * 8); cudaMalloc(&o1, n * 8);
    cudaMalloc(&dc, 8);
    cudaMemcpy(dp, p.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dw, w0.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), n * 8, cudaMemcpyHostToDevice);
    long long c0, c1;
    k<<<1, 1>>>(0, dp, dw, db, o0, dc, n); cudaMemcpy(&c0, dc, 8, cudaMemcpyDeviceToHost);
    k<<<1, 1>>>(1, dp, dw, db, o1, dc, n); cudaMemcpy(&c1, dc, 8, cudaMemcpyDeviceToHost);
    long long c2;
    double* o2;
    cudaMalloc(&o2, n * 8);
    k<<<1, 1>>>(2, dp, dw, db, o2, dc, n); cudaMemcpy(&c2, dc, 8, cudaMemcpyDeviceToHost);
    std::vector<double> r0(n), r1(n), r2(n);
    cudaMemcpy(r0.data(), o0, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(r1.data(), o1, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(r2.data(), o2, n * 8, cudaMemcpyDeviceToHost);
    double m1 = 0, m2 = 0;
    for (int i = 0; i < n; ++i) {
        m1 = fmax(m1, fabs(r1[i] - r0[i]) / fmax(1.0, fabs(r0[i])));
        m2 = fmax(m2, fabs(r2[i] - r0[i]) / fmax(1.0, fabs(r0[i])));
    }
    printf("ref %.0f cycles/prox; mix %.0f (max rel diff %.3e); fast %.0f (max rel diff %.3e)\n", (double)c0 / n,
           (double)c1 / n, m1, (double)c2 / n, m2);
    return 0;
}
