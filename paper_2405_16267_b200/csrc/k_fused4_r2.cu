// k_fused4_r2.cu -- instances of the single-pass sweep (k_fused4.cuh) with row batches of 2.
#include "k_fused4.cuh"

namespace bic {

int f4_launch_r2(int dtype, int GR, int EV, const Fused2Args& a, int loss, double rho, int nring, int dly, size_t smem,
                 int grid, cudaStream_t s) {
#define F4_GR(TT)                                                                             \
    switch (GR) {                                                                             \
    case 1: return f4_launch_inst<TT, 1, 2>(EV, a, loss, rho, nring, dly, smem, grid, s);      \
    case 2: return f4_launch_inst<TT, 2, 2>(EV, a, loss, rho, nring, dly, smem, grid, s);      \
    case 3: return f4_launch_inst<TT, 3, 2>(EV, a, loss, rho, nring, dly, smem, grid, s);      \
    case 4: return f4_launch_inst<TT, 4, 2>(EV, a, loss, rho, nring, dly, smem, grid, s);      \
    case 6: return f4_launch_inst<TT, 6, 2>(EV, a, loss, rho, nring, dly, smem, grid, s);      \
    default: return BICADMM_ERR_INVALID;                                                      \
    }
    if (dtype == BICADMM_F64) { F4_GR(double) } else { F4_GR(float) }
#undef F4_GR
}

int f4_trace_set_r2(void* p) {
#ifdef BIC_F4_TRACE
    long long* q = static_cast<long long*>(p);
    return cudaMemcpyToSymbol(g_f4_trace, &q, sizeof(q)) == cudaSuccess ? 0 : -6;
#else
    (void)p;
    return 0;
#endif
}

int f4_errors_r2(unsigned long long* out) {
#ifdef BIC_F4_CHECK
    return cudaMemcpyFromSymbol(out, g_f4_errors, sizeof(*out)) == cudaSuccess ? 0 : -6;
#else
    *out = 0;
    return 0;
#endif
}

}  // namespace bic
