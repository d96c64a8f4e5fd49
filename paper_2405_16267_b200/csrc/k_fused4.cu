// k_fused4.cu -- host side of the single-HBM-read inner sweep on CTA pairs (SURVEY 8(f)
// row 1; the kernel and its design notes are in k_fused4.cuh): row groups, row batches,
// ring depth, axpy delay, launch.
#include <stdlib.h>

#include "k_fused4.cuh"

namespace bic {

// Compiled per-lane vector counts EV (2-element vectors of the half-row per main-warp lane):
// up to 9 (E = 18 doubles in registers for x and for the axpy accumulator each); more spills.
constexpr int kF4EVMax = 9;
static int f4_evmax(int dtype) { (void)dtype; return kF4EVMax; }
static int f4_vt(int dtype) { (void)dtype; return 2; }
// vectors per lane for a half-row of `half` elements over g row groups
static int64_t f4_ev(int dtype, int64_t half, int g) {
    const int64_t nv = (half + f4_vt(dtype) - 1) / f4_vt(dtype);
    const int64_t gt = 32 * (kF4Main / g);
    return (nv + gt - 1) / gt;
}

int fused4_max_cols(int dtype) { return 2 * kF4MainT * f4_vt(dtype) * f4_evmax(dtype); }

static size_t f4_half_elems(int64_t max_cols) { return (size_t)(((((max_cols + 3) / 4) * 4) / 2 + 3) / 4) * 4 + 4; }

// axpy delay D (in the group's own batches; the ring holds about ngrp (D + 1) batches):
// D = 2 (measured best at C2 FP64, 5 slots; BICADMM_F4_D overrides) but, with one group, at
// most nring - 3, so 2 slots keep loading (C3 shard, 4 slots of 50 KB: D = 1 runs at
// 6.15 TB/s, D = 2 at 5.87).  Always ngrp * D <= nring - 2.
static int f4_delay(int nring, int ngrp) {
    static int d = [] { const char* e = getenv("BICADMM_F4_D"); return e ? (atoi(e) < 1 ? 1 : atoi(e)) : 0; }();
    // ngrp > 1: D = 2 where the ring still keeps 2 slots loading, else 1 (C5 shard width
    // n_j = 6,250, two groups: FP64 4.33 vs 4.44 ms, FP32 3.10 vs 3.21 ms per 25 GB sweep;
    // tools/f4_plansweep.sh, profiles/r02_plansweep.md)
    int v = d ? d : 2;
    if (v < 1) v = 1;
    while (v > 1 && ngrp * v > nring - 2) --v;
    if (!d && ngrp == 1 && v > nring - 3) v = nring - 3 < 1 ? 1 : nring - 3;
    return v;
}

// The launch plan of a sweep whose widest node has max_cols columns:
//   R    rows per batch: slots of R half-rows stay <= 42 KB (at least 5 in the ring);
//        BICADMM_F4_R overrides (1, 2 or 4);
//   GR   row groups: the largest in {6, 4, 3, 2} whose W = 12 / GR warps still cover a
//        half-row within the compiled vector count (round 1, one row per batch: n = 4000 FP64
//        3 groups 1.87 ms per sweep vs 2 groups 2.05 ms; C5 shard (n_j = 6,250) 2 groups 17.7
//        ms vs 1 group 23.9), and for which the slot-reuse bound below leaves a ring of at
//        least GR + 2 slots (else fewer groups; BICADMM_F4_GROUPS overrides);
//   ring slots, axpy delay D: the dot / q / token slots are reused kF4Q / R batches later; the
//        peer CTA may run ahead of this CTA's prox warps by at most nring + GR (D + 1) batches
//         and CTA 1 sends its "inputs read" tokens P = kF4Prox batches ahead, so
//        nring + GR (D + 1) + P + 1 <= kF4Q / R (a tighter ring than that raced: R = 4 with
//        two row groups produced NaN at n = 300).
struct F4Plan {
    int R = 1, GR = 1, EV = -1, nring = 0, D = 1;
};
static F4Plan f4_plan(int dtype, int64_t max_cols) {
    max_cols = ((max_cols + 3) / 4) * 4;   // the same plan for the node width and its padded width
    F4Plan p;
    const size_t es = dtype == BICADMM_F64 ? 8 : 4;
    const size_t hb = f4_half_elems(max_cols) * es;
    static const int envR = [] { const char* e = getenv("BICADMM_F4_R"); return e ? atoi(e) : 0; }();
    static const int envG = [] { const char* e = getenv("BICADMM_F4_GROUPS"); return e ? atoi(e) : 0; }();
    p.R = (envR == 1 || envR == 2 || envR == 4) ? envR : 4 * hb <= 42 * 1024 ? 4 : 2 * hb <= 42 * 1024 ? 2 : 1;
    const int64_t half = ((max_cols / 2 + 3) / 4) * 4;   // the kernel's ch of the widest row (the larger half)
    auto fits = [&](int g, F4Plan& q) {   // EV within the compiled set and a feasible ring
        if (f4_ev(dtype, half, g) > f4_evmax(dtype)) return false;
        int nring = (int)(kF4RingBytes / (q.R * hb));
        if (const char* e = getenv("BICADMM_F4_RING")) nring = atoi(e) < nring ? atoi(e) : nring;
        nring = nring > kF4RingMax ? kF4RingMax : nring;
        const int QB = kF4Q / q.R;
        auto need = [&](int nr) { return nr + g * (f4_delay(nr, g) + 1) + kF4Prox + 1; };
        while (nring > 4 && need(nring) > QB) --nring;
        if (nring < 4 || nring < g + 2 || need(nring) > QB) return false;
        q.GR = g;
        q.nring = nring;
        q.D = f4_delay(nring, g);
        const int64_t ev = f4_ev(dtype, half, g);
        q.EV = ev <= 1 ? 1 : ev <= 2 ? 2 : ev <= 4 ? 4 : ev <= 6 ? 6 : ev <= 7 ? 7 : ev <= 8 ? 8 : ev <= 9 ? 9 : -1;
        return q.EV > 0;
    };
    for (; p.R >= 1; p.R /= 2) {
        if ((envG == 1 || envG == 2 || envG == 3 || envG == 4 || envG == 6) && fits(envG, p)) return p;
        const int cand[5] = {6, 4, 3, 2, 1};
        for (int k = 0; k < 5; ++k)
            if (fits(cand[k], p)) return p;
    }
    p.EV = -1;
    return p;
}

bool fused4_plan_ok(int dtype, int64_t max_cols) { return f4_plan(dtype, max_cols).EV > 0; }

int fused4_groups(int dtype, int64_t max_cols) {
    const F4Plan p = f4_plan(dtype, max_cols);
    return p.EV > 0 ? p.GR : 1;
}

extern "C" int bicadmm_debug_f4_trace(void* dev_buf) {   // trace builds only (BIC_F4_TRACE); else a no-op
    const int r1 = f4_trace_set_r1(dev_buf), r2 = f4_trace_set_r2(dev_buf), r4 = f4_trace_set_r4(dev_buf);
    return r1 ? r1 : r2 ? r2 : r4;
}

// 1 in a protocol-check build (tools/build_f4_variant.sh f4check -DBIC_F4_CHECK), 0 in the product
extern "C" int bicadmm_debug_f4_check_build(void) {
#ifdef BIC_F4_CHECK
    return 1;
#else
    return 0;
#endif
}

// check builds only (BIC_F4_CHECK): tag mismatches seen so far (0 in product builds)
extern "C" unsigned long long bicadmm_debug_f4_errors(void) {
    unsigned long long a = 0, b = 0, c = 0;
    f4_errors_r1(&a);
    f4_errors_r2(&b);
    f4_errors_r4(&c);
    return a + b + c;
}

int launch_fused4(int dtype, const Fused2Args& a, int loss, double rho, int grid, cudaStream_t s) {
    int64_t maxc = 0;
    for (int k = 0; k < a.nn; ++k) maxc = a.ncols[k] > maxc ? a.ncols[k] : maxc;
    if (a.max_cols_pad < maxc || (grid & 1)) return BICADMM_ERR_INVALID;
    const F4Plan p = f4_plan(dtype, a.max_cols_pad);
    if (p.EV < 0) return BICADMM_ERR_INVALID;
    const size_t es = dtype == BICADMM_F64 ? 8 : 4;
    // TMA bulk copies: both half-rows start 16-byte aligned (ch % 4 == 0, lda * size % 16 == 0);
    // a half-row of an odd number of float pairs is copied rounded up to 16 bytes, inside lda
    for (int k = 0; k < a.nn; ++k)
        if ((a.ncols[k] & 1) || (a.lda[k] * (int64_t)es) % 16) return BICADMM_ERR_INVALID;
    const size_t half_el = (size_t)(((a.max_cols_pad / 2 + 3) / 4) * 4 + 4);   // the kernel's half_pad
    const size_t smem = (size_t)p.nring * p.R * half_el * es;
    if (smem > (size_t)kF4RingBytes) return BICADMM_ERR_INVALID;
    int rc;
    switch (p.R) {
    case 1: rc = f4_launch_r1(dtype, p.GR, p.EV, a, loss, rho, p.nring, p.D, smem, grid, s); break;
    case 2: rc = f4_launch_r2(dtype, p.GR, p.EV, a, loss, rho, p.nring, p.D, smem, grid, s); break;
    case 4: rc = f4_launch_r4(dtype, p.GR, p.EV, a, loss, rho, p.nring, p.D, smem, grid, s); break;
    default: rc = BICADMM_ERR_INVALID;
    }
    if (rc) return rc;
    BIC_LAUNCHED();
    return BICADMM_OK;
}

}  // namespace bic
