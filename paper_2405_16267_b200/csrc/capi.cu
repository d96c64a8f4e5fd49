// capi.cu -- the C ABI of libbicadmm (include/bicadmm.h): handle, workspace
// plan, one-time setup, the outer/inner iteration driver, finalize, NCCL comm.
//
// Iteration order (Eq. (7) order, DESIGN R2), per outer iteration k:
//   Algorithm 2, K_in sweeps for every local node:
//      a1+a2  gemv_t : r_ij = rho_l A_ij^T (p_ij + delta_i) + rho_c (z_j - u_ij)
//      a3     gemv   : x_ij = H_ij r_ij
//      a4     gemv   : p_ij = A_ij x_ij
//      a5     block sum (+ NCCL AllReduce over the node group when blocks span GPUs)
//      a6+a7  prox   : abar, omega_bar (22), nu (23), delta
//   Algorithm 1, replicated on every rank:
//      a9  Collect   : wsum = sum_i (x_i + u_i) (+ NCCL AllReduce over all ranks)
//      a10 (7b)      : z, t
//      a11 (13)      : s
//      a12 (14)      : v;  (9) u_i += x_i - z;  (15) p_r, d_r, b_r -> host (one sync)
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/bicadmm.h"
#include "../../include/bicadmm_ops.h"
#include "comm.h"
#include "common.cuh"
#include "kernels.h"

// NVTX ranges around the ABI entry points (header-only NVTX v3: no-ops unless a profiler
// injects itself, e.g. nsys; names "bicadmm_setup", "bicadmm_iterate", ...)
#include <nvtx3/nvToolsExt.h>
namespace {
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

using namespace bic;

// ======================================================================= handle
namespace {

struct LBlock {      // a local block (i, j), sorted by (node, block)
    int node, block, user_index, li, jl;
    const void* A;
    int64_t lda, m, c0, nj;
    void* ready = nullptr;   // caller's cudaEvent_t for A (setup only; bicadmm_block.ready_event)
    void* H;         // tall block: H = (rho_l A^T A + c I)^{-1} (nj x nj); fat block (Woodbury,
    int64_t ldh;     // m < nj): K^{-1} = ((c/rho_l) I + A A^T)^{-1} (m x m)
    bool fat = false;
    int64_t kd = 0;  // factor order: fat ? m : nj
    double* t1 = nullptr;   // fat: m * C scratch (A (z - u), then K^{-1} q)
    double* w0 = nullptr;   // fat: (rho_c/rho_l) K^{-1} A (z - u), fixed within an inner loop
    double* qd = nullptr;   // fat: q of the last sweep, then q - p (x materialization)
    double* zu = nullptr;   // fat: z_j - u_ij (n_j * C)
    bool hpack = false;     // H stored as packed lower tiles (k_symv.cu); C == 1 only
    double* hpart = nullptr;
    double *x, *u, *r, *p, *partial, *pobj;
    double* partial2 = nullptr;   // single-pass sweep: [clusters touching the node x row groups][nj]
    double* xt = nullptr;         // C > 1: class-major scratch (nj * C)
};
struct LNode {
    int node, li;
    int64_t m;
    const void* b;
    double *nu, *delta, *S, *p_base, *pobj_base, *sq_partial, *obj_partial, *obar;
    int np;
    int64_t nprox_ctas;
};

struct Bump {  // 256-byte aligned bump allocator over the workspace (base may be null to size)
    char* base;
    size_t off = 0;
    explicit Bump(void* b) : base((char*)b) {}
    void* take(size_t bytes) {
        off = (off + 255) / 256 * 256;
        void* p = base ? base + off : nullptr;
        off += bytes;
        return p;
    }
    template <typename T> T* arr(int64_t n) { return (T*)take(sizeof(T) * (size_t)(n > 0 ? n : 1)); }
};

int64_t rup(int64_t a, int64_t b) { return (a + b - 1) / b * b; }
constexpr int kLoopRows = 4096;   // outer iterations per device-loop launch

// Static row split of all local rows over `units` equal ranges (one per CTA or CTA pair):
// for each node, the first unit touching it and how many units touch it.
void touching_units(const std::vector<int64_t>& node_rows, int units, std::vector<int64_t>& lo_out,
                    std::vector<int64_t>& n_out) {
    const size_t nl = node_rows.size();
    int64_t tot = 0;
    std::vector<int64_t> off;
    for (size_t k = 0; k < nl; ++k) { off.push_back(tot); tot += node_rows[k]; }
    lo_out.assign(nl, 0);
    n_out.assign(nl, 0);
    for (size_t k = 0; k < nl; ++k) {
        const int64_t r0 = off[k], r1 = off[k] + node_rows[k];
        int64_t lo = -1, hi = -1;
        for (int c = 0; c < units; ++c) {
            const int64_t cb = (int64_t)c * tot / units, ce = (int64_t)(c + 1) * tot / units;
            if (cb < ce && cb < r1 && ce > r0) { if (lo < 0) lo = c; hi = c; }
        }
        lo_out[k] = lo < 0 ? 0 : lo;
        n_out[k] = lo < 0 ? 0 : hi - lo + 1;
    }
}

}  // namespace

struct bicadmm_handle {
    // problem
    int N = 0, M = 0, C = 1, loss = 0, dtype = 0;
    int64_t n = 0, len = 0, lenp = 0;   // lenp: 64-byte aligned per-node stride of x_all / u_all
    std::vector<int64_t> m, col_start;
    bicadmm_params prm{};
    bicadmm_comm* comm = nullptr;
    int gsize = 1;              // ranks of this rank's node group (comm_group_size at setup)
    double* S_all = nullptr;    // block sums S_i of all local nodes, contiguous (nod[].S point into it)
    int64_t S_total = 0;
    bool split_blocks = false;  // some node's blocks live on other ranks
    bool any_fat = false;       // some local block takes the Woodbury path
    cudaStream_t st = nullptr;
    int sm_count = 148, gemv_cap = 148;
    size_t ws_bytes = 0;
    // layout
    std::vector<LBlock> blk;
    std::vector<LNode> nod;
    double *x_all = nullptr, *u_all = nullptr, *z = nullptr, *z_prev = nullptr, *s = nullptr, *wbar = nullptr,
           *wsum = nullptr, *x_final = nullptr, *node_sq = nullptr, *upart = nullptr, *gram = nullptr,
           *fws = nullptr, *node_obj = nullptr;
    int fbatch = 1;                          // blocks factored together (factor_inverse_batched)
    void* gtc_ws = nullptr;                  // tcgen05 Gram scratch (int8 slices + column scales)
    size_t gtc_bytes = 0;
    // logistic refit on the support (DESIGN R29): gathered support columns and Newton scratch
    int64_t rf_kp = 0, rf_rows = 0, rf_nparts = 0;
    double *rf_AT = nullptr, *rf_BT = nullptr, *rf_b = nullptr, *rf_w = nullptr, *rf_psi = nullptr,
           *rf_sd = nullptr, *rf_obj = nullptr, *rf_x = nullptr, *rf_g = nullptr, *rf_d = nullptr,
           *rf_F = nullptr, *rf_H = nullptr, *rf_ws = nullptr, *rf_part = nullptr, *rf_r = nullptr,
           *rf_U = nullptr, *rf_W = nullptr, *rf_G = nullptr, *rf_P = nullptr, *rf_F2 = nullptr, *rf_X = nullptr,
           *rf_Y = nullptr, *rf_xt = nullptr;   // softmax (C classes)
    GemvTDesc rf_gt{};
    int rf_newton = 0;
    int64_t gram_stride = 0, fws_stride = 0; // per-job setup scratch (doubles)
    double *x_old = nullptr, *dpart = nullptr, *node_dx = nullptr, *node_res = nullptr;
    double *mask = nullptr, *cg_r = nullptr, *cg_p = nullptr, *cg_Ap = nullptr, *cg_rhs = nullptr, *cg_sc = nullptr;
    int refit_iters = 0;
    // single-pass sweep (k_fused4.cu): CTA-pair clusters over static row ranges
    bool fused = false;
    int fused_kind = 0;            // 0 two-pass, 4 single pass (k_fused4), 5 small nodes in one CTA
                                   // (k_small_sweeps); BICADMM_FIELD_SWEEP_KIND
    std::vector<SmallNode> small;  // kind 5: one descriptor per node
    std::vector<GemvTDesc> gtf;
    Fused2Args f2{};
    int f2grid = 0;
    std::vector<int64_t> f2_cta_lo, f2_cta_n;   // per local node: first cluster touching it, count
    OuterScalars* sc = nullptr;
    int64_t* support = nullptr;
    int64_t* support_count = nullptr;
    // launch descriptors
    std::vector<GemvTDesc> gt;
    std::vector<BlockVec> bv;
    // host state
    OuterScalars* host_sc = nullptr;  // pinned
    int64_t* host_i64 = nullptr;      // pinned
    int outer_done = 0;
    int64_t inner_total = 0;
    std::vector<std::array<double, 6>> trace;
    std::vector<int32_t> inner_counts;
    std::vector<int32_t> schedule;
    int sched_start = 0, sched_rows = 0;
    bool dead = false, finalized = false, converged = false;
    int64_t support_len = 0;
    double objective = 0.0, ms_setup = 0.0, ms_solve = 0.0;
    int64_t launches0 = 0;
    std::string err;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int32_t host_i32[2] = {};
    bool capturing = false;   // inside the stream capture of graph_outer
    // device-resident solve loop (bicadmm_solve): a CUDA-graph while node around one outer
    // iteration, terminated on the device; trace rows appended on the device
    double* dtrace = nullptr;         // [kLoopRows][6]
    int* dcount = nullptr;
    int* label_bad = nullptr;         // setup's label-domain check (BICADMM_ERR_DOMAIN)
    double* place_chk = nullptr;      // setup's collective placement check: 2 (N M) + 1 doubles
    struct Loop {
        cudaGraphExec_t exec = nullptr;
        int sweeps = -1;
        int64_t launches = 0;
        bool failed = false;
    } loop;
    cudaStream_t cap_st = nullptr;   // private capture stream (the caller's may be the legacy stream)
    // per-phase profiling (bicadmm_set_profiling)
    bool prof = false;
    std::vector<cudaEvent_t> evpool;
    size_t evused = 0;
    struct Pending { int phase; cudaEvent_t a, b; int64_t launches; };
    std::vector<Pending> pending;
    // CUDA graph of one outer iteration (fixed inner schedule): captured once, replayed
    struct Graph {
        cudaGraphExec_t exec = nullptr;
        bool prof = false, failed = false;
        int sweeps = -1;
        int64_t launches = 0;
        std::vector<Pending> pending;   // phase events recorded by the graph's event nodes
    } graph;
    double phase_ms[BICADMM_NPHASE] = {};
    int64_t phase_cnt[BICADMM_NPHASE] = {};
};

// Record a phase event; inside a stream capture it becomes an event-record node.
static void rec_event(bicadmm_handle* h, cudaEvent_t e) { record_event(e, h->st); }

static cudaEvent_t next_event(bicadmm_handle* h) {
    if (h->evused == h->evpool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        h->evpool.push_back(e);
    }
    return h->evpool[h->evused++];
}

// Resolve recorded phase events (call only after the stream has been synchronised).
static void resolve_phases(bicadmm_handle* h) {
    for (auto& p : h->pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) h->phase_ms[p.phase] += ms;
        h->phase_cnt[p.phase] += p.launches;
    }
    h->pending.clear();
    h->evused = 0;
}

static int fail(bicadmm_handle* h, int rc, const std::string& msg) {
    if (h) {
        h->err = msg;
        if (rc == BICADMM_ERR_CUDA || rc == BICADMM_ERR_NCCL) h->dead = true;
    }
    return rc;
}

#define H_CUDA(h, expr)                                                                                \
    do {                                                                                               \
        cudaError_t _e = (expr);                                                                       \
        if (_e != cudaSuccess) return fail(h, BICADMM_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(_e)); \
    } while (0)
#define H_RC(h, expr)                                                                                  \
    do {                                                                                               \
        int _r = (expr);                                                                               \
        if (_r != BICADMM_OK) {                                                                        \
            if (_r == BICADMM_ERR_CUDA) return fail(h, _r, std::string(#expr ": ") + cudaGetErrorString(cudaGetLastError())); \
            return fail(h, _r, #expr);                                                                 \
        }                                                                                              \
    } while (0)

// ----------------------------------------------------------------------- validation
static int validate(const bicadmm_problem* P, const bicadmm_params* R, std::string* why) {
    if (!P || !R || !P->m || !P->col_start || (P->n_blocks > 0 && !P->blocks) || !P->b) { *why = "null pointer"; return BICADMM_ERR_INVALID; }
    if (P->N < 1 || P->M < 1 || P->n < 1 || P->C < 1) { *why = "N, M, n, C must be >= 1"; return BICADMM_ERR_DIM; }
    if (P->loss < 0 || P->loss > 3) { *why = "unknown loss"; return BICADMM_ERR_INVALID; }
    if (P->dtype != BICADMM_F64 && P->dtype != BICADMM_F32) { *why = "unknown dtype"; return BICADMM_ERR_INVALID; }
    if ((P->loss == BICADMM_SOFTMAX) != (P->C > 1)) { *why = "C > 1 iff softmax"; return BICADMM_ERR_DIM; }
    if (P->C > 16) { *why = "C <= 16 classes"; return BICADMM_ERR_INVALID; }
    if (P->col_start[0] != 0 || P->col_start[P->M] != P->n) { *why = "col_start must span [0, n]"; return BICADMM_ERR_DIM; }
    for (int j = 0; j < P->M; ++j) {
        if (P->col_start[j + 1] <= P->col_start[j]) { *why = "col_start not increasing"; return BICADMM_ERR_DIM; }
        if (P->col_start[j] % 4) { *why = "col_start[j] must be a multiple of 4"; return BICADMM_ERR_INVALID; }
    }
    for (int i = 0; i < P->N; ++i) if (P->m[i] < 1) { *why = "m_i must be >= 1"; return BICADMM_ERR_DIM; }
    if (P->n_blocks < 1) { *why = "no local blocks"; return BICADMM_ERR_PLACEMENT; }
    std::vector<char> seen((size_t)P->N * P->M, 0);
    for (int k = 0; k < P->n_blocks; ++k) {
        const bicadmm_block& b = P->blocks[k];
        if (b.node < 0 || b.node >= P->N || b.block < 0 || b.block >= P->M) { *why = "block id out of range"; return BICADMM_ERR_PLACEMENT; }
        if (seen[(size_t)b.node * P->M + b.block]++) { *why = "duplicate block"; return BICADMM_ERR_PLACEMENT; }
        const int64_t nj = P->col_start[b.block + 1] - P->col_start[b.block];
        if (!b.A) { *why = "null block pointer"; return BICADMM_ERR_INVALID; }
        if (b.lda < nj || b.lda % 4 || ((uintptr_t)b.A) % 16) { *why = "A must be 16-byte aligned with lda >= n_j, lda % 4 == 0"; return BICADMM_ERR_INVALID; }
        if (!P->b[b.node]) { *why = "missing labels for a node with a local block"; return BICADMM_ERR_PLACEMENT; }
    }
    if (R->kappa < 0 || R->kappa > P->n * P->C) { *why = "kappa outside [0, n*C]"; return BICADMM_ERR_INVALID; }
    if (!(R->rho_c > 0) || !(R->rho_l > 0) || !(R->lambda > 0)) { *why = "penalties must be > 0"; return BICADMM_ERR_INVALID; }
    if (!(R->alpha > 0 && R->alpha <= 1)) { *why = "alpha must be in (0, 1]"; return BICADMM_ERR_INVALID; }
    if (R->eps_p < 0 || R->eps_d < 0 || R->eps_b < 0 || R->eps_inner < 0) { *why = "tolerances must be >= 0"; return BICADMM_ERR_INVALID; }
    if (R->inner_fixed < 0 || (R->inner_fixed == 0 && R->max_inner < 1)) { *why = "inner schedule"; return BICADMM_ERR_INVALID; }
    return BICADMM_OK;
}

// Layout of the workspace (also used to size it).  Returns bytes.
static size_t plan(bicadmm_handle* h, const bicadmm_problem* P, void* base) {
    Bump b(base);
    const int C = P->C;
    const int64_t len = P->n * C;
    const int64_t lenp = rup(len, 8);
    h->lenp = lenp;
    h->blk.clear();
    h->nod.clear();
    for (int k = 0; k < P->n_blocks; ++k) {
        LBlock L{};
        L.node = P->blocks[k].node;
        L.block = P->blocks[k].block;
        L.user_index = k;
        L.A = P->blocks[k].A;
        L.lda = P->blocks[k].lda;
        L.ready = P->blocks[k].ready_event;
        L.m = P->m[L.node];
        L.c0 = P->col_start[L.block];
        L.nj = P->col_start[L.block + 1] - L.c0;
        h->blk.push_back(L);
    }
    std::sort(h->blk.begin(), h->blk.end(), [](const LBlock& a, const LBlock& c) {
        return a.node != c.node ? a.node < c.node : a.block < c.block;
    });
    for (auto& L : h->blk) {
        if (h->nod.empty() || h->nod.back().node != L.node) {
            LNode nd{};
            nd.node = L.node;
            nd.li = (int)h->nod.size();
            nd.m = L.m;
            nd.b = P->b[L.node];
            h->nod.push_back(nd);
        }
        L.li = h->nod.back().li;
        L.jl = h->nod.back().np++;
    }
    const int nl = (int)h->nod.size();
    // Woodbury fat-block path (R27) unless BICADMM_WOODBURY=0
    const char* wb = getenv("BICADMM_WOODBURY");
    const bool wb_on = !(wb && atoi(wb) == 0);
    int64_t kdmax = 0;
    for (auto& L : h->blk) {
        L.fat = wb_on && L.m < L.nj;
        L.kd = L.fat ? L.m : L.nj;
        kdmax = std::max(kdmax, L.kd);
        h->any_fat = h->any_fat || L.fat;
    }
    // matrices
    const size_t es = P->dtype == BICADMM_F64 ? 8 : 4;
    const char* hp = getenv("BICADMM_HPACK");
    const bool hp_on = C == 1 && !(hp && atoi(hp) == 0);
    for (auto& L : h->blk) {
        L.ldh = rup(L.kd, 4);
        L.hpack = hp_on;
        L.H = b.take(es * (size_t)(L.hpack ? symv_packed_elems(L.kd) : L.ldh * L.kd));
        L.hpart = L.hpack ? b.arr<double>(symv_part_doubles(L.kd)) : nullptr;
    }
    // global vectors
    h->x_all = b.arr<double>(lenp * nl);
    h->u_all = b.arr<double>(lenp * nl);
    h->z = b.arr<double>(len);
    h->z_prev = b.arr<double>(len);
    h->s = b.arr<double>(len);
    h->wbar = b.arr<double>(len);
    h->wsum = b.arr<double>(len);
    h->x_final = b.arr<double>(len);
    h->node_sq = b.arr<double>(P->N);
    h->node_obj = b.arr<double>(P->N);
    h->sc = b.arr<OuterScalars>(1);
    h->support = b.arr<int64_t>(P->n * C);
    h->support_count = b.arr<int64_t>(1);
    int64_t uparts = 0;
    for (auto& L : h->blk) uparts += (L.nj * C + kUThreads * 4 - 1) / (kUThreads * 4);
    h->upart = b.arr<double>(uparts);
    h->dpart = b.arr<double>(uparts);
    h->x_old = b.arr<double>(lenp * nl);
    h->node_dx = b.arr<double>(P->N);
    h->node_res = b.arr<double>(P->N);
    // per node; the block sums S_i of all local nodes are contiguous, so Algorithm 2's
    // per-sweep AllReduce is one collective over all of them
    int64_t s_total = 0;
    for (auto& nd : h->nod) s_total += nd.m * C;
    h->S_all = b.arr<double>(s_total);
    h->S_total = s_total;
    int64_t s_off = 0;
    for (auto& nd : h->nod) {
        nd.nu = b.arr<double>(nd.m * C);
        nd.delta = b.arr<double>(nd.m * C);
        nd.S = h->S_all + (base ? s_off : 0);
        s_off += nd.m * C;
        nd.obar = b.arr<double>(nd.m * C);
        nd.p_base = b.arr<double>(nd.m * C * nd.np);
        nd.pobj_base = b.arr<double>(nd.m * C * nd.np);
        nd.nprox_ctas = (nd.m + kProxThreads - 1) / kProxThreads;
        nd.sq_partial = b.arr<double>(nd.nprox_ctas);
        nd.obj_partial = b.arr<double>(nd.nprox_ctas);
    }
    // per block vectors + gemv_t scratch
    h->gt.assign(h->blk.size(), GemvTDesc{});
    for (size_t k = 0; k < h->blk.size(); ++k) {
        h->gt[k].rows = h->blk[k].m;
        h->gt[k].cols = h->blk[k].nj;
    }
    std::vector<int64_t> need(h->blk.size());
    plan_gemv_t(P->dtype, h->gt.data(), (int)h->gt.size(), h->sm_count, need.data(), C);
    for (size_t k = 0; k < h->blk.size(); ++k) {
        LBlock& L = h->blk[k];
        LNode& nd = h->nod[L.li];
        L.x = h->x_all + (base ? (int64_t)L.li * lenp + L.c0 * C : 0);
        L.u = h->u_all + (base ? (int64_t)L.li * lenp + L.c0 * C : 0);
        L.p = nd.p_base + (base ? (int64_t)L.jl * nd.m * C : 0);
        L.r = b.arr<double>(L.nj * C);
        L.xt = C > 1 ? b.arr<double>(L.nj * C) : nullptr;
        L.pobj = nd.pobj_base + (base ? (int64_t)L.jl * nd.m * C : 0);
        L.partial = b.arr<double>(need[k]);
        L.t1 = L.fat ? b.arr<double>(L.m * C) : nullptr;
        L.w0 = L.fat ? b.arr<double>(L.m * C) : nullptr;
        L.qd = L.fat ? b.arr<double>(L.m * C) : nullptr;
        L.zu = L.fat ? b.arr<double>(L.nj * C) : nullptr;
    }
    // setup scratch: FP64 Gram / factor workspace
    const int64_t ldg = rup(kdmax, 8);
    h->mask = b.arr<double>(len);
    h->dtrace = b.arr<double>((int64_t)kLoopRows * 6);
    h->dcount = b.arr<int>(2);
    h->label_bad = b.arr<int>(1);
    h->place_chk = b.arr<double>(2 * (int64_t)P->N * P->M + 1);
    if (((P->loss == BICADMM_LOGISTIC && C == 1) || P->loss == BICADMM_SOFTMAX) && h->prm.refit) {
        int64_t rows = 0;
        for (auto& nd : h->nod) rows += nd.m;
        const int64_t kk = std::max<int64_t>(1, std::min<int64_t>(h->prm.kappa, len));
        const int64_t kp = rup(kk, 4);
        h->rf_kp = kp;
        h->rf_rows = rows;
        h->rf_nparts = rf_logit_parts(rows);
        h->rf_AT = b.arr<double>(rows * kp);
        h->rf_BT = b.arr<double>(rows * kp);
        h->rf_b = b.arr<double>(rows);
        h->rf_w = b.arr<double>(rows);
        h->rf_psi = b.arr<double>(rows);
        h->rf_sd = b.arr<double>(rows);
        h->rf_obj = b.arr<double>(h->rf_nparts);
        h->rf_x = b.arr<double>(kp);
        h->rf_g = b.arr<double>(kp);
        h->rf_d = b.arr<double>(kp);
        h->rf_r = b.arr<double>(kp);
        h->rf_F = b.arr<double>(rup(kp, 8) * kp);
        h->rf_H = b.arr<double>(kp * kp);
        h->rf_ws = b.arr<double>((int64_t)factor_ws_doubles(kp));
        GemvTDesc g{};
        g.rows = rows; g.cols = kp;
        int64_t need = 0;
        plan_gemv_t(BICADMM_F64, &g, 1, h->sm_count, &need, C);
        h->rf_gt = g;
        h->rf_part = b.arr<double>(need);
        if (C > 1) {
            h->rf_U = b.arr<double>(rows * kp);
            h->rf_W = b.arr<double>(rows * C);
            h->rf_G = b.arr<double>(rows * C);
            h->rf_P = b.arr<double>(rows * C);
            h->rf_F2 = b.arr<double>(rup(kp, 8) * kp);
            h->rf_X = b.arr<double>(kp * C);
            h->rf_Y = b.arr<double>(kp * C);
            h->rf_xt = b.arr<double>(kp * C);
        }
    }
    h->cg_r = b.arr<double>(len);
    h->cg_p = b.arr<double>(len);
    h->cg_Ap = b.arr<double>(len);
    h->cg_rhs = b.arr<double>(len);
    h->cg_sc = b.arr<double>(8);
    {   // single-pass sweep: static row ranges of the CTA pairs; partials per node over the
        // (cluster, row group) pairs touching it
        std::vector<int64_t> rows;
        for (auto& nd : h->nod) rows.push_back(nd.m);
        std::vector<int64_t> lo4, n4;
        touching_units(rows, std::max(1, h->sm_count / 2), lo4, n4);
        int64_t maxc = 0;
        for (auto& L : h->blk) maxc = std::max(maxc, L.nj);
        const int64_t g4 = fused4_groups(P->dtype, maxc);
        for (auto& L : h->blk)
            if (L.jl == 0) L.partial2 = b.arr<double>(std::max<int64_t>(1, n4[L.li] * g4) * L.nj * C);
    }
    {   // setup scratch for up to 8 blocks factored in lockstep (BICADMM_FACTOR_BATCH caps it;
        // the extra scratch is limited to ~8 GB)
        h->gram_stride = rup(ldg * kdmax, 32);
        h->fws_stride = rup((int64_t)factor_ws_doubles(kdmax), 32);
        const double per_job = 8.0 * (double)(h->gram_stride + h->fws_stride);
        int fb = (int)std::min<int64_t>(8, (int64_t)h->blk.size());
        while (fb > 1 && per_job * (fb - 1) > 8e9) --fb;
        if (const char* e = getenv("BICADMM_FACTOR_BATCH")) fb = std::max(1, std::min(fb, atoi(e)));
        h->fbatch = std::max(1, fb);
        h->gram = b.arr<double>(h->gram_stride * h->fbatch);
        h->fws = b.arr<double>(h->fws_stride * h->fbatch);
        // tcgen05 Ozaki-scheme Gram (k_gram_tc.cu) for tall blocks: slices of up to 32,768 rows
        // and the factor's large products (factor_inverse_batched), sharing the scratch
        size_t gtc = 0;
        if (gram_tc_enabled())
            for (auto& L : h->blk) {
                if (!L.fat) gtc = std::max(gtc, gram_tc_scratch_bytes(P->dtype, L.m, L.nj));
                gtc = std::max(gtc, factor_tc_scratch_bytes(L.kd));
            }
        h->gtc_bytes = gtc;
        h->gtc_ws = gtc ? b.take(gtc) : nullptr;
    }
    return b.off + 256;
}

static void build_descs(bicadmm_handle* h) {
    const int C = h->C;
    (void)C;
    for (size_t k = 0; k < h->blk.size(); ++k) {
        LBlock& L = h->blk[k];
        GemvTDesc& g = h->gt[k];
        g.A = L.A; g.lda = L.lda; g.rows = L.m; g.cols = L.nj;
        g.p = L.p; g.delta = h->nod[L.li].delta;
        g.z = h->z + L.c0 * h->C; g.u = L.u; g.r = L.r; g.partial = L.partial;
    }
    h->bv.clear();
    for (auto& L : h->blk) {
        BlockVec v{};
        v.x = L.x; v.u = L.u; v.c0 = L.c0 * h->C; v.len = L.nj * h->C; v.node = L.node;
        h->bv.push_back(v);
    }
}

// Single-pass sweep (k_fused4.cu) eligibility: every node's blocks local and one block per
// node, C == 1, tall blocks, 16-byte row pieces, rows up to fused4_max_cols with a feasible plan.
static bool fused4_eligible(bicadmm_handle* h) {
    if (h->split_blocks || h->C != 1 || (int)h->nod.size() > kF2MaxNodes || h->sm_count < 2) return false;
    for (auto& nd : h->nod) if (nd.np != 1) return false;
    const int64_t es = h->dtype == BICADMM_F64 ? 8 : 4;
    int64_t maxc = 0;
    for (auto& L : h->blk) {
        // whole 2-element vectors per half-row; rows 16-byte aligned (a half-row whose bytes are
        // not a 16-byte multiple is copied rounded up into the row's own padding, inside lda)
        if (L.fat || L.nj > fused4_max_cols(h->dtype) || L.nj < 8 || (L.nj & 1) || (L.lda * es) % 16) return false;
        maxc = std::max(maxc, L.nj);
    }
    // and a launch plan exists for the widest row: FP64 half-rows past 52.5 KB (n_j > 13,432)
    // leave fewer than 4 ring slots
    return fused4_plan_ok(h->dtype, maxc);
}

static int build_fused4(bicadmm_handle* h) {
    Fused2Args& a = h->f2;
    a = Fused2Args{};
    int64_t R = 0, maxc = 0;
    // row ranges per CTA pair (cluster of 2); each cluster writes one partial row per row group
    std::vector<int64_t> rows;
    for (auto& nd : h->nod) rows.push_back(nd.m);
    touching_units(rows, h->sm_count / 2, h->f2_cta_lo, h->f2_cta_n);
    int64_t mc = 0;
    for (auto& L : h->blk) mc = std::max(mc, L.nj);
    const int64_t groups = fused4_groups(h->dtype, mc);
    a.nn = (int)h->nod.size();
    for (auto& L : h->blk) {
        const LNode& nd = h->nod[L.li];
        const int k = L.li;
        a.A[k] = L.A; a.b[k] = nd.b; a.x[k] = L.x; a.p[k] = L.p; a.nu[k] = nd.nu; a.delta[k] = nd.delta;
        a.partial[k] = L.partial2; a.lda[k] = L.lda; a.ncols[k] = L.nj; a.row_off[k] = R;
        a.cta_lo[k] = h->f2_cta_lo[k];
        R += L.m;
        maxc = std::max(maxc, L.nj);
        H_CUDA(h, cudaMemsetAsync(L.partial2, 0, sizeof(double) * std::max<int64_t>(1, h->f2_cta_n[k] * groups) * L.nj,
                                  h->st));
    }
    a.total_rows = R;
    a.max_cols_pad = rup(maxc, 4);
    h->f2grid = (h->sm_count / 2) * 2;
    h->gtf.clear();
    for (auto& L : h->blk) {
        GemvTDesc g{};
        g.A = L.A; g.lda = L.lda; g.rows = L.m; g.cols = L.nj;
        g.z = h->z + L.c0 * h->C; g.u = L.u; g.r = L.r; g.partial = L.partial2;
        g.nchunks = (int32_t)std::max<int64_t>(1, h->f2_cta_n[L.li] * groups); g.nstrips = 1; g.chunk_rows = 0;
        h->gtf.push_back(g);
    }
    return BICADMM_OK;
}

// ======================================================================= ABI: misc
extern "C" {

int bicadmm_version(void) { return BICADMM_ABI_VERSION; }

const char* bicadmm_rc_string(int rc) {
    switch (rc) {
    case BICADMM_OK: return "ok";
    case BICADMM_ERR_INVALID: return "invalid argument";
    case BICADMM_ERR_DIM: return "dimension mismatch";
    case BICADMM_ERR_DOMAIN: return "label outside the loss domain";
    case BICADMM_ERR_PLACEMENT: return "invalid block placement";
    case BICADMM_ERR_OOM: return "workspace too small";
    case BICADMM_ERR_CUDA: return "CUDA error";
    case BICADMM_ERR_NCCL: return "NCCL error";
    case BICADMM_ERR_STATE: return "invalid handle state";
    }
    return "unknown";
}

int64_t bicadmm_launch_count(void) { return g_launches.load(); }

int bicadmm_workspace_size(const bicadmm_problem* P, const bicadmm_params* R, size_t* bytes) {
    std::string why;
    if (!bytes) return BICADMM_ERR_INVALID;
    int rc = validate(P, R, &why);
    if (rc) return rc;
    bicadmm_handle tmp;
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&tmp.sm_count, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) tmp.sm_count = 148;
    tmp.C = P->C;
    tmp.prm = *R;
    *bytes = plan(&tmp, P, nullptr);
    return BICADMM_OK;
}

}  // extern "C"

// ======================================================================= collectives
// the handle runs the multi-rank path (NCCL collectives, no graphs)
static bool multi_rank(const bicadmm_handle* h) { return h->comm && (h->comm->world > 1 || h->comm->self); }

// In-place sum over the node group (group = true: Algorithm 2's per-sweep AllReduce)
// or over all ranks (the outer "Collect"); a no-op on a single rank.
static int allreduce(bicadmm_handle* h, double* buf, int64_t count, bool group) {
    if (!multi_rank(h) || count <= 0) return BICADMM_OK;
    if (group && h->gsize == 1 && !h->comm->self) return BICADMM_OK;
    std::string why;
    const int rc = comm_allreduce(h->comm, buf, count, group, h->st, &why);
    return rc ? fail(h, rc, why) : BICADMM_OK;
}
static int allreduce_many(bicadmm_handle* h, double* const* bufs, const int64_t* counts, int n, bool group) {
    if (!multi_rank(h) || n <= 0) return BICADMM_OK;
    if (group && h->gsize == 1 && !h->comm->self) return BICADMM_OK;
    std::string why;
    const int rc = comm_allreduce_many(h->comm, bufs, counts, n, group, h->st, &why);
    return rc ? fail(h, rc, why) : BICADMM_OK;
}

// Collective placement check (multi-rank setup; every rank of the world calls it): each
// (node, block) pair is held by exactly one rank, and the ranks of a node group together
// hold every block of each of their nodes -- otherwise the per-sweep AllReduce would sum
// the wrong blocks or NCCL would wait forever.  All ranks return the same code.
static int check_placement(bicadmm_handle* h) {
    const int64_t nm = (int64_t)h->N * h->M;
    std::vector<double> mask(2 * nm + 1, 0.0);
    for (auto& L : h->blk) mask[(size_t)L.node * h->M + L.block] = mask[(size_t)(nm + L.node * h->M + L.block)] = 1.0;
    H_CUDA(h, cudaMemcpyAsync(h->place_chk, mask.data(), sizeof(double) * 2 * nm, cudaMemcpyHostToDevice, h->st));
    H_RC(h, allreduce(h, h->place_chk, nm, false));        // over all ranks
    H_RC(h, allreduce(h, h->place_chk + nm, nm, true));    // over this rank's node group
    H_CUDA(h, cudaMemcpyAsync(mask.data(), h->place_chk, sizeof(double) * 2 * nm, cudaMemcpyDeviceToHost, h->st));
    H_CUDA(h, cudaStreamSynchronize(h->st));
    double bad = 0.0;
    for (int64_t k = 0; k < nm; ++k) bad += mask[(size_t)k] != 1.0;
    for (auto& nd : h->nod)
        for (int j = 0; j < h->M; ++j) bad += mask[(size_t)(nm + (int64_t)nd.node * h->M + j)] != 1.0;
    H_CUDA(h, cudaMemcpyAsync(h->place_chk + 2 * nm, &bad, sizeof(double), cudaMemcpyHostToDevice, h->st));
    H_RC(h, allreduce(h, h->place_chk + 2 * nm, 1, false));
    H_CUDA(h, cudaMemcpyAsync(&bad, h->place_chk + 2 * nm, sizeof(double), cudaMemcpyDeviceToHost, h->st));
    H_CUDA(h, cudaStreamSynchronize(h->st));
    return bad > 0.0 ? BICADMM_ERR_PLACEMENT : BICADMM_OK;
}

// ======================================================================= setup
// Small nodes (kind 5, auto schedule only): single rank, C == 1, every block tall and local, a
// node's blocks and factors fit one CTA's shared memory.  configs[0] (2 x 100 x 50): the whole
// inner loop is one launch instead of ~6 per sweep (the path is launch-bound there).
static bool build_small(bicadmm_handle* h) {
    static const bool on = [] { const char* e = getenv("BICADMM_SMALL"); return !(e && atoi(e) == 0); }();
    if (!on || h->comm || h->C != 1 || h->loss == BICADMM_SOFTMAX || h->split_blocks) return false;
    std::vector<SmallNode> v(h->nod.size());
    for (size_t li = 0; li < h->nod.size(); ++li) {
        const LNode& nd = h->nod[li];
        SmallNode& N = v[li];
        N = SmallNode{};
        N.b = nd.b; N.nu = nd.nu; N.delta = nd.delta; N.omega = nd.obar; N.m = nd.m;
        for (auto& L : h->blk) {
            if (L.li != (int)li) continue;
            if (L.fat || N.nb >= kSmallMaxBlocks) return false;
            SmallBlock& B = N.blk[N.nb++];
            B.A = L.A; B.lda = L.lda; B.nj = L.nj; B.c0 = L.c0; B.cs = N.ncols;
            B.H = L.H; B.ldh = L.ldh; B.hpack = L.hpack ? 1 : 0;
            B.x = L.x; B.r = L.r; B.p = L.p; B.u = L.u;
            N.ncols += L.nj;
        }
        small_sweep_plan(N);
        if (N.nb != h->M || N.ncols > kSmallMaxCols || small_sweep_smem_bytes(N) > kSmallSmemMax) return false;
    }
    h->small = v;
    return true;
}

extern "C" int bicadmm_setup(const bicadmm_problem* P, const bicadmm_params* R, bicadmm_comm* comm, void* ws,
                             size_t ws_bytes, void* stream, bicadmm_handle** out) {
    NvtxRange nvtx_range("bicadmm_setup");
    if (!out) return BICADMM_ERR_INVALID;
    *out = nullptr;
    std::string why;
    int rc = validate(P, R, &why);
    if (rc) return rc;
    bicadmm_handle* h = new bicadmm_handle();
    h->N = P->N; h->M = P->M; h->C = P->C; h->loss = P->loss; h->dtype = P->dtype;
    h->n = P->n; h->len = P->n * P->C;
    h->m.assign(P->m, P->m + P->N);
    h->col_start.assign(P->col_start, P->col_start + P->M + 1);
    h->prm = *R;
    h->comm = comm;
    h->st = (cudaStream_t)stream;
    h->launches0 = g_launches.load();
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, dev);
    h->gemv_cap = gemv_grid_cap(P->dtype, h->sm_count);
    const size_t need = plan(h, P, nullptr);
    if (!ws || ws_bytes < need) { delete h; return BICADMM_ERR_OOM; }
    if (((uintptr_t)ws) % 256) { delete h; return BICADMM_ERR_INVALID; }
    plan(h, P, ws);
    h->ws_bytes = ws_bytes;
    h->gsize = comm_group_size(comm);
    if (comm && comm->self) {
        // one-rank NCCL test mode; BICADMM_NCCL_SELF=2 also routes every node's block sum
        // through the per-sweep group AllReduce (the split-block path of block-major placements)
        for (auto& nd : h->nod) if (nd.np != P->M) { delete h; return BICADMM_ERR_PLACEMENT; }
        h->split_blocks = comm->self_mode >= 2;
    } else if (comm && comm->world > 1) {
        // a node whose M blocks are not all local has its block sum all-reduced per sweep
        for (auto& nd : h->nod) if (nd.np != P->M) h->split_blocks = true;
        if (h->split_blocks && h->gsize < 2) { delete h; return BICADMM_ERR_PLACEMENT; }
    } else {
        for (auto& nd : h->nod) if (nd.np != P->M) { delete h; return BICADMM_ERR_PLACEMENT; }
        if ((int)h->nod.size() != P->N) { delete h; return BICADMM_ERR_PLACEMENT; }
    }
    if (multi_rank(h) && !comm->self) {
        const int rc2 = check_placement(h);
        if (rc2) { delete h; return rc2; }
    }
    build_descs(h);
    {   // inner-sweep schedule (bicadmm_params.sweep)
        const bool ok4 = fused4_eligible(h);
        int kind = 0;
        if (R->sweep == 2) {
            if (!ok4) { delete h; return BICADMM_ERR_INVALID; }
            kind = 4;
        } else if (R->sweep == 0) {
            // auto: the CTA-pair single-pass sweep (k_fused4) where eligible and the rows are at
            // least 5.5 KB; narrower rows leave it bound by its per-batch chain.  Measured on B200
            // (round 2, row batches; 4 nodes x 60M / n rows, sweeps/s single vs two passes,
            // tools/crossover.sh): FP64 n = 500 859 vs 971, n = 800 1,270 vs 1,201, n = 2000
            // 2,410 vs 1,277; FP32 n = 1000 1,524 vs 1,604, n = 1400 1,882 vs 1,757, n = 3000
            // 2,844 vs 1,888.  (Round 1, one row per batch: the crossover was 14 KB.)
            int64_t maxc = 0;
            for (auto& L : h->blk) maxc = std::max(maxc, L.nj);
            const int64_t row_bytes = maxc * (P->dtype == BICADMM_F64 ? 8 : 4);
            kind = ok4 && row_bytes >= 5632 ? 4 : 0;
        }
        if (kind == 0 && R->sweep == 0 && build_small(h)) kind = 5;
        h->fused_kind = kind;
        h->fused = kind == 4;
        if (kind == 4 && build_fused4(h) != BICADMM_OK) { delete h; return BICADMM_ERR_CUDA; }
    }
    if (cudaMallocHost(&h->host_sc, sizeof(OuterScalars)) != cudaSuccess ||
        cudaMallocHost(&h->host_i64, sizeof(int64_t) * 4) != cudaSuccess) {
        bicadmm_destroy(h);
        return BICADMM_ERR_CUDA;
    }
    cudaEventCreate(&h->e0);
    cudaEventCreate(&h->e1);
    // zero all state (DESIGN R10)
    const int C = h->C;
    const int64_t len = h->len;
    const int nl = (int)h->nod.size();
    auto zero = [&](void* p, size_t bytes) { return cudaMemsetAsync(p, 0, bytes, h->st); };
    if (zero(h->x_all, sizeof(double) * h->lenp * nl) || zero(h->u_all, sizeof(double) * h->lenp * nl) ||
        zero(h->z, sizeof(double) * len) || zero(h->z_prev, sizeof(double) * len) ||
        zero(h->s, sizeof(double) * len) || zero(h->wbar, sizeof(double) * len) ||
        zero(h->x_final, sizeof(double) * len) || zero(h->sc, sizeof(OuterScalars))) {
        int r2 = fail(h, BICADMM_ERR_CUDA, "memset");
        bicadmm_destroy(h);
        return r2;
    }
    for (auto& nd : h->nod) {
        if (zero(nd.nu, sizeof(double) * nd.m * C) || zero(nd.delta, sizeof(double) * nd.m * C) ||
            zero(nd.p_base, sizeof(double) * nd.m * C * nd.np) || zero(nd.S, sizeof(double) * nd.m * C) ||
            zero(nd.obar, sizeof(double) * nd.m * C)) {
            bicadmm_destroy(h);
            return BICADMM_ERR_CUDA;
        }
    }
    // label domain (BICADMM_ERR_DOMAIN): one pass over every local node's labels; the flag
    // is read back with setup's final synchronisation
    // (launched per node right after its first block's ready event, below)
    if (zero(h->label_bad, sizeof(int))) { bicadmm_destroy(h); return BICADMM_ERR_CUDA; }
    // one-time block factors (a0)
    cudaEventRecord(h->e0, h->st);
    const double c = R->lambda / (double)P->N + R->rho_c;   // 1/(N gamma) + rho_c
    for (size_t b0 = 0; b0 < h->blk.size(); b0 += h->fbatch) {
        const int nb = (int)std::min<size_t>(h->fbatch, h->blk.size() - b0);
        std::vector<FactorJob> jobs;
        for (int k = 0; k < nb && !rc; ++k) {
            LBlock& L = h->blk[b0 + k];
            const int64_t ldg = rup(L.kd, 8);
            double* G = h->gram + k * h->gram_stride;
            if (L.ready && cudaStreamWaitEvent(h->st, (cudaEvent_t)L.ready, 0) != cudaSuccess) {
                rc = BICADMM_ERR_CUDA;
                break;
            }
            if (L.jl == 0 && launch_check_labels(P->dtype, P->loss, P->C, L.m, h->nod[L.li].b, h->label_bad, h->st)) {
                rc = BICADMM_ERR_CUDA;
                break;
            }
            if (L.fat)   // K = (c/rho_l) I + A A^T  (Woodbury, R27)
                rc = launch_gram_rows(P->dtype, L.m, L.nj, L.A, L.lda, 1.0, c / R->rho_l, G, ldg, h->st);
            else if (h->gtc_ws)   // F = rho_l A^T A + c I  (Eq. (24)), tcgen05 Ozaki-scheme Gram
                rc = launch_gram_tc(P->dtype, L.m, L.nj, L.A, L.lda, R->rho_l, c, G, ldg, h->gtc_ws, h->gtc_bytes, h->st);
            else         // F = rho_l A^T A + c I  (Eq. (24)), FP64 DMMA Gram
                rc = launch_gram(P->dtype, L.m, L.nj, L.A, L.lda, R->rho_l, c, G, ldg, false, h->st);
            // packed H: the full FP64 inverse goes into the (consumed) Gram scratch, then packed
            jobs.push_back(FactorJob{L.kd, G, ldg, L.hpack ? (void*)G : L.H, L.hpack ? ldg : L.ldh,
                                     L.hpack ? (int)BICADMM_F64 : P->dtype, h->fws + k * h->fws_stride});
        }
        if (!rc) rc = factor_inverse_batched(jobs.data(), (int)jobs.size(), h->st, h->gtc_ws, h->gtc_bytes);
        for (int k = 0; k < nb && !rc; ++k) {
            LBlock& L = h->blk[b0 + k];
            if (L.hpack) rc = launch_symv_pack(P->dtype, L.kd, h->gram + k * h->gram_stride, rup(L.kd, 8), L.H, h->st);
        }
        if (rc) {
            std::string msg = rc == BICADMM_ERR_CUDA ? std::string("factor: ") + cudaGetErrorString(cudaGetLastError())
                                                     : std::string("factor: matrix not positive definite");
            fail(h, rc, msg);
            fprintf(stderr, "bicadmm_setup: %s\n", msg.c_str());
            bicadmm_destroy(h);
            return rc;
        }
    }
    for (auto& L : h->blk) L.ready = nullptr;   // not retained (bicadmm_block.ready_event)
    cudaEventRecord(h->e1, h->st);
    if (cudaMemcpyAsync(h->host_i32, h->label_bad, sizeof(int), cudaMemcpyDeviceToHost, h->st) != cudaSuccess ||
        cudaStreamSynchronize(h->st) != cudaSuccess) {
        bicadmm_destroy(h);
        return BICADMM_ERR_CUDA;
    }
    if (h->host_i32[0]) { bicadmm_destroy(h); return BICADMM_ERR_DOMAIN; }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->e0, h->e1);
    h->ms_setup = ms;
    *out = h;
    return BICADMM_OK;
}

// ======================================================================= iterate
// A batch of GEMV descriptors plus packed-symmetric H-applies (k_symv.cu), one phase.
struct GemvList {
    std::vector<GemvDesc> g;
    std::vector<SymvDesc> s;
    void gemv(const GemvDesc& d) { g.push_back(d); }
    void happly(const LBlock& L, const double* x, double* y, double alpha) {   // y = alpha H x
        if (L.hpack) {
            SymvDesc d{};
            d.H = L.H; d.n = L.kd; d.x = x; d.y = y; d.alpha = alpha; d.part = L.hpart;
            s.push_back(d);
        } else {
            GemvDesc d{L.H, L.ldh, L.kd, L.kd, x, y, 0, L.xt};
            d.alpha = alpha;
            g.push_back(d);
        }
    }
    int launch(bicadmm_handle* h) const;
};

int GemvList::launch(bicadmm_handle* h) const {
    if (!g.empty()) H_RC(h, launch_gemv(h->dtype, const_cast<GemvDesc*>(g.data()), (int)g.size(), h->gemv_cap, h->st, h->C));
    if (!s.empty()) H_RC(h, launch_symv_packed(h->dtype, s.data(), (int)s.size(), h->st));
    return BICADMM_OK;
}

static int inner_sweep_fused(bicadmm_handle* h, const std::vector<int>& active_nodes, bool tol) {
    std::vector<GemvTDesc> gt;
    GemvList hx;
    std::vector<char> act(h->nod.size(), 0);
    for (int li : active_nodes) act[li] = 1;
    for (size_t k = 0; k < h->blk.size(); ++k) {
        const LBlock& L = h->blk[k];
        if (!act[L.li]) continue;
        gt.push_back(h->gtf[k]);
        hx.happly(L, L.r, L.x, 1.0);
    }
    cudaEvent_t ev[4] = {};
    int64_t lc[4] = {};
    auto mark = [&](int k) {
        if (!h->prof) return;
        ev[k] = next_event(h);
        rec_event(h, ev[k]);
        lc[k] = g_launches.load();
    };
    mark(0);   // r = rho_l sum_chunks partial + rho_c (z - u)   (partials from the previous fused pass)
    H_RC(h, launch_gemv_t_reduce(gt.data(), (int)gt.size(), h->prm.rho_l, h->prm.rho_c, h->st, h->C));
    mark(1);
    if (tol)
        H_CUDA(h, cudaMemcpyAsync(h->x_old, h->x_all, sizeof(double) * h->lenp * h->nod.size(),
                                  cudaMemcpyDeviceToDevice, h->st));
    H_RC(h, hx.launch(h));
    mark(2);
    {
        Fused2Args a = h->f2;
        for (size_t li = 0; li < h->nod.size(); ++li) {
            a.active[li] = act[li];
            a.e2row[li] = tol ? h->nod[li].S : nullptr;   // S is unused on the single-rank fused path
        }
        H_RC(h, launch_fused4(h->dtype, a, h->loss, h->prm.rho_l, h->f2grid, h->st));
    }
    mark(3);
    if (h->prof) {
        h->pending.push_back({1, ev[0], ev[1], lc[1] - lc[0]});
        h->pending.push_back({2, ev[1], ev[2], lc[2] - lc[1]});
        h->pending.push_back({7, ev[2], ev[3], lc[3] - lc[2]});
    }
    return BICADMM_OK;
}

static int inner_sweep(bicadmm_handle* h, const std::vector<int>& active_nodes, bool tol = false) {
    if (h->fused) return inner_sweep_fused(h, active_nodes, tol);
    // descriptors for the active nodes' blocks
    std::vector<GemvTDesc> gt;
    GemvList hx, ax;
    std::vector<FatEw> fq, fc;   // Woodbury blocks: q = p + delta; p = q + t1 + w0, qd = q - p
    std::vector<ProxNode> px;
    std::vector<char> act(h->nod.size(), 0);
    for (int li : active_nodes) act[li] = 1;
    for (size_t k = 0; k < h->blk.size(); ++k) {
        const LBlock& L = h->blk[k];
        if (!act[L.li]) continue;
        if (L.fat) {
            // Woodbury sweep entirely in m-space (R27):
            //   p = (1/rho_l) K^{-1} A r = q - (c/rho_l) K^{-1} q + w0,  w0 = (rho_c/rho_l) K^{-1} A (z - u)
            const double cc = h->prm.lambda / (double)h->N + h->prm.rho_c;
            const int64_t mc = L.m * h->C;
            fq.push_back(FatEw{L.p, h->nod[L.li].delta, nullptr, L.qd, nullptr, mc});
            hx.happly(L, L.qd, L.t1, -cc / h->prm.rho_l);
            fc.push_back(FatEw{L.qd, L.t1, L.w0, L.p, L.qd, mc});
            continue;
        }
        gt.push_back(h->gt[k]);
        hx.happly(L, L.r, L.x, 1.0);
        ax.gemv(GemvDesc{L.A, L.lda, L.m, L.nj, L.x, L.p, 0, L.xt});
    }
    for (int li : active_nodes) {
        const LNode& nd = h->nod[li];
        ProxNode p{};
        p.b = nd.b; p.p = nd.p_base; p.S = h->split_blocks ? nd.S : nullptr; p.nu = nd.nu; p.delta = nd.delta;
        p.omega = nd.obar; p.sq_partial = tol ? nd.sq_partial : nullptr; p.m = nd.m; p.pstride = nd.m * h->C;
        p.np = nd.np;
        px.push_back(p);
    }
    cudaEvent_t ev[7] = {};
    int64_t l0 = g_launches.load(), lc[7] = {};
    auto mark = [&](int k) {
        if (!h->prof) return;
        ev[k] = next_event(h);
        rec_event(h, ev[k]);
        lc[k] = g_launches.load();
    };
    mark(0);
    cudaEvent_t mid = h->prof ? next_event(h) : nullptr;
    if (!gt.empty())
        H_RC(h, launch_gemv_t(h->dtype, gt.data(), (int)gt.size(), h->prm.rho_l, h->prm.rho_c, h->st, mid, h->C));
    else if (mid)
        record_event(mid, h->st);
    const int64_t l_partial = (int64_t)(gt.size() + kMaxDesc - 1) / kMaxDesc;
    mark(2);
    if (tol)   // keep x^k for the ||x^{k+1} - x^k|| criterion
        H_CUDA(h, cudaMemcpyAsync(h->x_old, h->x_all, sizeof(double) * h->lenp * h->nod.size(),
                                  cudaMemcpyDeviceToDevice, h->st));
    if (!fq.empty()) H_RC(h, launch_fat_ew(fq.data(), (int)fq.size(), 0, h->st));
    H_RC(h, hx.launch(h));
    mark(3);
    H_RC(h, ax.launch(h));
    if (!fc.empty()) H_RC(h, launch_fat_ew(fc.data(), (int)fc.size(), 1, h->st));
    mark(4);
    if (h->split_blocks) {
        H_RC(h, launch_psum(h->C, px.data(), (int)px.size(), nullptr, h->st));
        // Algorithm 2's AllReduce: every local node's S_i in one collective (they are
        // contiguous); with a subset of nodes active (tolerance mode) one grouped call
        if (active_nodes.size() == h->nod.size()) {
            H_RC(h, allreduce(h, h->S_all, h->S_total, true));
        } else {
            std::vector<double*> bufs;
            std::vector<int64_t> cnts;
            for (int li : active_nodes) { bufs.push_back(h->nod[li].S); cnts.push_back(h->nod[li].m * h->C); }
            H_RC(h, allreduce_many(h, bufs.data(), cnts.data(), (int)bufs.size(), true));
        }
    }
    mark(5);
    H_RC(h, launch_prox(h->loss, h->dtype, h->C, h->M, h->prm.rho_l, px.data(), (int)px.size(), h->st));
    mark(6);
    if (h->prof) {
        h->pending.push_back({0, ev[0], mid, l_partial});
        h->pending.push_back({1, mid, ev[2], lc[2] - l0 - l_partial});
        h->pending.push_back({2, ev[2], ev[3], lc[3] - lc[2]});
        h->pending.push_back({3, ev[3], ev[4], lc[4] - lc[3]});
        h->pending.push_back({4, ev[4], ev[5], lc[5] - lc[4]});
        h->pending.push_back({5, ev[5], ev[6], lc[6] - lc[5]});
    }
    return BICADMM_OK;
}

// Fat blocks (Woodbury, R27) carry p_ij = A_ij x_ij exactly through the sweep
// without forming x_ij; x_ij = (r - rho_l A^T p_ij) / c = (rho_l A^T (q - p) + rho_c (z - u)) / c
// is materialized only where it is read: before the outer step (Collect, Eq. (7)) and per
// sweep in tolerance mode.  fat_prepare computes the per-inner-loop constant
// w0 = (rho_c/rho_l) K^{-1} A (z - u) (z and u are fixed during an inner loop).
static int fat_prepare(bicadmm_handle* h, const std::vector<int>& nodes) {
    std::vector<char> act(h->nod.size(), 0);
    for (int li : nodes) act[li] = 1;
    std::vector<FatEw> zu;
    std::vector<GemvDesc> aw;
    GemvList kw;
    for (auto& L : h->blk) {
        if (!L.fat || !act[L.li]) continue;
        zu.push_back(FatEw{h->z + L.c0 * h->C, L.u, nullptr, L.zu, nullptr, L.nj * h->C});
        aw.push_back(GemvDesc{L.A, L.lda, L.m, L.nj, L.zu, L.t1, 0, L.xt});
        kw.happly(L, L.t1, L.w0, h->prm.rho_c / h->prm.rho_l);
    }
    if (zu.empty()) return BICADMM_OK;
    H_RC(h, launch_fat_ew(zu.data(), (int)zu.size(), 2, h->st));
    H_RC(h, launch_gemv(h->dtype, aw.data(), (int)aw.size(), h->gemv_cap, h->st, h->C));
    H_RC(h, kw.launch(h));
    return BICADMM_OK;
}

static int materialize_x(bicadmm_handle* h, const std::vector<int>& nodes) {
    std::vector<char> act(h->nod.size(), 0);
    for (int li : nodes) act[li] = 1;
    std::vector<GemvTDesc> gt;
    for (size_t k = 0; k < h->blk.size(); ++k) {
        const LBlock& L = h->blk[k];
        if (!L.fat || !act[L.li]) continue;
        GemvTDesc g = h->gt[k];   // x = (rho_l A^T (q - p) + rho_c (z - u)) / c
        g.p = L.qd; g.delta = nullptr; g.r = L.x;
        gt.push_back(g);
    }
    if (gt.empty()) return BICADMM_OK;
    cudaEvent_t a = nullptr, b = nullptr;
    const int64_t l0 = g_launches.load();
    if (h->prof) { a = next_event(h); rec_event(h, a); }
    const double c = h->prm.lambda / (double)h->N + h->prm.rho_c;
    H_RC(h, launch_gemv_t(h->dtype, gt.data(), (int)gt.size(), h->prm.rho_l / c, h->prm.rho_c / c, h->st, nullptr, h->C));
    if (h->prof) {
        b = next_event(h);
        rec_event(h, b);
        h->pending.push_back({0, a, b, g_launches.load() - l0});
    }
    return BICADMM_OK;
}

static int outer_step(bicadmm_handle* h, bool readback = true) {
    const double rho_b = h->prm.alpha * h->prm.rho_c;
    cudaEvent_t oa = nullptr, ob = nullptr;
    const int64_t lo0 = g_launches.load();
    if (h->prof) { oa = next_event(h); rec_event(h, oa); }
    const double sqrtN_rho_c = std::sqrt((double)h->N) * h->prm.rho_c;
    // single rank, short vectors: Collect runs inside k_zt and the residuals inside k_node_sq
    // (same arithmetic, same order; two launches fewer per outer iteration)
    const bool fuse = !multi_rank(h) && h->len * (int64_t)h->nod.size() <= (int64_t)1 << 16;
    WsumIn cw;
    if (fuse) {
        cw.x_all = h->x_all; cw.u_all = h->u_all; cw.stride = h->lenp; cw.nl = (int)h->nod.size();
    } else {
        H_RC(h, launch_wsum(h->len, h->lenp, h->x_all, h->u_all, (int)h->nod.size(), h->wsum, h->st));
        H_RC(h, allreduce(h, h->wsum, h->len, false));
    }
    H_RC(h, launch_zt(h->len, h->N, h->prm.rho_c, rho_b, h->wsum, h->s, h->wbar, h->z, h->z_prev, h->sc, h->st, cw));
    H_RC(h, launch_s_update(h->len, h->prm.kappa, h->z, h->s, h->sc, h->st));
    H_RC(h, launch_u_update(h->bv.data(), (int)h->bv.size(), h->z, h->upart, h->st));
    H_RC(h, launch_node_sq(h->bv.data(), (int)h->bv.size(), h->upart, h->N, h->node_sq, h->st,
                           multi_rank(h) ? nullptr : h->sc, sqrtN_rho_c));
    if (multi_rank(h)) {
        // every (i, j) contributes exactly once: node_sq partials are per local block
        H_RC(h, allreduce(h, h->node_sq, h->N, false));
        H_RC(h, launch_residuals(h->N, sqrtN_rho_c, h->node_sq, h->sc, h->st));
    }
    if (h->prof) {
        ob = next_event(h);
        rec_event(h, ob);
        h->pending.push_back({6, oa, ob, g_launches.load() - lo0});
    }
    if (readback) H_CUDA(h, cudaMemcpyAsync(h->host_sc, h->sc, sizeof(OuterScalars), cudaMemcpyDeviceToHost, h->st));
    return BICADMM_OK;
}

// after outer_step's work (eager or graph replay): wait for the 6 scalars
static int outer_finish(bicadmm_handle* h) {
    H_CUDA(h, cudaStreamSynchronize(h->st));
    if (h->prof) resolve_phases(h);
    return BICADMM_OK;
}

// Per-node inner criteria after a tol-mode sweep: res[i] = ||abar_i - obar_i||^2,
// dx[i] = ||x_i^new - x_i^old||^2 (both FP64, fixed-order sums; dx all-reduced over
// the node group when a node's blocks span ranks).
static int inner_criteria(bicadmm_handle* h, const std::vector<int>& active, std::vector<double>& res,
                          std::vector<double>& dx) {
    std::vector<BlockVec> bv;
    for (auto& L : h->blk) {
        bool on = false;
        for (int li : active) on |= li == L.li;
        if (!on) continue;
        BlockVec v{};
        v.x = L.x; v.u = h->x_old + (L.x - h->x_all); v.c0 = 0; v.len = L.nj * h->C; v.node = L.node;
        bv.push_back(v);
    }
    H_CUDA(h, cudaMemsetAsync(h->node_dx, 0, sizeof(double) * h->N, h->st));
    H_RC(h, launch_u_update(bv.data(), (int)bv.size(), nullptr, h->dpart, h->st, 1));
    H_RC(h, launch_node_sq(bv.data(), (int)bv.size(), h->dpart, h->N, h->node_dx, h->st));
    if (h->split_blocks) H_RC(h, allreduce(h, h->node_dx, h->N, true));
    std::vector<const double*> ptr;
    std::vector<int64_t> cnt;
    std::vector<int32_t> node;
    for (int li : active) {
        ptr.push_back(h->nod[li].sq_partial);
        cnt.push_back(h->nod[li].nprox_ctas);
        node.push_back(h->nod[li].node);
    }
    if (h->fused) {   // the single-pass kernel leaves (abar - omega)^2 per row in S
        for (int li : active) H_RC(h, launch_sum(h->nod[li].m, h->nod[li].S, h->node_res + h->nod[li].node, h->st));
    } else {
        H_RC(h, launch_seg_sums(ptr.data(), cnt.data(), node.data(), (int)ptr.size(), h->node_res, h->st));
    }
    res.assign(h->N, 0.0);
    dx.assign(h->N, 0.0);
    H_CUDA(h, cudaMemcpyAsync(res.data(), h->node_res, sizeof(double) * h->N, cudaMemcpyDeviceToHost, h->st));
    H_CUDA(h, cudaMemcpyAsync(dx.data(), h->node_dx, sizeof(double) * h->N, cudaMemcpyDeviceToHost, h->st));
    H_CUDA(h, cudaStreamSynchronize(h->st));
    return BICADMM_OK;
}

// One outer iteration with a fixed per-node sweep count: Woodbury preparation, the
// sweeps, x materialization (enqueue only; outer_step follows).
static int enqueue_fixed(bicadmm_handle* h, const std::vector<int>& want, int maxs) {
    std::vector<int> swept;
    for (size_t li = 0; li < h->nod.size(); ++li) if (want[li] > 0) swept.push_back((int)li);
    if (h->any_fat) H_RC(h, fat_prepare(h, swept));
    if (!h->small.empty() && maxs > 0 && (int)swept.size() == (int)h->nod.size() &&
        std::all_of(want.begin(), want.end(), [&](int w) { return w == maxs; })) {
        // every node the same K sweeps: the whole inner loop in one launch (kind 5)
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        const int64_t l0 = g_launches.load();
        if (h->prof) { e0 = next_event(h); rec_event(h, e0); }
        H_RC(h, launch_small_sweeps(h->loss, h->dtype, h->small.data(), (int)h->small.size(), h->z, maxs, h->M,
                                    h->prm.rho_l, h->prm.rho_c, h->st));
        if (h->prof) {
            e1 = next_event(h);
            rec_event(h, e1);
            h->pending.push_back({7, e0, e1, g_launches.load() - l0});
        }
        return BICADMM_OK;
    }
    for (int sw = 0; sw < maxs; ++sw) {
        std::vector<int> active;
        for (size_t li = 0; li < h->nod.size(); ++li) if (want[li] > sw) active.push_back((int)li);
        H_RC(h, inner_sweep(h, active));
    }
    if (h->any_fat) H_RC(h, materialize_x(h, swept));
    return BICADMM_OK;
}

static bool graph_nccl_enabled() {   // BICADMM_GRAPH_NCCL=0: multi-rank runs stay eager
    static const bool on = [] { const char* e = getenv("BICADMM_GRAPH_NCCL"); return !(e && atoi(e) == 0); }();
    return on;
}
static bool graph_enabled() {   // BICADMM_GRAPH=0: eager launches (read per outer iteration)
    const char* e = getenv("BICADMM_GRAPH");
    return !(e && atoi(e) == 0);
}

// Capture (once per sweep count / profiling state) and replay one outer iteration as a
// CUDA graph: K_in sweeps + the global step + the 96-byte D2H read of the scalars, one
// cudaGraphLaunch instead of ~5 K_in + 8 launches.  Returns BICADMM_ERR_STATE if the
// capture is refused (the caller then runs the same work eagerly).
static int graph_outer(bicadmm_handle* h, const std::vector<int>& want, int maxs) {
    auto& G = h->graph;
    if (!G.exec || G.prof != h->prof || G.sweeps != maxs) {
        if (G.exec) { cudaGraphExecDestroy(G.exec); G.exec = nullptr; }
        h->pending.clear();
        h->evused = 0;
        const int64_t l0 = g_launches.load();
        if (!h->cap_st && cudaStreamCreateWithFlags(&h->cap_st, cudaStreamNonBlocking) != cudaSuccess) {
            cudaGetLastError();
            G.failed = true;
            return BICADMM_ERR_STATE;
        }
        cudaStream_t st0 = h->st;
        h->st = h->cap_st;   // the graph is captured on the private stream, launched on the caller's
        if (cudaStreamBeginCapture(h->st, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
            h->st = st0;
            cudaGetLastError();
            G.failed = true;
            return BICADMM_ERR_STATE;
        }
        h->capturing = true;
        int rc = enqueue_fixed(h, want, maxs);
        if (!rc) rc = outer_step(h);
        cudaGraph_t graph = nullptr;
        const cudaError_t e = cudaStreamEndCapture(h->st, &graph);
        h->capturing = false;
        h->st = st0;
        cudaGraphExec_t exec = nullptr;
        if (!rc && e == cudaSuccess && graph && cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess) {
            G.exec = exec;
        }
        if (graph) cudaGraphDestroy(graph);
        const int64_t captured = g_launches.load() - l0;
        g_launches.fetch_sub(captured);   // counted again at every replay
        if (!G.exec) {   // refused: forget the capture and run eagerly from now on
            if (getenv("BICADMM_GRAPH_DEBUG")) fprintf(stderr, "bicadmm: graph capture refused (rc %d, %s)\n", rc, cudaGetErrorString(e));
            cudaGetLastError();
            h->dead = false;
            h->err.clear();
            h->pending.clear();
            h->evused = 0;
            G.failed = true;
            return BICADMM_ERR_STATE;
        }
        if (getenv("BICADMM_GRAPH_DEBUG")) fprintf(stderr, "bicadmm: captured outer-iteration graph (%lld launches)\n", (long long)captured);
        G.launches = captured;
        G.pending = h->pending;
        h->pending.clear();
        G.prof = h->prof;
        G.sweeps = maxs;
    }
    H_CUDA(h, cudaGraphLaunch(G.exec, h->st));
    g_launches.fetch_add(G.launches);
    if (h->prof) h->pending = G.pending;
    return BICADMM_OK;
}

static int sweeps_for(bicadmm_handle* h, int k, int li) {
    if (!h->schedule.empty()) {
        const int row = k - h->sched_start;
        if (row >= 0 && row < h->sched_rows) return h->schedule[(size_t)row * h->N + h->nod[li].node];
    }
    return h->prm.inner_fixed > 0 ? h->prm.inner_fixed : h->prm.max_inner;
}

extern "C" int bicadmm_iterate(bicadmm_handle* h, int n_outer, bicadmm_step_info* info) {
    NvtxRange nvtx_range("bicadmm_iterate");
    if (!h) return BICADMM_ERR_INVALID;
    if (h->dead) return BICADMM_ERR_STATE;
    if (n_outer < 0) return fail(h, BICADMM_ERR_INVALID, "n_outer < 0");
    int sweeps_call = 0;
    for (int it = 0; it < n_outer; ++it) {
        const int k = h->outer_done;
        const int srow = k - h->sched_start;
        const bool replay = !h->schedule.empty() && srow >= 0 && srow < h->sched_rows;
        const bool tol = !replay && h->prm.inner_fixed == 0;
        std::vector<int> want(h->nod.size());
        int maxs = 0;
        int orc = BICADMM_OK;
        if (!tol) {
            bool uniform = true;
            for (size_t li = 0; li < h->nod.size(); ++li) {
                want[li] = sweeps_for(h, k, (int)li);
                maxs = std::max(maxs, want[li]);
                uniform = uniform && want[li] == want[0];
            }
            // from the second outer iteration on, a fixed uniform schedule replays one CUDA graph;
            // with NCCL its collectives are captured into it too (NCCL supports stream capture;
            // every rank captures the same sequence).  The emulated communicator meets at host
            // barriers, which a graph cannot hold: eager launches there.
            const bool use_graph = graph_enabled() && !replay && uniform && k >= 1 && !h->graph.failed &&
                                   !(h->comm && h->comm->emu) && (!multi_rank(h) || graph_nccl_enabled());
            static const bool gdbg = getenv("BICADMM_GRAPH_DEBUG") != nullptr;
            if (gdbg) fprintf(stderr, "bicadmm: outer %d use_graph %d (replay %d uniform %d failed %d)\n", k, (int)use_graph,
                              (int)replay, (int)uniform, (int)h->graph.failed);
            orc = use_graph ? graph_outer(h, want, maxs) : BICADMM_ERR_STATE;
            if (orc == BICADMM_ERR_STATE) {   // eager (or the capture was refused)
                orc = enqueue_fixed(h, want, maxs);
                if (!orc) orc = outer_step(h);
            }
        } else {
            // tolerance mode: sweep node i until ||abar - obar|| <= eps sqrt(m_i C) and
            // ||x_i^new - x_i^old|| <= eps, at most max_inner sweeps
            std::vector<int> active;
            for (size_t li = 0; li < h->nod.size(); ++li) active.push_back((int)li);
            std::vector<double> res, dx;
            if (h->any_fat) {
                int rc = fat_prepare(h, active);
                if (rc) return rc;
            }
            for (int sw = 0; sw < h->prm.max_inner && !active.empty(); ++sw) {
                int rc = inner_sweep(h, active, true);
                if (!rc && h->any_fat) rc = materialize_x(h, active);
                if (!rc) rc = inner_criteria(h, active, res, dx);
                if (rc) return rc;
                std::vector<int> still;
                for (int li : active) {
                    want[li] = sw + 1;
                    const int i = h->nod[li].node;
                    const bool done = std::sqrt(res[i]) <= h->prm.eps_inner * std::sqrt((double)(h->nod[li].m * h->C)) &&
                                      std::sqrt(dx[i]) <= h->prm.eps_inner;
                    if (!done) still.push_back(li);
                }
                active.swap(still);
                maxs = sw + 1;
            }
            orc = outer_step(h);
        }
        int rc = orc ? orc : outer_finish(h);
        if (rc) return rc;
        const OuterScalars& s = *h->host_sc;
        h->trace.push_back({s.p_r, s.d_r, s.b_r, s.t, s.v, s.tau});
        std::vector<int32_t> row(h->N, 0);
        for (size_t li = 0; li < h->nod.size(); ++li) row[h->nod[li].node] = want[li];
        h->inner_counts.insert(h->inner_counts.end(), row.begin(), row.end());
        h->outer_done++;
        h->inner_total += maxs;
        sweeps_call += maxs;
        h->converged = s.p_r <= h->prm.eps_p && s.d_r <= h->prm.eps_d && s.b_r <= h->prm.eps_b;
        h->finalized = false;
    }
    if (info) {
        info->outer_iters = h->outer_done;
        info->inner_sweeps = sweeps_call;
        const OuterScalars& s = *h->host_sc;
        info->p_r = s.p_r; info->d_r = s.d_r; info->b_r = s.b_r;
        info->t = s.t; info->v = s.v; info->tau = s.tau;
        info->converged = h->converged ? 1 : 0;
    }
    return BICADMM_OK;
}

// ======================================================================= finalize
__global__ void k_scatter_support(const double* __restrict__ z, const int64_t* __restrict__ sup,
                                  const int64_t* __restrict__ cnt, double* __restrict__ xf) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < *cnt) xf[sup[k]] = z[sup[k]];
}
__global__ void k_scale(int64_t n, double a, double* __restrict__ x) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) x[i] *= a;
}

__global__ void k_sum_partials(const double* __restrict__ parts, int64_t n, double* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int64_t k = 0; k < n; ++k) s += parts[k];
        *out = s;
    }
}
__global__ void k_sqnorm(int64_t len, const double* __restrict__ x, double* out) {
    __shared__ double scratch[32];
    double a = 0.0;
    for (int64_t l = threadIdx.x; l < len; l += blockDim.x) a += x[l] * x[l];
    a = block_sum(a, scratch);
    if (threadIdx.x == 0) *out = a;
}

// Support = top-kappa of |z| with z != 0 (ties to the lower index), x_final = z on
// the support (DESIGN R19), objective (1) at x_final (DESIGN R20).
// out = mask * (2 sum_i A_i^T (w_i) + lambda v), where w_i = sum_j A_ij v_j (use_v) or
// w_i = b_i (rhs mode, lambda term dropped).  Same GEMV / GEMV-T kernels as the sweep.
static int refit_apply(bicadmm_handle* h, const double* v, double* out, bool rhs_mode) {
    if (!rhs_mode) {
        std::vector<GemvDesc> ax;
        for (auto& L : h->blk) ax.push_back(GemvDesc{L.A, L.lda, L.m, L.nj, v + L.c0, L.pobj, 0});
        H_RC(h, launch_gemv(h->dtype, ax.data(), (int)ax.size(), h->gemv_cap, h->st, 1));
        for (auto& nd : h->nod) {
            ProxNode p{};
            p.p = nd.pobj_base; p.np = nd.np; p.pstride = nd.m; p.m = nd.m; p.S = nd.S;
            H_RC(h, launch_psum(1, &p, 1, nullptr, h->st));
        }
        if (h->split_blocks) H_RC(h, allreduce(h, h->S_all, h->S_total, true));   // C == 1 here
    } else {
        for (auto& nd : h->nod) H_RC(h, launch_to_f64(h->dtype, nd.m, nd.b, nd.S, h->st));
    }
    std::vector<GemvTDesc> gt;
    for (size_t k = 0; k < h->blk.size(); ++k) {
        GemvTDesc g = h->gt[k];
        g.p = h->nod[h->blk[k].li].S; g.delta = nullptr; g.z = nullptr; g.u = nullptr;
        gt.push_back(g);
    }
    H_RC(h, launch_gemv_t(h->dtype, gt.data(), (int)gt.size(), 2.0, 0.0, h->st, nullptr, 1));
    H_CUDA(h, cudaMemsetAsync(out, 0, sizeof(double) * h->len, h->st));
    for (auto& L : h->blk) H_RC(h, launch_axpy_into(L.nj, L.r, out + L.c0, h->st));
    H_RC(h, allreduce(h, out, h->len, false));
    H_RC(h, launch_ridge_mask(h->len, h->mask, rhs_mode ? out : v, rhs_mode ? 0.0 : h->prm.lambda, out, h->st));
    return BICADMM_OK;
}

// LS ridge refit on the support (DESIGN R19): CG on the SPD system restricted to T,
// warm-started at z|_T, to a relative residual of 1e-14.
static int do_refit(bicadmm_handle* h) {
    const int64_t len = h->len;
    const int64_t cap = std::max<int64_t>(1, std::min<int64_t>(h->prm.kappa, len));
    H_CUDA(h, cudaMemsetAsync(h->mask, 0, sizeof(double) * len, h->st));
    H_RC(h, launch_support_mask(cap, h->support, h->support_count, h->mask, h->st));
    H_RC(h, refit_apply(h, nullptr, h->cg_rhs, true));                    // rhs = 2 A_T^T b
    H_RC(h, refit_apply(h, h->x_final, h->cg_Ap, false));                 // A x0
    H_CUDA(h, cudaMemcpyAsync(h->cg_r, h->cg_rhs, sizeof(double) * len, cudaMemcpyDeviceToDevice, h->st));
    H_RC(h, launch_axpy_scaled(len, -1.0, h->cg_Ap, h->cg_r, h->st));    // r = rhs - A x0
    H_CUDA(h, cudaMemcpyAsync(h->cg_p, h->cg_r, sizeof(double) * len, cudaMemcpyDeviceToDevice, h->st));
    H_RC(h, launch_dot(len, h->cg_r, h->cg_r, h->cg_sc + 0, h->st));
    H_RC(h, launch_dot(len, h->cg_rhs, h->cg_rhs, h->cg_sc + 3, h->st));
    double hs[4] = {0, 0, 0, 0};
    H_CUDA(h, cudaMemcpyAsync(hs, h->cg_sc, sizeof(double) * 4, cudaMemcpyDeviceToHost, h->st));
    H_CUDA(h, cudaStreamSynchronize(h->st));
    const double tol2 = 1e-28 * hs[3];
    h->refit_iters = 0;
    if (hs[0] <= tol2) return BICADMM_OK;
    for (int it = 0; it < 500; ++it) {
        H_RC(h, refit_apply(h, h->cg_p, h->cg_Ap, false));
        H_RC(h, launch_dot(len, h->cg_p, h->cg_Ap, h->cg_sc + 1, h->st));
        H_RC(h, launch_cg_xr(len, h->cg_sc, h->cg_p, h->cg_Ap, h->x_final, h->cg_r, h->st));
        H_RC(h, launch_dot(len, h->cg_r, h->cg_r, h->cg_sc + 2, h->st));
        H_RC(h, launch_cg_p(len, h->cg_sc, h->cg_r, h->cg_p, h->st));
        H_CUDA(h, cudaMemcpyAsync(h->cg_sc, h->cg_sc + 2, sizeof(double), cudaMemcpyDeviceToDevice, h->st));
        H_CUDA(h, cudaMemcpyAsync(hs + 2, h->cg_sc + 2, sizeof(double), cudaMemcpyDeviceToHost, h->st));
        H_CUDA(h, cudaStreamSynchronize(h->st));
        h->refit_iters = it + 1;
        if (!(hs[2] > tol2)) break;
    }
    return BICADMM_OK;
}

// Logistic / softmax refit on the support T (DESIGN R29), the oracle's algorithm on the GPU:
// damped Newton from z on T with the exact k x k Hessian, Armijo backtracking on the objective
// while it can resolve the predicted decrease; the support columns of every local row are
// gathered once into AT (rows x kp, FP64).  Logistic: w = AT x, Hessian = Gram of the
// row-scaled AT (sqrt(s(1-s))) + lambda I.  Softmax (entries a = l*C + c, c_a = a % C):
// W = AT X with X[a][c] = x_a [c = c_a] (DMMA multi-class GEMV), gradient weights P - E_y,
// Hessian = [c_a = c_b] Gram(sqrt(P_{c_a}) AT) - Gram(P_{c_a} AT) + lambda I.  The k-vectors'
// scalar logic (step, stopping) runs on the host.
static int do_refit_newton(bicadmm_handle* h) {
    const int64_t kp = h->rf_kp, rows = h->rf_rows, len = h->len;
    const int C = h->C;
    const bool sm = h->loss == BICADMM_SOFTMAX;
    cudaStream_t st = h->st;
    // Multi-rank (DESIGN R29): a node's support columns are gathered on every rank that holds
    // some of its blocks and summed over the node group (the others are zero), so each rank
    // of a group holds the node's whole support matrix and computes the node's terms
    // identically; node sums (objective, gradient, Hessian) are then summed over all ranks and
    // divided by the group size gs (a node's terms are replicated gs times; gs is a power of
    // two in every placement built here, so the division is exact).  The ridge term enters
    // once: lambda / G_n per rank, G_n = world / gs node groups.  The Newton decisions are then
    // taken on identical bits on every rank.
    const bool mr = multi_rank(h);
    const double gs = (mr && h->split_blocks) ? (double)h->gsize : 1.0;
    const double gn = mr ? (double)h->comm->world / gs : 1.0;
    const double lam = h->prm.lambda;
    const double lam_part = lam / gn;
    auto node_sum = [&](double* buf, int64_t n) -> int {   // world sum / gs (no-op on one rank)
        if (!mr) return BICADMM_OK;
        H_RC(h, allreduce(h, buf, n, false));
        if (gs != 1.0) {
            k_scale<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1184), 256, 0, st>>>(n, 1.0 / gs, buf);
            BIC_LAUNCHED();
        }
        return BICADMM_OK;
    };
    H_CUDA(h, cudaMemsetAsync(h->rf_AT, 0, sizeof(double) * rows * kp, st));
    {
        int64_t off = 0;
        for (auto& nd : h->nod) {
            for (auto& L : h->blk)
                if (L.li == nd.li)
                    H_RC(h, launch_rf_gather(h->dtype, L.A, L.lda, L.m, L.c0, L.nj, h->support, h->support_count,
                                             h->rf_AT, kp, off, st, C));
            H_RC(h, launch_to_f64(h->dtype, nd.m, nd.b, h->rf_b + off, st));
            off += nd.m;
        }
        if (mr && h->split_blocks) H_RC(h, allreduce(h, h->rf_AT, rows * kp, true));   // the node's other blocks
    }
    int64_t cnt = 0;
    H_CUDA(h, cudaMemcpyAsync(&cnt, h->support_count, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    H_CUDA(h, cudaStreamSynchronize(st));
    if (cnt <= 0) return BICADMM_OK;
    std::vector<int64_t> sup(cnt);
    std::vector<double> zf(len), x(kp, 0.0), xn(kp, 0.0), g(kp), d(kp), Xh(sm ? kp * C : 0), Yh(sm ? kp * C : 0);
    H_CUDA(h, cudaMemcpyAsync(sup.data(), h->support, sizeof(int64_t) * cnt, cudaMemcpyDeviceToHost, st));
    H_CUDA(h, cudaMemcpyAsync(zf.data(), h->x_final, sizeof(double) * len, cudaMemcpyDeviceToHost, st));
    H_CUDA(h, cudaStreamSynchronize(st));
    for (int64_t a = 0; a < cnt; ++a) x[a] = zf[sup[a]];   // start: z on T
    std::vector<double> parts(h->rf_nparts);
    GemvDesc aw{h->rf_AT, kp, rows, kp, h->rf_x, h->rf_w, 0};
    GemvDesc awc{h->rf_AT, kp, rows, kp, h->rf_X, h->rf_W, 0, h->rf_xt};
    // f(v): leaves w = AT v (logistic) or W = AT X(v) (softmax) on the device
    auto objective = [&](const std::vector<double>& v, double& f) -> int {
        if (sm) {
            std::fill(Xh.begin(), Xh.end(), 0.0);
            for (int64_t a = 0; a < cnt; ++a) Xh[a * C + sup[a] % C] = v[a];
            H_CUDA(h, cudaMemcpyAsync(h->rf_X, Xh.data(), sizeof(double) * kp * C, cudaMemcpyHostToDevice, st));
            H_RC(h, launch_gemv(BICADMM_F64, &awc, 1, h->gemv_cap, st, C));
            H_RC(h, launch_rf_sm_rows(rows, C, h->rf_b, h->rf_W, nullptr, nullptr, h->rf_obj, st));
        } else {
            H_CUDA(h, cudaMemcpyAsync(h->rf_x, v.data(), sizeof(double) * kp, cudaMemcpyHostToDevice, st));
            H_RC(h, launch_gemv(BICADMM_F64, &aw, 1, h->gemv_cap, st, 1));
            H_RC(h, launch_rf_logit(rows, h->rf_b, h->rf_w, nullptr, nullptr, h->rf_obj, st));
        }
        H_CUDA(h, cudaMemcpyAsync(parts.data(), h->rf_obj, sizeof(double) * parts.size(), cudaMemcpyDeviceToHost, st));
        H_CUDA(h, cudaStreamSynchronize(st));
        double sum = 0.0, xx = 0.0;
        for (double p : parts) sum += p;
        if (mr) {   // the data term summed over the ranks' nodes (the partial counts differ by rank)
            H_CUDA(h, cudaMemcpyAsync(h->rf_d, &sum, sizeof(double), cudaMemcpyHostToDevice, st));
            H_RC(h, node_sum(h->rf_d, 1));
            H_CUDA(h, cudaMemcpyAsync(&sum, h->rf_d, sizeof(double), cudaMemcpyDeviceToHost, st));
            H_CUDA(h, cudaStreamSynchronize(st));
        }
        for (int64_t a = 0; a < kp; ++a) xx += v[a] * v[a];
        f = sum + 0.5 * lam * xx;
        return BICADMM_OK;
    };
    double f = 0.0;
    H_RC(h, objective(x, f));
    const int64_t ldf = rup(kp, 8);
    h->rf_newton = 0;
    for (int it = 0; it < 100; ++it) {
        GemvTDesc gt = h->rf_gt;
        gt.A = h->rf_AT; gt.lda = kp; gt.delta = nullptr; gt.z = nullptr; gt.u = nullptr; gt.partial = h->rf_part;
        if (sm) {
            H_RC(h, launch_rf_sm_rows(rows, C, h->rf_b, h->rf_W, h->rf_G, h->rf_P, h->rf_obj, st));
            gt.p = h->rf_G; gt.r = h->rf_Y;
            H_RC(h, launch_gemv_t(BICADMM_F64, &gt, 1, 1.0, 0.0, st, nullptr, C));   // Y = AT^T (P - E_y)
            H_RC(h, launch_rf_sm_scale(rows, kp, C, h->rf_AT, h->rf_P, h->support, h->support_count, h->rf_BT, h->rf_U, st));
            H_RC(h, launch_gram(BICADMM_F64, rows, kp, h->rf_BT, kp, 1.0, lam_part, h->rf_F, ldf, false, st));
            H_RC(h, launch_gram(BICADMM_F64, rows, kp, h->rf_U, kp, 1.0, 0.0, h->rf_F2, ldf, false, st));
            H_RC(h, launch_rf_sm_combine(kp, ldf, C, h->support, h->support_count, h->rf_F, h->rf_F2, st));
            H_RC(h, node_sum(h->rf_Y, kp * C));
            H_RC(h, node_sum(h->rf_F, ldf * kp));
        } else {
            H_RC(h, launch_rf_logit(rows, h->rf_b, h->rf_w, h->rf_psi, h->rf_sd, h->rf_obj, st));
            gt.p = h->rf_psi; gt.r = h->rf_g;
            H_RC(h, launch_gemv_t(BICADMM_F64, &gt, 1, 1.0, 0.0, st, nullptr, 1));    // AT^T psi
            H_RC(h, launch_rf_scale_rows(rows, kp, h->rf_AT, h->rf_sd, h->rf_BT, st));
            H_RC(h, launch_gram(BICADMM_F64, rows, kp, h->rf_BT, kp, 1.0, lam_part, h->rf_F, ldf, false, st));
            H_RC(h, node_sum(h->rf_g, kp));
            H_RC(h, node_sum(h->rf_F, ldf * kp));
        }
        // (padding columns >= |T| are zero in AT: their Hessian rows are lambda I, step 0)
        int rc = factor_inverse(kp, h->rf_F, ldf, h->rf_H, kp, BICADMM_F64, h->rf_ws, st);
        if (rc) return fail(h, rc, "refit: Hessian not positive definite");
        if (sm) {
            H_CUDA(h, cudaMemcpyAsync(Yh.data(), h->rf_Y, sizeof(double) * kp * C, cudaMemcpyDeviceToHost, st));
            H_CUDA(h, cudaStreamSynchronize(st));
            for (int64_t a = 0; a < kp; ++a) g[a] = a < cnt ? Yh[a * C + sup[a] % C] : 0.0;
        } else {
            H_CUDA(h, cudaMemcpyAsync(g.data(), h->rf_g, sizeof(double) * kp, cudaMemcpyDeviceToHost, st));
            H_CUDA(h, cudaStreamSynchronize(st));
        }
        for (int64_t a = 0; a < kp; ++a) g[a] += lam * x[a];
        // d = -H^{-1} g
        H_CUDA(h, cudaMemcpyAsync(h->rf_r, g.data(), sizeof(double) * kp, cudaMemcpyHostToDevice, st));
        GemvDesc hd{h->rf_H, kp, kp, kp, h->rf_r, h->rf_d, 0};
        hd.alpha = -1.0;
        H_RC(h, launch_gemv(BICADMM_F64, &hd, 1, h->gemv_cap, st, 1));
        H_CUDA(h, cudaMemcpyAsync(d.data(), h->rf_d, sizeof(double) * kp, cudaMemcpyDeviceToHost, st));
        H_CUDA(h, cudaStreamSynchronize(st));
        h->rf_newton = it + 1;
        double gd = 0.0, dmax = 0.0, xmax = 1.0;
        for (int64_t a = 0; a < cnt; ++a) {
            gd += g[a] * d[a];
            dmax = std::max(dmax, std::fabs(d[a]));
            xmax = std::max(xmax, std::fabs(x[a]));
        }
        if (dmax <= 1e-13 * xmax) {
            for (int64_t a = 0; a < cnt; ++a) x[a] += d[a];
            break;
        }
        const bool resolve = -gd > 1e-12 * (1.0 + std::fabs(f));   // as in the oracle (R29)
        double alpha = 1.0, fn = f;
        for (int ls = 0; ls < 60; ++ls, alpha *= 0.5) {
            for (int64_t a = 0; a < kp; ++a) xn[a] = a < cnt ? x[a] + alpha * d[a] : 0.0;
            H_RC(h, objective(xn, fn));
            if (!resolve || fn <= f + 1e-4 * alpha * gd) break;
        }
        x = xn;   // the device state (w / W) belongs to the accepted point
        f = fn;
    }
    H_CUDA(h, cudaMemcpyAsync(h->rf_x, x.data(), sizeof(double) * kp, cudaMemcpyHostToDevice, st));
    H_RC(h, launch_rf_scatter(kp, h->rf_x, h->support, h->support_count, h->x_final, st));
    h->refit_iters = h->rf_newton;
    return BICADMM_OK;
}

static int do_finalize(bicadmm_handle* h) {
    const int64_t len = h->len;
    H_RC(h, launch_support(len, h->prm.kappa, h->z, h->support, h->support_count, h->st));
    H_CUDA(h, cudaMemsetAsync(h->x_final, 0, sizeof(double) * len, h->st));
    const int64_t kk = std::max<int64_t>(1, std::min<int64_t>(h->prm.kappa, len));
    k_scatter_support<<<(unsigned)((kk + 255) / 256), 256, 0, h->st>>>(h->z, h->support, h->support_count, h->x_final);
    BIC_LAUNCHED();
    if (h->prm.refit && h->loss == BICADMM_LS) H_RC(h, do_refit(h));
    // logistic / softmax refit (DESIGN R29), single- or multi-rank
    if (h->prm.refit && (h->loss == BICADMM_LOGISTIC || h->loss == BICADMM_SOFTMAX) && h->rf_AT)
        H_RC(h, do_refit_newton(h));
    // data term per node from p = sum_j A_ij x_final_j
    std::vector<GemvDesc> ax;
    for (auto& L : h->blk) ax.push_back(GemvDesc{L.A, L.lda, L.m, L.nj, h->x_final + L.c0 * h->C, L.pobj, 0, L.xt});
    H_RC(h, launch_gemv(h->dtype, ax.data(), (int)ax.size(), h->gemv_cap, h->st, h->C));
    std::vector<ProxNode> px;
    for (auto& nd : h->nod) {
        ProxNode p{};
        p.b = nd.b; p.m = nd.m; p.p = nd.pobj_base; p.pstride = nd.m * h->C; p.np = nd.np;
        p.sq_partial = nd.obj_partial;
        if (h->split_blocks) {
            p.S = nd.S;
            H_RC(h, launch_psum(h->C, &p, 1, nullptr, h->st));
        }
        px.push_back(p);
    }
    if (h->split_blocks) H_RC(h, allreduce(h, h->S_all, h->S_total, true));
    H_RC(h, launch_loss(h->loss, h->dtype, h->C, px.data(), (int)px.size(), h->st));
    H_CUDA(h, cudaMemsetAsync(h->node_obj, 0, sizeof(double) * h->N, h->st));
    for (auto& nd : h->nod) {
        k_sum_partials<<<1, 32, 0, h->st>>>(nd.obj_partial, nd.nprox_ctas, h->node_obj + nd.node);
        BIC_LAUNCHED();
    }
    // a node's loss is replicated on every rank of its group; the world sum divided by the
    // group size restores it (group sizes are powers of two in every placement we build)
    H_RC(h, allreduce(h, h->node_obj, h->N, false));
    k_sqnorm<<<1, 1024, 0, h->st>>>(len, h->x_final, h->wsum);
    BIC_LAUNCHED();
    H_CUDA(h, cudaMemcpyAsync(h->host_i64, h->support_count, sizeof(int64_t), cudaMemcpyDeviceToHost, h->st));
    std::vector<double> nobj(h->N + 1);
    H_CUDA(h, cudaMemcpyAsync(nobj.data(), h->node_obj, sizeof(double) * h->N, cudaMemcpyDeviceToHost, h->st));
    H_CUDA(h, cudaMemcpyAsync(nobj.data() + h->N, h->wsum, sizeof(double), cudaMemcpyDeviceToHost, h->st));
    H_CUDA(h, cudaStreamSynchronize(h->st));
    double obj = 0.0;
    const double gs = (multi_rank(h) && h->split_blocks) ? (double)h->gsize : 1.0;
    for (int i = 0; i < h->N; ++i) obj += nobj[i] / gs;
    obj += 0.5 * h->prm.lambda * nobj[h->N];
    h->objective = obj;
    h->support_len = h->host_i64[0];
    h->finalized = true;
    return BICADMM_OK;
}

static void fill_report(bicadmm_handle* h, bicadmm_report* rep) {
    if (!rep) return;
    rep->converged = h->converged;
    rep->outer_iters = h->outer_done;
    rep->inner_sweeps = h->inner_total;
    rep->support_len = h->support_len;
    rep->objective = h->objective;
    const OuterScalars& s = *h->host_sc;
    rep->p_r = s.p_r; rep->d_r = s.d_r; rep->b_r = s.b_r;
    rep->ms_setup = h->ms_setup;
    rep->ms_solve = h->ms_solve;
}

extern "C" int bicadmm_finalize(bicadmm_handle* h, bicadmm_report* rep) {
    NvtxRange nvtx_range("bicadmm_finalize");
    if (!h) return BICADMM_ERR_INVALID;
    if (h->dead) return BICADMM_ERR_STATE;
    int rc = do_finalize(h);
    if (rc) return rc;
    fill_report(h, rep);
    return BICADMM_OK;
}

// One thread: append (p_r, d_r, b_r, t, v, tau) to the device trace, and keep the while
// node running until the residual test (15) passes or `limit` iterations were done.
__global__ void k_loop_ctl(cudaGraphConditionalHandle hnd, const OuterScalars* __restrict__ sc,
                           double* __restrict__ trace, int* __restrict__ count, double ep, double ed, double eb) {
    const int c = count[0], limit = count[1];   // count[1]: iteration budget of this launch
    double* row = trace + (int64_t)c * 6;
    row[0] = sc->p_r; row[1] = sc->d_r; row[2] = sc->b_r; row[3] = sc->t; row[4] = sc->v; row[5] = sc->tau;
    count[0] = c + 1;
    const bool conv = sc->p_r <= ep && sc->d_r <= ed && sc->b_r <= eb;
    cudaGraphSetConditional(hnd, (!conv && c + 1 < limit) ? 1u : 0u);
}

// Device-resident outer loop: the fixed-schedule outer iteration as the
// body of a CUDA-graph while node; the loop ends on the device (converged or the iteration
// budget), so the host waits once per launch instead of once per outer iteration.
// Returns BICADMM_ERR_STATE when not applicable (the caller iterates from the host).
static int solve_device_loop(bicadmm_handle* h) {
    if (!graph_enabled() || h->prof || h->loop.failed || multi_rank(h) ||
        h->prm.inner_fixed <= 0 || h->outer_done < 1 || h->converged)
        return BICADMM_ERR_STATE;
    if (!h->schedule.empty() && h->outer_done - h->sched_start < h->sched_rows) return BICADMM_ERR_STATE;
    std::vector<int> want(h->nod.size(), h->prm.inner_fixed);
    const int maxs = h->prm.inner_fixed;
    auto& Lp = h->loop;
    if (!Lp.exec || Lp.sweeps != maxs) {
        if (Lp.exec) { cudaGraphExecDestroy(Lp.exec); Lp.exec = nullptr; }
        if (!h->cap_st && cudaStreamCreateWithFlags(&h->cap_st, cudaStreamNonBlocking) != cudaSuccess) {
            cudaGetLastError();
            Lp.failed = true;
            return BICADMM_ERR_STATE;
        }
        cudaGraph_t g = nullptr;
        cudaGraphConditionalHandle hnd = 0;
        cudaGraphNode_t node = nullptr;
        cudaGraphNodeParams cp{};
        bool ok = cudaGraphCreate(&g, 0) == cudaSuccess &&
                  cudaGraphConditionalHandleCreate(&hnd, g, 1, cudaGraphCondAssignDefault) == cudaSuccess;
        if (ok) {
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = hnd;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            ok = cudaGraphAddNode(&node, g, nullptr, 0, &cp) == cudaSuccess;
        }
        const int64_t l0 = g_launches.load();
        int rc = BICADMM_OK;
        if (ok) {
            cudaGraph_t body = cp.conditional.phGraph_out[0];
            cudaStream_t st0 = h->st;
            h->st = h->cap_st;
            ok = cudaStreamBeginCaptureToGraph(h->st, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) ==
                 cudaSuccess;
            if (ok) {
                h->capturing = true;
                rc = enqueue_fixed(h, want, maxs);
                if (!rc) rc = outer_step(h, false);
                if (!rc) {
                    k_loop_ctl<<<1, 1, 0, h->st>>>(hnd, h->sc, h->dtrace, h->dcount, h->prm.eps_p, h->prm.eps_d,
                                                  h->prm.eps_b);
                    count_launch();
                }
                cudaGraph_t out_g = nullptr;
                ok = cudaStreamEndCapture(h->st, &out_g) == cudaSuccess && rc == BICADMM_OK;
                h->capturing = false;
            }
            h->st = st0;
        }
        cudaGraphExec_t exec = nullptr;
        if (ok && cudaGraphInstantiate(&exec, g, 0) == cudaSuccess) Lp.exec = exec;
        if (g) cudaGraphDestroy(g);
        const int64_t captured = g_launches.load() - l0;
        g_launches.fetch_sub(captured);   // counted per executed iteration below
        if (!Lp.exec) {
            if (getenv("BICADMM_GRAPH_DEBUG")) fprintf(stderr, "bicadmm: device loop refused (rc %d)\n", rc);
            cudaGetLastError();
            h->dead = false;
            h->err.clear();
            h->pending.clear();
            h->evused = 0;
            Lp.failed = true;
            return BICADMM_ERR_STATE;
        }
        Lp.launches = captured;
        Lp.sweeps = maxs;
    }
    while (!h->converged && h->outer_done < h->prm.max_outer) {
        const int budget = (int)std::min<int64_t>(kLoopRows, h->prm.max_outer - h->outer_done);
        h->host_i32[0] = 0;
        h->host_i32[1] = budget;
        H_CUDA(h, cudaMemcpyAsync(h->dcount, h->host_i32, sizeof(int) * 2, cudaMemcpyHostToDevice, h->st));
        H_CUDA(h, cudaGraphLaunch(Lp.exec, h->st));
        int cnt = 0;
        H_CUDA(h, cudaMemcpyAsync(&cnt, h->dcount, sizeof(int), cudaMemcpyDeviceToHost, h->st));
        H_CUDA(h, cudaStreamSynchronize(h->st));
        std::vector<double> rows((size_t)cnt * 6);
        if (cnt > 0)
            H_CUDA(h, cudaMemcpy(rows.data(), h->dtrace, sizeof(double) * rows.size(), cudaMemcpyDeviceToHost));
        H_CUDA(h, cudaMemcpy(h->host_sc, h->sc, sizeof(OuterScalars), cudaMemcpyDeviceToHost));
        g_launches.fetch_add(Lp.launches * cnt);
        for (int k = 0; k < cnt; ++k) {
            const double* r = rows.data() + (size_t)k * 6;
            h->trace.push_back({r[0], r[1], r[2], r[3], r[4], r[5]});
            std::vector<int32_t> row(h->N, 0);
            for (size_t li = 0; li < h->nod.size(); ++li) row[h->nod[li].node] = maxs;
            h->inner_counts.insert(h->inner_counts.end(), row.begin(), row.end());
            h->converged = r[0] <= h->prm.eps_p && r[1] <= h->prm.eps_d && r[2] <= h->prm.eps_b;
        }
        h->outer_done += cnt;
        h->inner_total += (int64_t)cnt * maxs;
        h->finalized = false;
        if (cnt == 0) break;
    }
    return BICADMM_OK;
}

extern "C" int bicadmm_solve(bicadmm_handle* h, bicadmm_report* rep) {
    NvtxRange nvtx_range("bicadmm_solve");
    if (!h) return BICADMM_ERR_INVALID;
    if (h->dead) return BICADMM_ERR_STATE;
    H_CUDA(h, cudaEventRecord(h->e0, h->st));
    if (!h->converged && h->outer_done < 1 && h->prm.max_outer > 0) {   // the loop graph starts at k >= 1
        int rc = bicadmm_iterate(h, 1, nullptr);
        if (rc) return rc;
    }
    if (!h->converged && h->outer_done < h->prm.max_outer) {
        const int rc = solve_device_loop(h);
        if (rc && rc != BICADMM_ERR_STATE) return rc;
    }
    while (!h->converged && h->outer_done < h->prm.max_outer) {
        int rc = bicadmm_iterate(h, 1, nullptr);
        if (rc) return rc;
    }
    int rc = do_finalize(h);
    if (rc) return rc;
    H_CUDA(h, cudaEventRecord(h->e1, h->st));
    H_CUDA(h, cudaEventSynchronize(h->e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->e0, h->e1);
    h->ms_solve = ms;
    fill_report(h, rep);
    return BICADMM_OK;
}

extern "C" int bicadmm_set_schedule(bicadmm_handle* h, const int32_t* counts, int n_rows) {
    if (!h || (n_rows > 0 && !counts) || n_rows < 0) return BICADMM_ERR_INVALID;
    for (int64_t k = 0; k < (int64_t)n_rows * h->N; ++k)
        if (counts[k] < 0) return fail(h, BICADMM_ERR_INVALID, "negative sweep count");
    h->schedule.assign(counts, counts + (size_t)n_rows * h->N);
    h->sched_start = h->outer_done;
    h->sched_rows = n_rows;
    return BICADMM_OK;
}

// ======================================================================= get / destroy
extern "C" int bicadmm_get(bicadmm_handle* h, int field, void* dst, size_t bytes, int on_device, size_t* bytes_out) {
    if (!h) return BICADMM_ERR_INVALID;
    const int64_t len = h->len;
    size_t sz = 0;
    const void* src = nullptr;
    bool host_src = false;
    std::vector<double> tmp;
    std::vector<const void*> pieces;
    std::vector<size_t> piece_sz;
    switch (field) {
    case BICADMM_FIELD_Z: sz = sizeof(double) * len; src = h->z; break;
    case BICADMM_FIELD_S: sz = sizeof(double) * len; src = h->s; break;
    case BICADMM_FIELD_WBAR: sz = sizeof(double) * len; src = h->wbar; break;
    case BICADMM_FIELD_X_FINAL: sz = sizeof(double) * len; src = h->x_final; break;
    case BICADMM_FIELD_SCALARS: {
        const OuterScalars& s = *h->host_sc;
        tmp = {s.t, s.v, s.tau, s.p_r, s.d_r, s.b_r};
        sz = sizeof(double) * 6; src = tmp.data(); host_src = true;
        break;
    }
    case BICADMM_FIELD_X_LOCAL:
    case BICADMM_FIELD_U_LOCAL: {
        std::vector<const LBlock*> order(h->blk.size());
        for (auto& L : h->blk) order[L.user_index] = &L;
        for (auto* L : order) {
            pieces.push_back(field == BICADMM_FIELD_X_LOCAL ? L->x : L->u);
            piece_sz.push_back(sizeof(double) * L->nj * h->C);
            sz += piece_sz.back();
        }
        break;
    }
    case BICADMM_FIELD_P_LOCAL:
    case BICADMM_FIELD_R_LOCAL: {
        std::vector<const LBlock*> order(h->blk.size());
        for (auto& L : h->blk) order[L.user_index] = &L;
        for (auto* L : order) {
            const bool pf = field == BICADMM_FIELD_P_LOCAL;
            pieces.push_back(pf ? L->p : L->r);
            piece_sz.push_back(sizeof(double) * (pf ? L->m : L->nj) * h->C);
            sz += piece_sz.back();
        }
        break;
    }
    case BICADMM_FIELD_NU:
        for (auto& nd : h->nod) { pieces.push_back(nd.nu); piece_sz.push_back(sizeof(double) * nd.m * h->C); sz += piece_sz.back(); }
        break;
    case BICADMM_FIELD_SUPPORT: sz = sizeof(int64_t) * h->support_len; src = h->support; break;
    case BICADMM_FIELD_TRACE:
        for (auto& row : h->trace) tmp.insert(tmp.end(), row.begin(), row.end());
        sz = sizeof(double) * tmp.size(); src = tmp.data(); host_src = true;
        break;
    case BICADMM_FIELD_INNER_COUNTS:
        sz = sizeof(int32_t) * h->inner_counts.size(); src = h->inner_counts.data(); host_src = true;
        break;
    case BICADMM_FIELD_LAUNCHES: {
        static thread_local int64_t nl;
        nl = g_launches.load() - h->launches0;
        sz = sizeof(int64_t); src = &nl; host_src = true;
        break;
    }
    case BICADMM_FIELD_PHASE_MS:
        tmp.assign(h->phase_ms, h->phase_ms + BICADMM_NPHASE);
        sz = sizeof(double) * BICADMM_NPHASE; src = tmp.data(); host_src = true;
        break;
    case BICADMM_FIELD_PHASE_COUNT:
        sz = sizeof(int64_t) * BICADMM_NPHASE; src = h->phase_cnt; host_src = true;
        break;
    case BICADMM_FIELD_SWEEP_KIND: {
        h->host_i32[0] = h->fused_kind;
        h->host_i32[1] = 0;
        for (auto& L : h->blk) h->host_i32[1] += L.fat ? 1 : 0;
        sz = sizeof(int32_t) * 2; src = h->host_i32; host_src = true;
        break;
    }
    default: return fail(h, BICADMM_ERR_INVALID, "unknown field");
    }
    if (bytes_out) *bytes_out = sz;
    if (!dst) return BICADMM_OK;
    if (bytes != sz) return fail(h, BICADMM_ERR_DIM, "bytes must equal the field size");
    if (sz == 0) return BICADMM_OK;
    if (h->dead) return BICADMM_ERR_STATE;
    const cudaMemcpyKind kind = host_src ? (on_device ? cudaMemcpyHostToDevice : cudaMemcpyHostToHost)
                                         : (on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost);
    if (!pieces.empty()) {
        size_t off = 0;
        for (size_t k = 0; k < pieces.size(); ++k) {
            H_CUDA(h, cudaMemcpyAsync((char*)dst + off, pieces[k], piece_sz[k],
                                      on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->st));
            off += piece_sz[k];
        }
    } else {
        H_CUDA(h, cudaMemcpyAsync(dst, src, sz, kind, h->st));
    }
    H_CUDA(h, cudaStreamSynchronize(h->st));
    return BICADMM_OK;
}

extern "C" int bicadmm_set_profiling(bicadmm_handle* h, int on) {
    if (!h) return BICADMM_ERR_INVALID;
    if (h->dead) return BICADMM_ERR_STATE;
    H_CUDA(h, cudaStreamSynchronize(h->st));
    resolve_phases(h);
    for (int k = 0; k < BICADMM_NPHASE; ++k) { h->phase_ms[k] = 0.0; h->phase_cnt[k] = 0; }
    h->prof = on != 0;
    return BICADMM_OK;
}

extern "C" const char* bicadmm_last_error(const bicadmm_handle* h) { return h ? h->err.c_str() : "null handle"; }

extern "C" int bicadmm_destroy(bicadmm_handle* h) {
    if (!h) return BICADMM_OK;
    if (h->st || true) cudaStreamSynchronize(h->st);
    if (h->host_sc) cudaFreeHost(h->host_sc);
    if (h->host_i64) cudaFreeHost(h->host_i64);
    if (h->e0) cudaEventDestroy(h->e0);
    if (h->e1) cudaEventDestroy(h->e1);
    for (auto e : h->evpool) cudaEventDestroy(e);
    if (h->graph.exec) cudaGraphExecDestroy(h->graph.exec);
    if (h->loop.exec) cudaGraphExecDestroy(h->loop.exec);
    if (h->cap_st) cudaStreamDestroy(h->cap_st);
    delete h;
    return BICADMM_OK;
}
