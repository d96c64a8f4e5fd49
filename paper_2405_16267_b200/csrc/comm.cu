// comm.cu -- bicadmm_comm: NCCL (dlopen) and the in-process emulated group (comm.h).
//
// The method has two exchange steps: Algorithm 2's per-sweep AllReduce
// of the m-vector block sums over the ranks holding blocks of the same nodes (P:244,
// P:252), and the per-outer AllReduce of sum_i (x_i + u_i) plus the node residuals over
// all ranks ("Collect").  Both are in-place FP64 sums.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <condition_variable>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/bicadmm.h"
#include "comm.h"
#include "common.cuh"

#if __has_include(<nccl.h>)
#include <nccl.h>
#define BIC_HAVE_NCCL 1
#else
#define BIC_HAVE_NCCL 0
#endif

namespace {

// ----------------------------------------------------------------------------- NCCL (dlopen)
#if BIC_HAVE_NCCL
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
    bool load() {
        if (h) return true;
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return false;
        GetUniqueId = (decltype(GetUniqueId))dlsym(h, "ncclGetUniqueId");
        CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
        CommSplit = (decltype(CommSplit))dlsym(h, "ncclCommSplit");
        AllReduce = (decltype(AllReduce))dlsym(h, "ncclAllReduce");
        GroupStart = (decltype(GroupStart))dlsym(h, "ncclGroupStart");
        GroupEnd = (decltype(GroupEnd))dlsym(h, "ncclGroupEnd");
        CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
        CommCount = (decltype(CommCount))dlsym(h, "ncclCommCount");
        return GetUniqueId && CommInitRank && CommSplit && AllReduce && GroupStart && GroupEnd && CommDestroy &&
               CommCount;
    }
};
NcclApi g_nccl;

// Pin the collective algorithm and protocol: the reduction order, and with it
// every replicated iterate, is then the same from run to run.  A caller's own NCCL_ALGO /
// NCCL_PROTO win (setenv without overwrite).
void pin_nccl_env() {
    setenv("NCCL_ALGO", "Ring", 0);
    setenv("NCCL_PROTO", "Simple", 0);
}
#endif

}  // namespace

// ----------------------------------------------------------------------------- emulation
// Host barrier with generations (the members of one group, or the whole world).
struct EmuBarrier {
    int arrived = 0;
    long gen = 0;
};
struct EmuSlot {
    bool registered = false;
    int color = 0;
    double* buf = nullptr;
    int64_t count = 0;
    cudaEvent_t ready = nullptr, done = nullptr;   // buffer written / group sum finished reading
    double* tmp = nullptr;                         // this rank's sum, copied back after barrier 2
    size_t tmp_cap = 0;
};
struct EmuGroup {
    int world = 0;
    std::mutex mu;
    std::condition_variable cv;
    std::vector<EmuSlot> slot;
    std::map<int, EmuBarrier> bars;   // key: group color, or -1 for the world
    bool failed = false;
};

namespace bic {

constexpr int kEmuMax = 64;
struct EmuPtrs { const double* p[kEmuMax]; };

// out[i] = sum over members k = 0, 1, ... (ascending rank) of in_k[i]: every member computes
// the same sum in the same order, so the replicated results are bit-identical.
__global__ void k_emu_sum(int64_t n, EmuPtrs in, int nm, double* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < nm; ++k) s += in.p[k][i];
        out[i] = s;
    }
}

static void emu_barrier(EmuGroup* g, int key, int n) {
    std::unique_lock<std::mutex> lk(g->mu);
    EmuBarrier& b = g->bars[key];
    const long gen = b.gen;
    if (++b.arrived == n) {
        b.arrived = 0;
        ++b.gen;
        g->cv.notify_all();
    } else {
        g->cv.wait(lk, [&] { return b.gen != gen; });
    }
}

static int emu_allreduce(bicadmm_comm* c, double* buf, int64_t count, bool group, cudaStream_t st, std::string* why) {
    EmuGroup* g = c->emu;
    std::vector<int> mem;
    for (int r = 0; r < g->world; ++r)
        if (g->slot[r].registered && (!group || g->slot[r].color == c->color)) mem.push_back(r);
    const int n = (int)mem.size();
    if (n > kEmuMax) { *why = "emulated group larger than 64 ranks"; return BICADMM_ERR_INVALID; }
    const int key = group ? c->color : -1;
    EmuSlot& me = g->slot[c->rank];
    if (me.tmp_cap < (size_t)count) {   // the communicator owns its scratch (as NCCL owns its buffers)
        if (me.tmp) cudaFree(me.tmp);
        me.tmp = nullptr;
        me.tmp_cap = 0;
        if (cudaMalloc(&me.tmp, sizeof(double) * (size_t)count) != cudaSuccess) { *why = "emu scratch"; return BICADMM_ERR_CUDA; }
        me.tmp_cap = (size_t)count;
    }
    me.buf = buf;
    me.count = count;
    if (cudaEventRecord(me.ready, st) != cudaSuccess) { *why = "emu event"; return BICADMM_ERR_CUDA; }
    emu_barrier(g, key, n);   // 1: every member's buffer is registered and its ready event recorded
    EmuPtrs ptrs{};
    bool same = true;
    for (int k = 0; k < n; ++k) {
        const EmuSlot& o = g->slot[mem[k]];
        ptrs.p[k] = o.buf;
        same = same && o.count == count;
        if (cudaStreamWaitEvent(st, o.ready, 0) != cudaSuccess) { *why = "emu wait"; return BICADMM_ERR_CUDA; }
    }
    if (!same) {   // a collective with mismatched sizes: every member sees it (NCCL would hang)
        emu_barrier(g, key, n);
        *why = "emulated AllReduce: members passed different counts";
        return BICADMM_ERR_NCCL;
    }
    const unsigned grid = (unsigned)std::min<int64_t>((count + 255) / 256, 148 * 8);
    k_emu_sum<<<grid, 256, 0, st>>>(count, ptrs, n, me.tmp);
    count_launch();
    if (cudaPeekAtLastError() != cudaSuccess || cudaEventRecord(me.done, st) != cudaSuccess) {
        *why = "emu sum";
        return BICADMM_ERR_CUDA;
    }
    emu_barrier(g, key, n);   // 2: every member's sum is enqueued (and its done event recorded)
    for (int k = 0; k < n; ++k)   // nobody overwrites its buffer before all sums have read it
        if (cudaStreamWaitEvent(st, g->slot[mem[k]].done, 0) != cudaSuccess) { *why = "emu wait"; return BICADMM_ERR_CUDA; }
    if (cudaMemcpyAsync(buf, me.tmp, sizeof(double) * (size_t)count, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
        *why = "emu copy";
        return BICADMM_ERR_CUDA;
    }
    return BICADMM_OK;
}

int comm_group_size(const bicadmm_comm* c) {
    if (!c) return 1;
    if (c->emu) {
        std::lock_guard<std::mutex> lk(c->emu->mu);
        int n = 0;
        for (auto& s : c->emu->slot) n += s.registered && s.color == c->color;
        return n;
    }
    return c->group_size;
}

int comm_allreduce(bicadmm_comm* c, double* buf, int64_t count, bool group, cudaStream_t st, std::string* why) {
    if (count <= 0) return BICADMM_OK;
    if (c->emu) return emu_allreduce(c, buf, count, group, st, why);
#if BIC_HAVE_NCCL
    ncclComm_t nc = (ncclComm_t)(group ? c->group_comm : c->world_comm);
    if (!nc || g_nccl.AllReduce(buf, buf, (size_t)count, ncclFloat64, ncclSum, nc, st) != ncclSuccess) {
        *why = "ncclAllReduce";
        return BICADMM_ERR_NCCL;
    }
    return BICADMM_OK;
#else
    (void)buf; (void)group; (void)st;
    *why = "built without NCCL";
    return BICADMM_ERR_NCCL;
#endif
}

int comm_allreduce_many(bicadmm_comm* c, double* const* bufs, const int64_t* counts, int n, bool group,
                        cudaStream_t st, std::string* why) {
    if (c->emu) {
        for (int k = 0; k < n; ++k) {
            const int rc = emu_allreduce(c, bufs[k], counts[k], group, st, why);
            if (rc) return rc;
        }
        return BICADMM_OK;
    }
#if BIC_HAVE_NCCL
    ncclComm_t nc = (ncclComm_t)(group ? c->group_comm : c->world_comm);
    if (!nc || g_nccl.GroupStart() != ncclSuccess) { *why = "ncclGroupStart"; return BICADMM_ERR_NCCL; }
    bool ok = true;
    for (int k = 0; k < n; ++k)
        if (counts[k] > 0)
            ok = ok && g_nccl.AllReduce(bufs[k], bufs[k], (size_t)counts[k], ncclFloat64, ncclSum, nc, st) == ncclSuccess;
    ok = g_nccl.GroupEnd() == ncclSuccess && ok;
    if (!ok) { *why = "ncclAllReduce (group)"; return BICADMM_ERR_NCCL; }
    return BICADMM_OK;
#else
    (void)bufs; (void)counts; (void)n; (void)group; (void)st;
    *why = "built without NCCL";
    return BICADMM_ERR_NCCL;
#endif
}

}  // namespace bic

// ----------------------------------------------------------------------------- C ABI
extern "C" {

int bicadmm_uid_size(void) {
#if BIC_HAVE_NCCL
    return (int)sizeof(ncclUniqueId);
#else
    return 128;
#endif
}

int bicadmm_get_unique_id(void* uid_out) {
#if BIC_HAVE_NCCL
    if (!uid_out) return BICADMM_ERR_INVALID;
    if (!g_nccl.load()) return BICADMM_ERR_NCCL;
    ncclUniqueId id;
    if (g_nccl.GetUniqueId(&id) != ncclSuccess) return BICADMM_ERR_NCCL;
    memcpy(uid_out, &id, sizeof(id));
    return BICADMM_OK;
#else
    (void)uid_out;
    return BICADMM_ERR_NCCL;
#endif
}

int bicadmm_comm_init(int world, int rank, int device, const void* uid, int group_color, bicadmm_comm** out) {
    if (!out || world < 1 || rank < 0 || rank >= world || group_color < 0) return BICADMM_ERR_INVALID;
    bicadmm_comm* c = new bicadmm_comm();
    c->world = world; c->rank = rank; c->device = device; c->color = group_color;
    if (cudaSetDevice(device) != cudaSuccess) { delete c; return BICADMM_ERR_CUDA; }
    const char* se = getenv("BICADMM_NCCL_SELF");
    c->self_mode = world == 1 && se ? atoi(se) : 0;
    c->self = c->self_mode != 0;
    if (world > 1 || c->self) {
#if BIC_HAVE_NCCL
        if ((!uid && !c->self) || !g_nccl.load()) { delete c; return BICADMM_ERR_NCCL; }
        pin_nccl_env();
        ncclUniqueId id;
        if (c->self) {
            if (g_nccl.GetUniqueId(&id) != ncclSuccess) { delete c; return BICADMM_ERR_NCCL; }
        } else {
            memcpy(&id, uid, sizeof(id));
        }
        ncclComm_t wc = nullptr, gc = nullptr;
        if (g_nccl.CommInitRank(&wc, world, id, rank) != ncclSuccess) { delete c; return BICADMM_ERR_NCCL; }
        if (g_nccl.CommSplit(wc, group_color, rank, &gc, nullptr) != ncclSuccess) {
            g_nccl.CommDestroy(wc);
            delete c;
            return BICADMM_ERR_NCCL;
        }
        g_nccl.CommCount(gc, &c->group_size);
        c->world_comm = wc;
        c->group_comm = gc;
#else
        delete c;
        return BICADMM_ERR_NCCL;
#endif
    }
    *out = c;
    return BICADMM_OK;
}

int bicadmm_comm_destroy(bicadmm_comm* c) {
    if (!c) return BICADMM_OK;
#if BIC_HAVE_NCCL
    if (c->group_comm) g_nccl.CommDestroy((ncclComm_t)c->group_comm);
    if (c->world_comm) g_nccl.CommDestroy((ncclComm_t)c->world_comm);
#endif
    if (c->emu) {
        std::lock_guard<std::mutex> lk(c->emu->mu);
        c->emu->slot[c->rank].registered = false;
    }
    delete c;
    return BICADMM_OK;
}

int bicadmm_emu_group_create(int world, bicadmm_emu_group** out) {
    if (!out || world < 1 || world > bic::kEmuMax) return BICADMM_ERR_INVALID;
    EmuGroup* g = new EmuGroup();
    g->world = world;
    g->slot.resize((size_t)world);
    for (auto& s : g->slot)
        if (cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming) != cudaSuccess) {
            bicadmm_emu_group_destroy(reinterpret_cast<bicadmm_emu_group*>(g));
            return BICADMM_ERR_CUDA;
        }
    *out = reinterpret_cast<bicadmm_emu_group*>(g);
    return BICADMM_OK;
}

int bicadmm_comm_init_emu(bicadmm_emu_group* grp, int rank, int device, int group_color, bicadmm_comm** out) {
    EmuGroup* g = reinterpret_cast<EmuGroup*>(grp);
    if (!g || !out || rank < 0 || rank >= g->world || group_color < 0) return BICADMM_ERR_INVALID;
    if (cudaSetDevice(device) != cudaSuccess) return BICADMM_ERR_CUDA;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        if (g->slot[rank].registered) return BICADMM_ERR_INVALID;
        g->slot[rank].registered = true;
        g->slot[rank].color = group_color;
    }
    bicadmm_comm* c = new bicadmm_comm();
    c->world = g->world; c->rank = rank; c->device = device; c->color = group_color;
    c->emu = g;
    *out = c;
    return BICADMM_OK;
}

int bicadmm_emu_group_destroy(bicadmm_emu_group* grp) {
    EmuGroup* g = reinterpret_cast<EmuGroup*>(grp);
    if (!g) return BICADMM_OK;
    for (auto& s : g->slot) {
        if (s.ready) cudaEventDestroy(s.ready);
        if (s.done) cudaEventDestroy(s.done);
        if (s.tmp) cudaFree(s.tmp);
    }
    delete g;
    return BICADMM_OK;
}

}  // extern "C"
