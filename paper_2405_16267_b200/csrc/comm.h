// comm.h -- private: the communicator behind bicadmm_comm (include/bicadmm.h).
//
// Two backends carry the method's two exchange steps:
//   * NCCL (dlopen'ed libnccl.so.2, one process per GPU over NVLink/NVSwitch);
//   * an in-process emulation (bicadmm_emu_group): G "ranks" are G handles of one
//     process on one device, each driven by its own host thread and stream.  Its
//     AllReduce is a fixed-order device sum over the members' buffers (ascending rank),
//     ordered across the members' streams by CUDA events; the ranks meet at host
//     barriers.  No kernel ever waits on another, so it is safe on a single GPU
//     (B200_PROFILING.md: ranks whose kernels wait on one another must not share a GPU).
//     It exists to run the multi-rank code path of block-major placements (split block
//     sums, Algorithm 2's AllReduce) on one GPU against the oracle.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

struct EmuGroup;

struct bicadmm_comm {
    int world = 1, rank = 0, device = 0, color = 0, group_size = 1;
    // BICADMM_NCCL_SELF at init (world == 1): 1 = a real one-rank NCCL communicator, so the
    // multi-rank code path runs on one GPU; 2 = also route every node's block sum through
    // the per-sweep group AllReduce (the split-block path)
    int self_mode = 0;
    bool self = false;
    EmuGroup* emu = nullptr;   // in-process emulated backend (bicadmm_comm_init_emu)
    void* world_comm = nullptr;   // ncclComm_t
    void* group_comm = nullptr;   // ncclComm_t (ranks of the same group_color)
};

namespace bic {

// In-place sum AllReduce of `count` doubles over the group (ranks of the same color) or
// the world, enqueued on `st`.  Returns BICADMM_OK or an error code with *why set.
int comm_allreduce(bicadmm_comm* c, double* buf, int64_t count, bool group, cudaStream_t st, std::string* why);
// Several in-place AllReduces over the same communicator as one collective step (NCCL group
// call; the emulation runs them back to back).
int comm_allreduce_many(bicadmm_comm* c, double* const* bufs, const int64_t* counts, int n, bool group,
                        cudaStream_t st, std::string* why);
// Ranks sharing this rank's group_color (the emulation counts registered ranks).
int comm_group_size(const bicadmm_comm* c);

}  // namespace bic
