// comm.hpp -- NCCL communicator for the data-parallel update.
// Bootstrap: rank 0 creates an ncclUniqueId, the Python side broadcasts its 128 bytes
// with torch.distributed, every rank calls ncclCommInitRank.  Gradients are summed with
// ncclAllReduce on the update stream (NVLink / NVSwitch on one B200 box).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sq {
struct Comm;
int comm_unique_id(void* out128);
int comm_init(Comm** c, const void* id128, int rank, int nranks);
void comm_destroy(Comm* c);
int comm_nranks(const Comm* c);
int comm_allreduce_sum(Comm* c, float* buf, int64_t n, cudaStream_t s);
// f1: peer-memory all-reduce fused with a sharded Adam.  mode 1 maps every
// rank's gradient / parameter buffers into each process (CUDA IPC over NVLink) so one kernel
// per group sums the rank's 1/G slice of the gradients from all peers, steps Adam on it and
// stores the stepped slice into every peer's parameters.
constexpr int kMaxRanks = 8;
int comm_rank(const Comm* c);
int comm_mode(const Comm* c);
int comm_set_mode(Comm* c, int mode);
int comm_peer_ptrs(Comm* c, const void* local, void** out /* [nranks] */);
unsigned* comm_flags(Comm* c);  // [kMaxRanks] arrivals per source rank, [kMaxRanks] = own epoch
const char* comm_error();
}  // namespace sq
