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
const char* comm_error();
}  // namespace sq
