// comm.cpp -- NCCL plumbing (compiled against the NCCL 2.28 headers torch ships, linked to
// the same libnccl.so.2 torch loads).
#include "comm.hpp"

#include <nccl.h>

#include <cstring>
#include <string>

namespace sq {

struct Comm {
  ncclComm_t nc;
  int rank, nranks;
};

static thread_local std::string g_comm_err;

const char* comm_error() { return g_comm_err.c_str(); }

static int nccl_fail(ncclResult_t r, const char* what) {
  g_comm_err = std::string(what) + ": " + ncclGetErrorString(r);
  return 1;
}

int comm_unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(out128, &id, sizeof(id));
  return 0;
}

int comm_init(Comm** c, const void* id128, int rank, int nranks) {
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  Comm* x = new Comm{nullptr, rank, nranks};
  ncclResult_t r = ncclCommInitRank(&x->nc, nranks, id, rank);
  if (r != ncclSuccess) {
    delete x;
    return nccl_fail(r, "ncclCommInitRank");
  }
  *c = x;
  return 0;
}

void comm_destroy(Comm* c) {
  if (!c) return;
  ncclCommDestroy(c->nc);
  delete c;
}

int comm_nranks(const Comm* c) { return c->nranks; }

int comm_allreduce_sum(Comm* c, float* buf, int64_t n, cudaStream_t s) {
  if (c->nranks == 1) return 0;
  ncclResult_t r = ncclAllReduce(buf, buf, (size_t)n, ncclFloat32, ncclSum, c->nc, s);
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
  return 0;
}

}  // namespace sq
