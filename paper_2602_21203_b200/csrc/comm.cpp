// comm.cpp -- NCCL plumbing (compiled against the NCCL 2.28 headers torch ships, linked to
// the same libnccl.so.2 torch loads).
#include "comm.hpp"

#include <nccl.h>

#include <cuda.h>

#include <cstring>
#include <map>
#include <string>
#include <vector>

namespace sq {

struct Comm {
  ncclComm_t nc;
  int rank, nranks;
  int mode = 0;  // 0: ncclAllReduce + replicated Adam, 1: peer-memory all-reduce fused with sharded Adam (f1)
  // peer mode: local pointer -> every rank's mapping of its copy (own rank: the pointer itself)
  std::map<uintptr_t, std::vector<char*>> peers;
  std::map<std::string, char*> bases;  // (rank, IPC handle) -> opened allocation base
  std::vector<char*> opened;      // IPC mappings to close
  unsigned* flags = nullptr;      // [kMaxRanks] barrier arrivals per source rank + [1] own epoch
  cudaStream_t xs = nullptr;      // host-synchronous exchanges
  void* xbuf = nullptr;           // device staging of the exchanged records
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
  for (char* p : c->opened) cudaIpcCloseMemHandle(p);
  if (c->flags) cudaFree(c->flags);
  if (c->xbuf) cudaFree(c->xbuf);
  if (c->xs) cudaStreamDestroy(c->xs);
  ncclCommDestroy(c->nc);
  delete c;
}

int comm_nranks(const Comm* c) { return c->nranks; }
int comm_rank(const Comm* c) { return c->rank; }
int comm_mode(const Comm* c) { return c->mode; }

static int cuda_fail(cudaError_t e, const char* what) {
  g_comm_err = std::string(what) + ": " + cudaGetErrorString(e);
  return 1;
}
#define CM_CK(x, what)                          \
  do {                                          \
    cudaError_t e_ = (x);                       \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

// One record per rank: the IPC handle of the allocation and the pointer's offset in it.
struct PeerRec {
  cudaIpcMemHandle_t h;
  int64_t off;
  int64_t base_size;
};

int comm_set_mode(Comm* c, int mode) {
  if (mode != 0 && mode != 1) {
    g_comm_err = "mode must be 0 or 1";
    return 1;
  }
  if (mode == 1 && c->nranks > kMaxRanks) {
    g_comm_err = "peer mode supports at most 8 ranks (one NVSwitch box)";
    return 1;
  }
  if (mode == 1 && !c->flags) {
    CM_CK(cudaMalloc(&c->flags, (kMaxRanks + 1) * sizeof(unsigned)), "cudaMalloc(flags)");
    CM_CK(cudaMemset(c->flags, 0, (kMaxRanks + 1) * sizeof(unsigned)), "cudaMemset(flags)");
    CM_CK(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  }
  c->mode = mode;
  return 0;
}

// Every rank's mapping of `local` (collective: all ranks call it for the same logical buffers
// in the same order).  Cached by pointer; the first call per pointer exchanges (cudaIpcMemHandle,
// offset) records with ncclAllGather -- the caching allocator may place the buffer at different
// offsets of its allocation on different ranks -- and opens each peer allocation once.
int comm_peer_ptrs(Comm* c, const void* local, void** out) {
  auto it = c->peers.find((uintptr_t)local);
  if (it == c->peers.end()) {
    std::vector<char*> ptrs(c->nranks, nullptr);
    ptrs[c->rank] = (char*)local;
    if (c->nranks > 1) {
      // the driver entry point through the runtime (no link-time libcuda dependency)
      using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
      static GetRange get_range = nullptr;
      if (!get_range) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        CM_CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q), "cudaGetDriverEntryPoint");
        if (!fn) {
          g_comm_err = "cuMemGetAddressRange not found";
          return 1;
        }
        get_range = reinterpret_cast<GetRange>(fn);
      }
      CUdeviceptr base = 0;
      size_t size = 0;
      if (get_range(&base, &size, (CUdeviceptr)local) != CUDA_SUCCESS) {
        g_comm_err = "cuMemGetAddressRange: pointer is not device memory";
        return 1;
      }
      PeerRec mine;
      memset(&mine, 0, sizeof(mine));
      CM_CK(cudaIpcGetMemHandle(&mine.h, (void*)base), "cudaIpcGetMemHandle");
      mine.off = (int64_t)((const char*)local - (const char*)base);
      mine.base_size = (int64_t)size;
      if (!c->xs) CM_CK(cudaStreamCreateWithFlags(&c->xs, cudaStreamNonBlocking), "cudaStreamCreate");
      if (!c->xbuf) CM_CK(cudaMalloc(&c->xbuf, sizeof(PeerRec) * kMaxRanks), "cudaMalloc(xbuf)");
      char* xb = (char*)c->xbuf;
      CM_CK(cudaMemcpy(xb + sizeof(PeerRec) * c->rank, &mine, sizeof(mine), cudaMemcpyHostToDevice), "cudaMemcpy");
      ncclResult_t r = ncclAllGather(xb + sizeof(PeerRec) * c->rank, xb, sizeof(PeerRec), ncclUint8, c->nc, c->xs);
      if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather(ipc handles)");
      CM_CK(cudaStreamSynchronize(c->xs), "cudaStreamSynchronize");
      std::vector<PeerRec> recs(c->nranks);
      CM_CK(cudaMemcpy(recs.data(), xb, sizeof(PeerRec) * c->nranks, cudaMemcpyDeviceToHost), "cudaMemcpy");
      for (int q = 0; q < c->nranks; ++q) {
        if (q == c->rank) continue;
        const std::string key = std::to_string(q) + ":" + std::string(recs[q].h.reserved, sizeof(recs[q].h.reserved));
        auto ob = c->bases.find(key);
        if (ob == c->bases.end()) {
          void* pb = nullptr;
          CM_CK(cudaIpcOpenMemHandle(&pb, recs[q].h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
          c->opened.push_back((char*)pb);
          ob = c->bases.emplace(key, (char*)pb).first;
        }
        ptrs[q] = ob->second + recs[q].off;
      }
    }
    it = c->peers.emplace((uintptr_t)local, ptrs).first;
  }
  for (int q = 0; q < c->nranks; ++q) out[q] = it->second[q];
  return 0;
}

unsigned* comm_flags(Comm* c) { return c->flags; }

int comm_allreduce_sum(Comm* c, float* buf, int64_t n, cudaStream_t s) {
  if (c->nranks == 1) return 0;
  ncclResult_t r = ncclAllReduce(buf, buf, (size_t)n, ncclFloat32, ncclSum, c->nc, s);
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
  return 0;
}

}  // namespace sq
