// tmap.cpp -- see tmap.hpp.
#include "tmap.hpp"

#include <cuda_runtime.h>

#include <cstring>
#include <mutex>
#include <unordered_map>

namespace sq {

namespace {
struct Key {
  uintptr_t p;
  int rows, cols, ld, box;
  bool operator==(const Key& o) const {
    return p == o.p && rows == o.rows && cols == o.cols && ld == o.ld && box == o.box;
  }
};
struct KeyHash {
  size_t operator()(const Key& k) const {
    size_t h = std::hash<uintptr_t>()(k.p);
    h ^= (size_t)k.rows * 0x9E3779B97F4A7C15ull + (size_t)k.cols * 0xC2B2AE3D27D4EB4Full + (size_t)k.ld * 131 +
         (size_t)k.box * 7;
    return h;
  }
};
std::mutex g_mu;
// cuTensorMapEncodeTiled through the runtime's driver entry point, so libsquint does not
// link libcuda (the CPU build box has no driver; the library must still load there).
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}
std::unordered_map<Key, CUtensorMap, KeyHash> g_cache;
}  // namespace

int tmap_get(const Mat& m, int box_rows, CUtensorMap* out) {
  if (!m.ptr || m.rows < 1 || m.cols < 1 || (m.ld * 2) % 16 || (reinterpret_cast<uintptr_t>(m.ptr) & 15) ||
      box_rows < 1 || box_rows > 256)
    return 1;
  Key k{reinterpret_cast<uintptr_t>(m.ptr), m.rows, m.cols, m.ld, box_rows};
  {
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_cache.find(k);
    if (it != g_cache.end()) {
      *out = it->second;
      return 0;
    }
  }
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)m.cols, (cuuint64_t)m.rows};
  cuuint64_t strides[1] = {(cuuint64_t)m.ld * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  EncodeFn enc = encode_fn();
  if (!enc) return 3;
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(m.ptr), dims,
                                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return 2;
  std::lock_guard<std::mutex> g(g_mu);
  if (g_cache.size() > 4096) g_cache.clear();
  g_cache[k] = map;
  *out = map;
  return 0;
}

}  // namespace sq
