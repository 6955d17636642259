// update_bf16.cu -- bf16 tensor-core update path (placeholder until the tcgen05 kernels land).
#include "update_bf16.cuh"

namespace sq {
size_t bf16_ws_bytes(const squint_dims&) { return 0; }
squint_status update_one_bf16(const squint_dims&, const squint_hparams&, const Layout&, char*, const squint_replay&,
                              const int64_t*, const uint8_t*, const float*, const squint_state&, float*, Comm*, float,
                              cudaStream_t, std::string* err) {
  *err = "bf16 tensor-core path not built yet";
  return SQUINT_EUNSUPPORTED;
}
}  // namespace sq
