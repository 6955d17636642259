// update_bf16.cuh -- bf16 tensor-core (tcgen05) update path.
#pragma once
#include <cuda_runtime.h>

#include <string>

#include "../../include/squint.h"
#include "comm.hpp"
#include "layout.hpp"

namespace sq {
size_t bf16_ws_bytes(const squint_dims& d);
squint_status update_one_bf16(const squint_dims& d, const squint_hparams& hp, const Layout& L, char* ws,
                              const squint_replay& R, const int64_t* idx, const uint8_t* sh, const float* eps,
                              const squint_state& st, float* metrics, Comm* comm, float inv_btotal, cudaStream_t s,
                              std::string* err);
}  // namespace sq
