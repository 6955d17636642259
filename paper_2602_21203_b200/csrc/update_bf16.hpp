// update_bf16.hpp -- entry points of the bf16 tensor-core path (update_bf16.cu), called
// by the C ABI in api.cu when dims.precision == SQUINT_BF16.
#pragma once
#include <cuda_runtime.h>

#include <string>

#include "../../include/squint.h"
#include "comm.hpp"

namespace sq {

// api.cu: records the thread-local error message, returns st.
squint_status set_error(squint_status st, const std::string& msg);

size_t bf16_workspace_bytes(const squint_dims& d);
bool bf16_region(const squint_dims& d, int region, size_t* offset, size_t* bytes);
squint_status bf16_update(const squint_dims& d, const squint_hparams& hp, const squint_replay& R,
                          const int64_t* idx, const uint8_t* shifts, const float* eps, int utd,
                          const squint_state& st, float* metrics, void* workspace, size_t workspace_bytes, Comm* comm,
                          cudaStream_t s);
// Creates the auxiliary stream/events of the encoder-backward branch (outside any capture) and
// returns whether the branch is in use.
bool bf16_prepare();
int bf16_options();  // squint_set_option state (part of the update graph cache key)
extern int g_check_enabled;  // squint_set_option key 3
extern int g_emul;           // squint_set_option key 4 (api.cu)
bool instrumentation_active();  // instrument.cu: launch / phase events requested
size_t bf16_act_workspace_bytes(const squint_dims& d, int64_t n);
squint_status bf16_act(const squint_dims& d, const squint_hparams& hp, const float* actor_params,
                       const float* critic_params, const uint8_t* frames, int64_t n, int factor, const float* proprio,
                       const float* eps, float* action_out, float* logp_out, uint8_t* ring, const int64_t* slots,
                       void* workspace, cudaStream_t s);

}  // namespace sq
