// layout.hpp -- host-side parameter layout and workspace plan for libsquint.
//
// Parameter groups (squint.h): CRITIC = encoder psi + critic projection +
// twin heads; TARGET = the CRITIC tensors except psi, at the same relative offsets, so the
// Polyak update is one contiguous axpby over CRITIC[enc_end:] and TARGET[0:];
// ACTOR = actor projection + MLP; ALPHA = log alpha.  Every tensor starts on a 32-float
// (128-byte) boundary so kernels can use 16-byte vector access.
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/squint.h"

namespace sq {

struct TInfo {
  std::string name;
  int group;
  int64_t off, numel;
  int ndim;
  int shape[4];
};

struct Layout {
  std::vector<TInfo> t;
  int64_t gsize[4] = {0, 0, 0, 0};
  int64_t enc_end = 0;  // CRITIC offset where the non-encoder tensors start
  int64_t off(int group, const std::string& name) const;
};

// Validates dims (returns false + message on error).
bool check_dims(const squint_dims& d, std::string* err);
Layout make_layout(const squint_dims& d);

// critic head width: n_atoms logits (C51) or one Q value (scalar MSE critic, f3)
inline int head_out(const squint_dims& d) { return d.critic_kind == SQUINT_CRITIC_MSE ? 1 : d.n_atoms; }
inline int conv1_out(const squint_dims& d) { return (d.img_h - 3) / 2 + 1; }
inline int conv2_out(const squint_dims& d) { return conv1_out(d) - 2; }
inline int flat_dim(const squint_dims& d) { return d.conv_ch * conv2_out(d) * conv2_out(d); }

// Bump allocator over the caller's workspace (256-byte aligned sub-buffers).
struct WsPlan {
  size_t top = 0;
  size_t take(size_t bytes) {
    size_t o = (top + 255) & ~size_t(255);
    top = o + bytes;
    return o;
  }
};

}  // namespace sq
