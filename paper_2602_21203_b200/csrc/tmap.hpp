// tmap.hpp -- host-side TMA tensor maps (cuTensorMapEncodeTiled) for bf16 row-major
// matrices, with a small cache keyed by (pointer, shape, stride, box).
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace sq {

// A bf16 row-major matrix in device memory: rows x cols logical, ld elements per row
// (ld * 2 bytes must be a multiple of 16).  Elements beyond rows/cols are never read: the
// TMA unit zero-fills out-of-bounds box elements, which is how K tails and N/M tails of
// every GEMM are padded.
struct Mat {
  const void* ptr;
  int rows, cols, ld;
};

// SWIZZLE_128B map with box {64 columns, box_rows rows}.  Returns 0 on success.
int tmap_get(const Mat& m, int box_rows, CUtensorMap* out);

}  // namespace sq
