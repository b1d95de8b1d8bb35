// blaz_types.h -- kernel-side views shared by all translation units.
#pragma once
#include <cstdint>

namespace blz {

// The 64-entry DCT basis t(i,u) (H/dct.hpp:14-26), passed BY VALUE as a
// kernel parameter: it lives in constant bank 0 and every warp reads the
// same entry at the same time, so DMUL takes it as a c[0x0][...] operand.
struct Basis {
  double t[64];
};

// Device view of a blz_cmat (SoA).
struct CMat {
  uint64_t rows, cols, br, bc;
  double* first;
  double* slope;
  uint8_t* scale;
  int8_t* coeffs;
  __host__ __device__ uint64_t nb() const { return br * bc; }
};

}  // namespace blz

namespace blz {
// Device error codes latched in the context (low byte of the latch word).
constexpr unsigned DERR_NONFINITE_CODE = 1;  // "normalize: non-finite input"          H/codec.hpp:21
constexpr unsigned DERR_PREDICT_CODE = 2;    // "predict: mean slope must be positive" H/codec.hpp:86
constexpr unsigned DERR_DOT_RANGE_CODE = 3;  // "mat_dot: index out of range"          H/matrix.hpp:160
constexpr unsigned DERR_IO_NONFINITE_CODE = 4;  // "write_compressed: non-finite block field" H/io.hpp:102-103
constexpr unsigned DERR_IO_ZERO_PHI_CODE = 5;   // "compressed matrix: zero scale factor in block t" H/io.hpp:129-130
}  // namespace blz
