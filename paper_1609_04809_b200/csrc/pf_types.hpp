// pf_types.hpp — plain types shared by the kernels and the host runtime.
#pragma once

#include <cstdint>

#ifndef __CUDACC__
#ifndef __restrict__
#define __restrict__ __restrict
#endif
#endif

namespace pf {

constexpr int kSlice = 32;     // SELL slice height == warp size
constexpr int kBlock = 256;    // threads per block of the row kernels
constexpr int kUnroll = 9;     // 27 = 3 x 9 entries per Q1 row: 9 loads in flight per chunk

struct SellView {
  const double* __restrict__ vals;
  const int32_t* __restrict__ cols;
  const int64_t* __restrict__ slice_ptr;
  const int32_t* __restrict__ row_len;
};

// One subdomain of the coarse level, for the sequential coarse solve.
struct CoarseSub {
  SellView A;
  const int32_t* host_of_own;  // device row of host own dof i (the device permutation)
  int32_t n_own;
  int64_t offset;  // subdomain position in the level vectors
};

}  // namespace pf
