// pf_types.hpp — plain types shared by the kernels and the host runtime.
#pragma once

#include <cstdint>

#include <cstddef>

#ifndef __CUDACC__
#ifndef __restrict__
#define __restrict__ __restrict
#endif
#define PF_HD
#else
#define PF_HD __host__ __device__
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

// The coarse level packed for a shared-memory solve: own rows of every subdomain in the
// order the sequential sweep visits them (subdomain ascending, host order inside), entries
// in stored order with level-global column indices; built once on the host.
struct CoarsePack {
  int32_t n_total;      // level vector length (all subdomains)
  int32_t n_rows;       // own rows, all subdomains
  int32_t nnz;
  int32_t n_sub;
  const int32_t* sub_rows;  // n_sub + 1: row range of each subdomain (norm grouping)
  const int32_t* rowptr;    // n_rows + 1
  const int32_t* rowdev;    // level-global index of each row
  const int32_t* cols;      // level-global
  const double* vals;
  const int32_t *ms_dst, *ms_src, *h1_dst, *h1_src;
  int32_t ms_n, h1_n;
};

PF_HD inline size_t coarse_pack_smem(const CoarsePack& P) {
  return sizeof(double) * (static_cast<size_t>(P.n_total) + P.n_rows + P.nnz) +
         sizeof(int32_t) * (static_cast<size_t>(P.n_rows) * 2 + 1 + P.nnz + P.n_sub + 1 +
                            2 * static_cast<size_t>(P.ms_n) + 2 * static_cast<size_t>(P.h1_n));
}

}  // namespace pf
