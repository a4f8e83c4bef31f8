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
#ifndef PF_BLOCK
#define PF_BLOCK 256
#endif
#ifndef PF_CHUNK_GROUPS
#define PF_CHUNK_GROUPS 1
#endif
constexpr int kBlock = PF_BLOCK;  // threads per block of the row kernels
constexpr int kUnroll = 9;     // 27 = 3 x 9 entries per Q1 row: 9 loads in flight per chunk
constexpr int kGroup = 4;      // SELL-32x4: 4 consecutive entries of a row are contiguous per lane
constexpr int kChunkGroups = PF_CHUNK_GROUPS;  // groups of 4 entries per chunk in the bandwidth kernels
#ifndef PF_SOR_GROUPS
#define PF_SOR_GROUPS 1
#endif
// colour sweeps are single-wave launches: a row's latency chain, not throughput, bounds them
constexpr int kSorChunkGroups = PF_SOR_GROUPS;
// Minimum resident blocks per SM of the row kernels.  4 x 256 threads leaves 64 registers,
// enough for the software-pipelined group loop without spills (measured at C2 against 8
// blocks / 32 registers with spills: sweep 97 -> 87 us, SOR colour sweep 153 -> 109 us).
// With the value table in shared memory the Jacobi / residual / norm kernels fit 48
// registers without spills, and 5 blocks (40 warps per SM) hide more of the x-gather
// latency: finest sweep 87.9 -> 75.7 us, C2 Jacobi solve 6.66 -> 6.34 ms.  6 blocks (40
// registers) is slower again (89 us), and the colour sweeps lose at 5 (106.5 -> 109.8 us).
#ifndef PF_SOR_MINB
#define PF_SOR_MINB 4
#endif
#ifndef PF_JAC_MINB
#define PF_JAC_MINB 5
#endif
#ifndef PF_ROW_MINB
#define PF_ROW_MINB 5
#endif

// The kernels' value-kind template argument (pf_kernels.cuh): bits 0-2 the stored value
// kind (0 fp64, 1 8-bit index, 2 16-bit index, kVKSmem = 8-bit index with the table staged
// in shared memory), bit 3 (kVKCached) the caching load policy; -1 = read from the view.
constexpr int kVKSmem = 4;
constexpr int kVKCached = 8;
template <int kVK>
constexpr int vk_kind() { return kVK < 0 ? kVK : (kVK & 7); }
template <int kVK>
constexpr bool vk_cached() { return kVK >= 0 && (kVK & kVKCached) != 0; }

// SELL-32x4 layout: slice s holds rows 32s..32s+31; entry j of lane l sits at
//   slice_ptr[s] + (j / 4) * 128 + 4 l + j % 4,
// so a lane reads 4 entries with one 16-byte column load (one 4-byte index / 32-byte value
// load) and a warp's load of one group is one contiguous 512 B (128 B / 1 KB) run.
PF_HD inline int64_t sell_row_base(const int64_t* slice_ptr, int32_t row) {
  return slice_ptr[row >> 5] + (static_cast<int64_t>(row & 31) << 2);
}
PF_HD inline int64_t sell_entry(int64_t row_base, int j) {
  return row_base + (static_cast<int64_t>(j >> 2) << 7) + (j & 3);
}

// SELL-32 operator view.  Values are stored either as fp64 (vkind 0) or, when the matrix
// has few distinct values (a constant-coefficient stencil has 6-8), as 8-bit (vkind 1) or
// 16-bit (vkind 2) indices into a table of the distinct values: lossless, the kernels read
// the exact same doubles, and the finest sweep streams 5 instead of 12 bytes per entry.
struct SellView {
  const double* __restrict__ vals;
  const int32_t* __restrict__ cols;
  const int64_t* __restrict__ slice_ptr;
  const int32_t* __restrict__ row_len;
  const void* __restrict__ vidx;
  const double* __restrict__ table;
  int32_t vkind;
  int32_t table_n;  // distinct values in the table
};

// Block-window view of an operator (pf_window.cuh): for every block of kBlock consecutive
// device rows the x entries its own rows read off the diagonal, covered by runs ("chunks")
// of kWinChunk consecutive doubles, and every stored column re-expressed as a 16-bit byte
// offset into the block's shared-memory window.  The row kernels copy the cover into shared
// memory with coalesced loads and gather from there: a stored entry costs 2 + value bytes
// instead of 4 + value bytes, and the per-entry x gather is a shared-memory read instead
// of an L1/L2 request.
// Window of a block: slots [0, kBlock) belong one to each thread (slot t = the diagonal
// entry of row block * kBlock + t, and the padding entries of its last group): the kernel
// puts there what the diagonal term must read — x_r for the residual-type rows, a signed
// zero for the smoothers, which leave the diagonal term out (a x 0 = +0.0 subtracts as the
// identity); the cover chunks follow, in ascending x order.
constexpr int kWinChunk = 16;
// Largest cover of a block: with the kBlock private slots 40 KB of window per block, so 5
// blocks of 256 threads fit an SM.  A block whose cover is larger keeps an empty chunk
// range and takes the plain row path.
constexpr int kWinChunksCap = 304;
struct WinView {
  const uint16_t* __restrict__ cols16;    // window byte offset of each stored entry's column (A.cols positions)
  const int32_t* __restrict__ chunk_ptr;  // [row blocks + 1] first chunk of each block
  const int32_t* __restrict__ chunks;     // first x index of each chunk; slot = kBlock + 16 * (chunk - first) + offset
  const uint8_t* __restrict__ dpos;       // per own row: position of its diagonal entry in the row
};

// Block schedule of a full-level row kernel (k_jacobi, k_residual).  Own rows sit
// colour-major on the device (each colour in lattice order), so the identity schedule
// sweeps colour 0 over the whole lattice, then colour 1, ...: each colour pass gathers its
// neighbours from all the other colours across the whole x, which on a level whose x
// exceeds L2 (512^3: 1.08 GB) re-reads x from HBM once per colour.  With n_col > 0 the
// blocks instead take chunk k of colour c at block k * n_col + c, so the blocks resident at
// any moment cover one lattice slab of every colour and x streams through L2 about once.
// Rows compute exactly the same values either way (each row is independent).
struct RowMap {
  int32_t n_col;      // 0: identity schedule
  int32_t chunks;     // blocks per colour (the largest colour)
  int32_t start[9];   // colour starts over the own rows; start[n_col] = n_own
};

// The row of this thread under map m (level of n rows, n_own own rows), or -1.
PF_HD inline int32_t map_row(const RowMap& m, int32_t block, int32_t thread, int32_t n_own) {
  if (m.n_col == 0) return block * kBlock + thread;
  const int32_t own_blocks = m.chunks * m.n_col;
  if (block >= own_blocks) return n_own + (block - own_blocks) * kBlock + thread;  // non-own rows
  const int32_t c = block % m.n_col, k = block / m.n_col;
  const int32_t row = m.start[c] + k * kBlock + thread;
  return row < m.start[c + 1] ? row : -1;
}


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
  int32_t max_row;  // longest row (products scratch of the sweep)
  // direct coarse solve (pf_hierarchy_set_coarse_direct), one subdomain: the inverse of the
  // own-own block (n_rows x n_rows, host order) or nullptr for Gauss-Seidel; columns >=
  // n_own_dev are the non-own (Dirichlet) ones
  const double* inv;
  int32_t n_own_dev;
};

PF_HD inline size_t coarse_pack_smem(const CoarsePack& P) {
  const size_t scratch = static_cast<size_t>(P.max_row > P.n_rows ? P.max_row : P.n_rows);
  return sizeof(double) * (static_cast<size_t>(P.n_total) + 2 * static_cast<size_t>(P.n_rows) + P.nnz + scratch + 1) +
         sizeof(int32_t) * (static_cast<size_t>(P.n_rows) * 3 + 1 + P.nnz + P.n_sub + 1 +
                            2 * static_cast<size_t>(P.ms_n) + 2 * static_cast<size_t>(P.h1_n));
}

}  // namespace pf
