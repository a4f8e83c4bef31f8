// pf_kernels.cuh — sm_100a kernels of the GMG V-cycle hot path.
//
// Storage: every level operator is SELL-32x4 (pf_types.hpp) — slices of 32 consecutive
// device rows; inside a slice entry j of lane l sits at slice_ptr[s] + 128 (j/4) + 4 l +
// j%4, so a lane reads four entries of its row with one 16-byte column load and a warp's
// load of one group of four is one contiguous 512 B run.  Values are an 8/16-bit index into
// a table of the operator's distinct doubles when it has at most 256/65,536 of them
// (lossless; the table is staged in shared memory), else fp64: 4 + 1 B per entry for the
// constant-coefficient Q1 stencil, 4 + 8 B with a per-cell coefficient.  Entries of a row
// keep the reference's CSR order (linalg.hpp:12-22), which fixes the summation order.
//
// Arithmetic: every product and sum is rounded separately (__dmul_rn / __dadd_rn /
// __dsub_rn / __ddiv_rn, never an FMA), reproducing the reference's x86-64 SSE2
// evaluation of the same expressions, so Jacobi iterates match bit for bit.
//
// HBM behaviour: the finest operator is streamed once per sweep with evict-first loads
// (plus a row-start L2 prefetch of its groups); the operators of coarser levels that fit
// L2 are read with the caching policy and stay resident across a cycle's sweeps; the x
// gather goes through the read-only path and stays L2-resident (17 MB at 128^3; on levels
// whose x outgrows L2 the colour-interleaved block schedule, RowMap, keeps it streaming
// through L2 once per sweep).
#pragma once

#include <cstdint>

#include "pf_types.hpp"

namespace pf {

// Programmatic dependent launch: every kernel of the chain waits for its predecessor's
// memory (griddepcontrol.wait — a no-op when launched without the PDL attribute) and then
// lets its own successor's blocks be scheduled, so launch latency overlaps the previous
// kernel's tail instead of adding to it.
#define PF_PDL_ENTRY()                                         \
  do {                                                         \
    asm volatile("griddepcontrol.wait;" ::: "memory");         \
    asm volatile("griddepcontrol.launch_dependents;" :::);     \
  } while (0)

// The kernels' value-kind template argument kVK: bits 0-2 the stored value kind (0 fp64,
// 1 8-bit index, 2 16-bit index, kVKSmem = 8-bit index with the table staged in shared
// memory by the kernel's prologue, vtab_stage, so the per-entry value lookup is a
// shared-memory broadcast instead of an L1 request competing with the x gathers), bit 3
// (kVKCached) the operator-stream load policy; -1 = everything read from the view.
//   * evict-first (ld.global.cs): levels whose operator is far larger than L2 (the finest
//     levels) are streamed once per sweep and must not push x out of L2;
//   * cached (ld.global.nc): the coarser levels whose operator fits L2 are re-read by every
//     sweep of the cycle and keep living there (C2: Jacobi solve 6.33 -> 6.21 ms, SOR
//     11.57 -> 10.91 ms).  Measured without gain: L1::no_allocate loads (Jacobi 6.37 ms,
//     SOR unchanged), plus an L2::evict_last cache policy (6.38 ms); caching the finest
//     level of a 64^3 hierarchy, whose 39 MB operator also fits, costs 6 %.
// (kVKSmem, kVKCached, vk_kind, vk_cached: pf_types.hpp, shared with the host dispatch)
static __shared__ double s_vtab[256];

// Resident blocks per SM of a row kernel: `minb` (pf_types.hpp), except for the streamed
// fp64 operators (kVK == 0: the per-cell-coefficient finest levels, at the HBM roofline),
// which keep 4 blocks / 64 registers (measured: lognormal C2 sweep 114 us at 4, 117 at 5),
// and the cached (L2-resident, coarser) operators: PF_CACHED_MINB = 4 (C2 Jacobi solve
// 5.78 -> 5.74 ms; 6 or 8 blocks: 6.24 ms).
#ifndef PF_CACHED_MINB
#define PF_CACHED_MINB 4
#endif
template <int kVK>
constexpr int minb_for(int minb) {
  return kVK == 0 ? 4 : (PF_CACHED_MINB > 0 && vk_cached<kVK>()) ? PF_CACHED_MINB : minb;
}

template <int kVK>
__device__ __forceinline__ void vtab_stage(const SellView& A) {
  if constexpr (vk_kind<kVK>() == kVKSmem) {
    for (int i = threadIdx.x; i < A.table_n; i += blockDim.x) s_vtab[i] = A.table[i];
    __syncthreads();
  }
}

#ifndef PF_LD_OP
#define PF_LD_OP __ldcs
#endif
template <int kVK, typename T>
__device__ __forceinline__ T ld_op(const T* p) {
  if constexpr (vk_cached<kVK>())
    return __ldg(p);
  else
    return PF_LD_OP(p);
}

// L2 prefetch of a row's groups 1..kPf (columns and value indices) at the start of the row,
// so the software-pipelined loop's loads find them in L2 without holding registers.  Only
// for the streamed (evict-first) index-valued operators, in the Jacobi / residual / norm kernels
// (measured at C2: 6 groups = a whole Q1 row, finest sweep 75.7 -> 73.9 us, Jacobi solve
// 6.18 -> 6.09 ms; the colour sweeps lose with it, 106.5 -> 117.9 us).
#ifndef PF_PREFETCH_GROUPS
#define PF_PREFETCH_GROUPS 6
#endif
constexpr int kPrefetch = PF_PREFETCH_GROUPS;
template <int kVK, int kPf>
__device__ __forceinline__ void row_prefetch(const SellView& A, int64_t base, int len) {
  if constexpr (kPf > 0 && !vk_cached<kVK>() && kVK > 0) {
    const int ng = (len + 3) / 4;
#pragma unroll
    for (int g = 1; g <= kPf; ++g) {
      if (g < ng) {
        const int64_t e = sell_entry(base, 4 * g);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(A.cols + e));
        if constexpr (vk_kind<kVK>() == 1 || vk_kind<kVK>() == kVKSmem)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(static_cast<const unsigned char*>(A.vidx) + e));
      }
    }
  }
}

// Value of stored entry e.  kVK = the view's value kind when known at compile time (the
// bandwidth kernels are instantiated per kind), -1 = read it from the view.
template <int kVK>
__device__ __forceinline__ double sell_val(const SellView& A, int64_t e) {
  constexpr int K = vk_kind<kVK>();
  if constexpr (K == 0) {
    return ld_op<kVK>(A.vals + e);
  } else if constexpr (K == 1) {
    return __ldg(A.table + ld_op<kVK>(static_cast<const unsigned char*>(A.vidx) + e));
  } else if constexpr (K == kVKSmem) {
    return s_vtab[ld_op<kVK>(static_cast<const unsigned char*>(A.vidx) + e)];
  } else if constexpr (K == 2) {
    return __ldg(A.table + ld_op<kVK>(static_cast<const unsigned short*>(A.vidx) + e));
  } else {
    if (A.vkind == 1) return __ldg(A.table + static_cast<const unsigned char*>(A.vidx)[e]);
    if (A.vkind == 2) return __ldg(A.table + static_cast<const unsigned short*>(A.vidx)[e]);
    return A.vals[e];
  }
}

// One group of 4 stored entries (SELL-32x4) starting at e (e % 4 == 0): columns and values.
template <int kVK>
__device__ __forceinline__ void sell_group_vals(const SellView& A, int64_t e, double v[4]);
template <int kVK>
__device__ __forceinline__ void sell_group(const SellView& A, int64_t e, int32_t c[4], double v[4]) {
  const int4 cc = ld_op<kVK>(reinterpret_cast<const int4*>(A.cols + e));
  c[0] = cc.x;
  c[1] = cc.y;
  c[2] = cc.z;
  c[3] = cc.w;
  sell_group_vals<kVK>(A, e, v);
}
// The four values of the group starting at e.
template <int kVK>
__device__ __forceinline__ void sell_group_vals(const SellView& A, int64_t e, double v[4]) {
  constexpr int K = vk_kind<kVK>();
  if constexpr (K == 1) {
    const unsigned int w = ld_op<kVK>(reinterpret_cast<const unsigned int*>(static_cast<const unsigned char*>(A.vidx) + e));
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __ldg(A.table + ((w >> (8 * k)) & 255u));
  } else if constexpr (K == kVKSmem) {
    const unsigned int w = ld_op<kVK>(reinterpret_cast<const unsigned int*>(static_cast<const unsigned char*>(A.vidx) + e));
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = s_vtab[(w >> (8 * k)) & 255u];
  } else if constexpr (K == 2) {
    const uint2 w = ld_op<kVK>(reinterpret_cast<const uint2*>(static_cast<const unsigned short*>(A.vidx) + e));
    v[0] = __ldg(A.table + (w.x & 0xffffu));
    v[1] = __ldg(A.table + (w.x >> 16));
    v[2] = __ldg(A.table + (w.y & 0xffffu));
    v[3] = __ldg(A.table + (w.y >> 16));
  } else if constexpr (K == 0) {
    const double2 a = ld_op<kVK>(reinterpret_cast<const double2*>(A.vals + e));
    const double2 b = ld_op<kVK>(reinterpret_cast<const double2*>(A.vals + e + 2));
    v[0] = a.x;
    v[1] = a.y;
    v[2] = b.x;
    v[3] = b.y;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = sell_val<-1>(A, e + k);
  }
}

// A group as loaded, before its values are looked up: the software-pipelined loops hold the
// NEXT group in this form (5 registers for an 8-bit operator instead of 12 decoded) and
// decode it after the current group's arithmetic.  Measured at C2 (bit-identical): finest
// Jacobi sweep 74.8 -> 73.4 us, Jacobi solve 5.444 -> 5.428 ms, SOR 9.539 -> 9.527 ms.  The
// registers it frees do not buy occupancy: 6 blocks/SM (40 registers, no spills now) 75.7 us;
// two raw groups in flight instead of the L2 prefetch 84.4 us, with it 79.1 us.
#ifndef PF_RAW_PIPE
#define PF_RAW_PIPE 1
#endif
struct SellRaw {
  int4 cc;
  uint32_t w0, w1;
  double v[4];
};
template <int kVK>
__device__ __forceinline__ void sell_load(const SellView& A, int64_t e, SellRaw& r) {
  constexpr int K = vk_kind<kVK>();
  r.cc = ld_op<kVK>(reinterpret_cast<const int4*>(A.cols + e));
  if constexpr (K == 1 || K == kVKSmem) {
    r.w0 = ld_op<kVK>(reinterpret_cast<const unsigned int*>(static_cast<const unsigned char*>(A.vidx) + e));
  } else if constexpr (K == 2) {
    const uint2 w = ld_op<kVK>(reinterpret_cast<const uint2*>(static_cast<const unsigned short*>(A.vidx) + e));
    r.w0 = w.x;
    r.w1 = w.y;
  } else {
    sell_group_vals<kVK>(A, e, r.v);
  }
}
template <int kVK>
__device__ __forceinline__ void sell_decode(const SellView& A, const SellRaw& r, int32_t c[4], double v[4]) {
  constexpr int K = vk_kind<kVK>();
  c[0] = r.cc.x;
  c[1] = r.cc.y;
  c[2] = r.cc.z;
  c[3] = r.cc.w;
  if constexpr (K == 1) {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __ldg(A.table + ((r.w0 >> (8 * k)) & 255u));
  } else if constexpr (K == kVKSmem) {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = s_vtab[(r.w0 >> (8 * k)) & 255u];
  } else if constexpr (K == 2) {
    v[0] = __ldg(A.table + (r.w0 & 0xffffu));
    v[1] = __ldg(A.table + (r.w0 >> 16));
    v[2] = __ldg(A.table + (r.w1 & 0xffffu));
    v[3] = __ldg(A.table + (r.w1 >> 16));
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = r.v[k];
  }
}

// acc := acc - sum_{c != row} a_rc x_c over the row's entries in stored order; diag := a_rr.
// This is the inner loop of one_local_sweep (solvers.cpp:21-51).  Entries are consumed a
// group of 4 at a time (one 16-byte column load, one index / value load, four x gathers),
// the next group's column and value loads issued before the current group's arithmetic;
// the last, partial group is predicated (entries past the row length are padding).
template <bool kReadOnlyX, bool kRes>
__device__ __forceinline__ void offdiag_group(const int32_t c[4], const double v[4], int n, int32_t row,
                                              const double* x, double x_row, double& acc, double& diag,
                                              double& r) {
  double xv[4];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    xv[k] = (k >= n || c[k] == row) ? x_row : (kReadOnlyX ? __ldg(x + c[k]) : x[c[k]]);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k < n) {
      const double p = __dmul_rn(v[k], xv[k]);
      if (kRes) r = __dsub_rn(r, p);
      if (c[k] == row)
        diag = v[k];
      else
        acc = __dsub_rn(acc, p);
    }
  }
}

// The x-independent start of a row: its SELL base, length and first group of columns and
// values (plus the L2 prefetch of the rest).  The operator never changes after upload, so
// the colour sweep issues this BEFORE griddepcontrol.wait: under programmatic dependent
// launch those loads overlap the previous colour's tail instead of opening this one's
// dependency chain (C2 SOR solve 10.63 -> 10.21 ms; the Jacobi sweep, whose predecessor
// is itself bandwidth-heavy, loses with it: 75.0 -> 79.4 us, so it keeps the plain order).
struct RowHead {
  int64_t base;
  int len;
  int32_t c[4];
  double v[4];
};
template <int kVK, int kPf = 0>
__device__ __forceinline__ void row_head(const SellView& A, int32_t row, RowHead& h) {
  h.base = sell_row_base(A.slice_ptr, row);
  h.len = A.row_len[row];
  row_prefetch<kVK, kPf>(A, h.base, h.len);
  if (h.len > 0) sell_group<kVK>(A, h.base, h.c, h.v);
}

// The rest of row_offdiag from a RowHead.
template <bool kReadOnlyX, bool kRes = false, int kVK = -1>
__device__ __forceinline__ void row_offdiag_from(const SellView& A, const RowHead& h, int32_t row, const double* x,
                                                 double& acc, double& diag, double* res = nullptr,
                                                 double x_row = 0.0) {
  double r = kRes ? *res : 0.0;
  const int len = h.len;
  if (len > 0) {
    int32_t c[4];
    double v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      c[k] = h.c[k];
      v[k] = h.v[k];
    }
    int j = 0;
    for (; j + 4 < len; j += 4) {
#if PF_RAW_PIPE
      SellRaw nx;
      sell_load<kVK>(A, sell_entry(h.base, j + 4), nx);
      offdiag_group<kReadOnlyX, kRes>(c, v, 4, row, x, x_row, acc, diag, r);
      sell_decode<kVK>(A, nx, c, v);
#else
      int32_t cn[4];
      double vn[4];
      sell_group<kVK>(A, sell_entry(h.base, j + 4), cn, vn);
      offdiag_group<kReadOnlyX, kRes>(c, v, 4, row, x, x_row, acc, diag, r);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        c[k] = cn[k];
        v[k] = vn[k];
      }
#endif
    }
    offdiag_group<kReadOnlyX, kRes>(c, v, len - j, row, x, x_row, acc, diag, r);
  }
  if (kRes) *res = r;
}

template <bool kReadOnlyX, bool kRes = false, int kVK = -1, int kGroups = kChunkGroups, int kPf = 0>
__device__ __forceinline__ void row_offdiag(const SellView& A, int32_t row, const double* x,
                                            double& acc, double& diag, double* res = nullptr,
                                            double x_row = 0.0) {
  // kRes: *res (starting at b_r) also subtracts every product in stored order, the
  // diagonal included — the reference's residual_norm row (linalg.cpp:66-70) bit for bit.
  RowHead h;
  row_head<kVK, kPf>(A, row, h);
  row_offdiag_from<kReadOnlyX, kRes, kVK>(A, h, row, x, acc, diag, res, x_row);
}

// acc := acc op sum_c a_rc x_c over all entries in stored order.
//   kSubtract: acc -= a x   (residual_norm, linalg.cpp:64-73: acc starts at b)
//   else:      acc += a x   (spmv, linalg.cpp:49-56: acc starts at 0)
template <bool kSubtract, bool kReadOnlyX>
__device__ __forceinline__ void dot_group(const int32_t c[4], const double v[4], int n, const double* x,
                                          double& acc) {
  double xv[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) xv[k] = k < n ? (kReadOnlyX ? __ldg(x + c[k]) : x[c[k]]) : 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (k < n) acc = kSubtract ? __dsub_rn(acc, __dmul_rn(v[k], xv[k])) : __dadd_rn(acc, __dmul_rn(v[k], xv[k]));
}

// The rest of row_dot from a RowHead (row_head issued before griddepcontrol.wait).
template <bool kSubtract, bool kReadOnlyX = true, int kVK = -1>
__device__ __forceinline__ double row_dot_from(const SellView& A, const RowHead& h, const double* __restrict__ x,
                                               double acc) {
  const int len = h.len;
  if (len > 0) {
    int32_t c[4];
    double v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      c[k] = h.c[k];
      v[k] = h.v[k];
    }
    int j = 0;
    for (; j + 4 < len; j += 4) {
#if PF_RAW_PIPE
      SellRaw nx;
      sell_load<kVK>(A, sell_entry(h.base, j + 4), nx);
      dot_group<kSubtract, kReadOnlyX>(c, v, 4, x, acc);
      sell_decode<kVK>(A, nx, c, v);
#else
      int32_t cn[4];
      double vn[4];
      sell_group<kVK>(A, sell_entry(h.base, j + 4), cn, vn);
      dot_group<kSubtract, kReadOnlyX>(c, v, 4, x, acc);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        c[k] = cn[k];
        v[k] = vn[k];
      }
#endif
    }
    dot_group<kSubtract, kReadOnlyX>(c, v, len - j, x, acc);
  }
  return acc;
}

// Which row kernels issue their operator-only row start before griddepcontrol.wait
// (PF_HEAD_EARLY, compile time): 0 the colour sweeps only, 1 also the kernels of the cached
// (coarser, L2-resident) operators, 2 every row kernel.
#ifndef PF_HEAD_EARLY
#define PF_HEAD_EARLY 1
#endif
template <int kVK>
constexpr bool head_early() {
  return PF_HEAD_EARLY >= 2 || (PF_HEAD_EARLY == 1 && vk_cached<kVK>());
}

template <bool kSubtract, bool kReadOnlyX = true, int kVK = -1, int kGroups = kChunkGroups, int kPf = kPrefetch>
__device__ __forceinline__ double row_dot(const SellView& A, int32_t row, const double* __restrict__ x,
                                          double acc) {
  const int64_t base = sell_row_base(A.slice_ptr, row);
  const int len = A.row_len[row];
  row_prefetch<kVK, kPf>(A, base, len);
  if (len > 0) {
    int32_t c[4];
    double v[4];
    sell_group<kVK>(A, base, c, v);
    int j = 0;
    for (; j + 4 < len; j += 4) {
#if PF_RAW_PIPE
      SellRaw nx;
      sell_load<kVK>(A, sell_entry(base, j + 4), nx);
      dot_group<kSubtract, kReadOnlyX>(c, v, 4, x, acc);
      sell_decode<kVK>(A, nx, c, v);
#else
      int32_t cn[4];
      double vn[4];
      sell_group<kVK>(A, sell_entry(base, j + 4), cn, vn);
      dot_group<kSubtract, kReadOnlyX>(c, v, 4, x, acc);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        c[k] = cn[k];
        v[k] = vn[k];
      }
#endif
    }
    dot_group<kSubtract, kReadOnlyX>(c, v, len - j, x, acc);
  }
  return acc;
}

// Damped Jacobi sweep (solvers.cpp:35-51) with ping-pong buffers instead of the
// reference's full scratch copy: own rows [0, n_own) are relaxed from x_old into
// x_new; every other row is carried over unchanged (the sweep never writes Slave,
// Halo or Dirichlet entries, solvers.hpp:16-20).
template <int kVK>
__global__ void __launch_bounds__(kBlock, minb_for<kVK>(PF_JAC_MINB)) k_jacobi(SellView A, const double* __restrict__ x_old,
                                                   double* __restrict__ x_new,
                                                   const double* __restrict__ b, int32_t n_own,
                                                   int32_t n, double omega, RowMap map) {
  vtab_stage<kVK>(A);
  const int32_t row = map_row(map, blockIdx.x, threadIdx.x, n_own);
  RowHead hd;
  if constexpr (head_early<kVK>())
    if (row >= 0 && row < n_own) row_head<kVK, kPrefetch>(A, row, hd);
  PF_PDL_ENTRY();
  if (row < 0 || row >= n) return;
  const double xo = x_old[row];
  if (row >= n_own) {
    x_new[row] = xo;
    return;
  }
  double acc = b[row], diag = 0.0;
  if constexpr (head_early<kVK>())
    row_offdiag_from<true, false, kVK>(A, hd, row, x_old, acc, diag);
  else
    row_offdiag<true, false, kVK, kChunkGroups, kPrefetch>(A, row, x_old, acc, diag);
  x_new[row] = __dadd_rn(__dmul_rn(1.0 - omega, xo), __ddiv_rn(__dmul_rn(omega, acc), diag));
}

// The two halves of a multi-process damped-Jacobi sweep whose exchange overlaps the
// interior rows (same per-row arithmetic as k_jacobi): the boundary rows from a list plus
// the carry-over of the non-own rows, then the interior own rows.
template <int kVK>
__global__ void __launch_bounds__(kBlock, minb_for<kVK>(PF_JAC_MINB)) k_jacobi_boundary(SellView A, const int32_t* __restrict__ list,
                                                                    int32_t n_list, const double* __restrict__ x_old,
                                                                    double* __restrict__ x_new,
                                                                    const double* __restrict__ b, int32_t n_own,
                                                                    int32_t n, double omega) {
  vtab_stage<kVK>(A);
  PF_PDL_ENTRY();
  const int32_t nb_blocks = max(1, (n_list + kBlock - 1) / kBlock);
  if (static_cast<int32_t>(blockIdx.x) >= nb_blocks) {  // non-own rows: carried over
    const int32_t row = n_own + (static_cast<int32_t>(blockIdx.x) - nb_blocks) * kBlock + threadIdx.x;
    if (row < n) x_new[row] = x_old[row];
    return;
  }
  const int32_t i = blockIdx.x * kBlock + threadIdx.x;
  if (i >= n_list) return;
  const int32_t row = list[i];
  double acc = b[row], diag = 0.0;
  row_offdiag<true, false, kVK, kChunkGroups, kPrefetch>(A, row, x_old, acc, diag);
  x_new[row] = __dadd_rn(__dmul_rn(1.0 - omega, x_old[row]), __ddiv_rn(__dmul_rn(omega, acc), diag));
}

template <int kVK>
__global__ void __launch_bounds__(kBlock, minb_for<kVK>(PF_JAC_MINB)) k_jacobi_interior(SellView A, const uint8_t* __restrict__ is_b,
                                                                    const double* __restrict__ x_old,
                                                                    double* __restrict__ x_new,
                                                                    const double* __restrict__ b, int32_t n_own,
                                                                    double omega) {
  vtab_stage<kVK>(A);
  PF_PDL_ENTRY();
  const int32_t row = blockIdx.x * kBlock + threadIdx.x;
  if (row >= n_own || is_b[row]) return;
  double acc = b[row], diag = 0.0;
  row_offdiag<true, false, kVK, kChunkGroups, kPrefetch>(A, row, x_old, acc, diag);
  x_new[row] = __dadd_rn(__dmul_rn(1.0 - omega, x_old[row]), __ddiv_rn(__dmul_rn(omega, acc), diag));
}

// State of a device-driven solve_outer (multigrid.cpp:210-246).
struct SolveState {
  double r0;
  double last;
  int32_t launches;  // outer iterations started (the norm just computed is of x_{launches})
  int32_t stop;
  int32_t converged;
  int32_t pad;
  double hist[1];  // [outer_max_cycles]
};

// The convergence test of solve_outer on the device: the ascending-rank sum of the
// per-subdomain squares (transport.cpp:139-149) gives ||b - A x_m||; m = 0 records r0,
// m >= 1 records the residual after cycle m and stops at <= tol * r0 or after max cycles.
// Sets the WHILE (next iteration) and IF (rest of the cycle) conditions of the graph.
static __global__ void k_decide(const double* __restrict__ sumsq, int n_parts, double tol, int max_cycles,
                         SolveState* st, cudaGraphConditionalHandle h_while,
                         cudaGraphConditionalHandle h_if) {
  PF_PDL_ENTRY();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0;
  for (int i = 0; i < n_parts; ++i) s = __dadd_rn(s, sumsq[i]);
  const double norm = sqrt(s);
  const int m = st->launches;
  int stop, conv;
  if (m == 0) {
    st->r0 = norm;
    conv = norm == 0.0;
    stop = conv;
  } else {
    st->hist[m - 1] = norm;
    conv = norm <= __dmul_rn(tol, st->r0);
    stop = conv || m >= max_cycles;
  }
  st->last = norm;
  st->launches = m + 1;
  st->stop = stop;
  st->converged = conv;
  cudaGraphSetConditional(h_while, stop ? 0u : 1u);
  if (h_if != h_while) cudaGraphSetConditional(h_if, stop ? 0u : 1u);
}

// One colour of multicolour Gauss-Seidel / SOR, in place, rows [row0, row1).  Rows of
// one colour never couple, so the result does not depend on the order in which the
// threads of this launch run.  kSor=false: x = acc/diag (solvers.cpp:21-34);
// kSor=true: x = (1-w) x + w acc/diag.
template <bool kSor, int kVK>
__global__ void __launch_bounds__(kBlock, PF_SOR_MINB) k_color_sweep(SellView A, double* x,
                                                        const double* __restrict__ b, int32_t row0,
                                                        int32_t row1, double omega) {
  vtab_stage<kVK>(A);
  const int32_t row = row0 + blockIdx.x * kBlock + threadIdx.x;
  RowHead hd;
  if (row < row1) row_head<kVK>(A, row, hd);  // operator only: before the wait
  PF_PDL_ENTRY();
  if (row >= row1) return;
  double acc = b[row], diag = 0.0;
  // Other colours are read-only during this launch and this row's own entry is
  // skipped by row_offdiag, so the read-only path is safe for the gather.
  row_offdiag_from<true, false, kVK>(A, hd, row, x, acc, diag);
  if (kSor)
    x[row] = __dadd_rn(__dmul_rn(1.0 - omega, x[row]), __ddiv_rn(__dmul_rn(omega, acc), diag));
  else
    x[row] = __ddiv_rn(acc, diag);
}

// The two halves of the last colour of a multi-process coloured sweep whose exchange
// overlaps the interior rows (same per-row arithmetic as k_color_sweep): the rows in `list`
// (those that send or read a non-own copy), then the other rows of [row0, row1).
template <bool kSor, int kVK>
__global__ void __launch_bounds__(kBlock, PF_SOR_MINB) k_color_sweep_list(SellView A, double* x,
                                                             const double* __restrict__ b,
                                                             const int32_t* __restrict__ list, int32_t n_list,
                                                             double omega) {
  vtab_stage<kVK>(A);
  PF_PDL_ENTRY();
  const int32_t i = blockIdx.x * kBlock + threadIdx.x;
  if (i >= n_list) return;
  const int32_t row = list[i];
  double acc = b[row], diag = 0.0;
  row_offdiag<true, false, kVK>(A, row, x, acc, diag);
  if (kSor)
    x[row] = __dadd_rn(__dmul_rn(1.0 - omega, x[row]), __ddiv_rn(__dmul_rn(omega, acc), diag));
  else
    x[row] = __ddiv_rn(acc, diag);
}
template <bool kSor, int kVK>
__global__ void __launch_bounds__(kBlock, PF_SOR_MINB) k_color_sweep_skip(SellView A, double* x,
                                                             const double* __restrict__ b, int32_t row0,
                                                             int32_t row1, const uint8_t* __restrict__ skip,
                                                             double omega) {
  vtab_stage<kVK>(A);
  const int32_t row = row0 + blockIdx.x * kBlock + threadIdx.x;
  const bool act = row < row1 && !skip[row];
  RowHead hd;
  if (act) row_head<kVK>(A, row, hd);  // operator only: before the wait
  PF_PDL_ENTRY();
  if (!act) return;
  double acc = b[row], diag = 0.0;
  row_offdiag_from<true, false, kVK>(A, hd, row, x, acc, diag);
  if (kSor)
    x[row] = __dadd_rn(__dmul_rn(1.0 - omega, x[row]), __ddiv_rn(__dmul_rn(omega, acc), diag));
  else
    x[row] = __ddiv_rn(acc, diag);
}

// k_color_sweep for long rows: one block per SELL slice (32 rows), kSplitBlock / 32 warps.
// Warp w loads groups w, w + 8, ... of all 32 rows (coalesced, as the row kernel's single
// warp would), gathers x and forms the products a_e x_c into shared memory (entry-major,
// conflict-free); then warp 0 — lane = row — subtracts them in stored order, skipping the
// diagonal, and applies the update.  Same operations in the same order as k_color_sweep.
constexpr int kSplitBlock = 256;
template <bool kSor, int kVK>
__global__ void __launch_bounds__(kSplitBlock) k_color_sweep_split(SellView A, double* x, const double* __restrict__ b,
                                                                  int32_t row0, int32_t row1, double omega,
                                                                  int32_t width) {
  extern __shared__ double prod[];  // [width][32]
  __shared__ double sdiag[32];
  __shared__ int32_t sdpos[32];
  vtab_stage<kVK>(A);
  PF_PDL_ENTRY();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int32_t slice = (row0 >> 5) + static_cast<int32_t>(blockIdx.x);
  const int32_t row = slice * 32 + lane;
  const bool active = row >= row0 && row < row1;
  const int len = active ? A.row_len[row] : 0;
  if (w == 0) {
    sdpos[lane] = -1;
    sdiag[lane] = 0.0;
  }
  __syncthreads();
  const int64_t base = A.slice_ptr[slice] + 4 * lane;
  for (int g = w; 4 * g < len; g += kSplitBlock / 32) {
    int32_t c[4];
    double v[4];
    sell_group<kVK>(A, base + 128 * static_cast<int64_t>(g), c, v);
    double xv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) xv[k] = (4 * g + k < len && c[k] != row) ? __ldg(x + c[k]) : 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = 4 * g + k;
      if (j < len) {
        if (c[k] == row) {
          sdpos[lane] = j;
          sdiag[lane] = v[k];
        } else {
          prod[j * 32 + lane] = __dmul_rn(v[k], xv[k]);
        }
      }
    }
  }
  __syncthreads();
  if (w != 0 || !active) return;
  const int dp = sdpos[lane];
  double acc = b[row];
  for (int j = 0; j < len; ++j)
    if (j != dp) acc = __dsub_rn(acc, prod[j * 32 + lane]);
  const double diag = sdiag[lane];
  if (kSor)
    x[row] = __dadd_rn(__dmul_rn(1.0 - omega, x[row]), __ddiv_rn(__dmul_rn(omega, acc), diag));
  else
    x[row] = __ddiv_rn(acc, diag);
}

// The slice-split form of the damped-Jacobi sweep (kJacobi) and of the cycle residual for
// long rows on small levels (Q2: up to 125 entries), where one thread per row walks a
// 32-group dependent chain: warp w of the slice's block forms the products of groups w,
// w + 8, ... into shared memory, then lane r of warp 0 sums row r's products in stored
// order — Jacobi: b_r minus the off-diagonal products, as k_jacobi; residual: the spmv sum
// from 0 over every entry, r = b - sum, as k_residual.  Rows [0, n); Jacobi carries the
// non-own rows over.
template <bool kJacobi, int kVK>
__global__ void __launch_bounds__(kSplitBlock) k_rows_split(SellView A, const double* __restrict__ x,
                                                           double* __restrict__ out, const double* __restrict__ b,
                                                           int32_t n_own, int32_t n, double omega) {
  extern __shared__ double prod[];  // [width][32]
  __shared__ double sdiag[32];
  __shared__ int32_t sdpos[32];
  vtab_stage<kVK>(A);
  PF_PDL_ENTRY();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int32_t slice = static_cast<int32_t>(blockIdx.x);
  const int32_t row = slice * 32 + lane;
  const bool active = row < n && (!kJacobi || row < n_own);
  const int len = active ? A.row_len[row] : 0;
  if (w == 0) {
    sdpos[lane] = -1;
    sdiag[lane] = 0.0;
  }
  __syncthreads();
  const int64_t base = A.slice_ptr[slice] + 4 * lane;
  for (int g = w; 4 * g < len; g += kSplitBlock / 32) {
    int32_t c[4];
    double v[4];
    sell_group<kVK>(A, base + 128 * static_cast<int64_t>(g), c, v);
    double xv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) xv[k] = (4 * g + k < len && (!kJacobi || c[k] != row)) ? __ldg(x + c[k]) : 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = 4 * g + k;
      if (j < len) {
        if (kJacobi && c[k] == row) {
          sdpos[lane] = j;
          sdiag[lane] = v[k];
        } else {
          prod[j * 32 + lane] = __dmul_rn(v[k], xv[k]);
        }
      }
    }
  }
  __syncthreads();
  if (w != 0 || row >= n) return;
  if (kJacobi) {
    const double xo = x[row];
    if (row >= n_own) {
      out[row] = xo;
      return;
    }
    const int dp = sdpos[lane];
    double acc = b[row];
    for (int j = 0; j < len; ++j)
      if (j != dp) acc = __dsub_rn(acc, prod[j * 32 + lane]);
    out[row] = __dadd_rn(__dmul_rn(1.0 - omega, xo), __ddiv_rn(__dmul_rn(omega, acc), sdiag[lane]));
  } else {
    double acc = 0.0;
    for (int j = 0; j < len; ++j) acc = __dadd_rn(acc, prod[j * 32 + lane]);
    out[row] = __dsub_rn(b[row], acc);
  }
}

// "Wide" rows for launches that fit one wave (the mid-size levels of a cycle, where a
// launch is bound by the latency chain of one row, not by throughput): the whole row's
// operator — every group of 4 columns and its 8-bit value indices — is loaded into
// registers BEFORE griddepcontrol.wait (the operator is immutable, so those loads overlap
// the previous kernel's tail), and after the wait all of the row's x gathers are issued at
// once: one dependent memory round trip instead of one per group.  The products are then
// formed and subtracted in stored order, the diagonal skipped, exactly as row_offdiag does.
// kG groups (Q1: 27 entries -> 7); rows longer than 4 kG never take these kernels.
template <int kG>
struct RowWide {
  int len;
  int32_t c[4 * kG];
  uint32_t w[kG];  // 4 value indices per word, entry j in byte j % 4 of word j / 4
};

template <int kVK, int kG>
__device__ __forceinline__ void row_wide_head(const SellView& A, int32_t row, RowWide<kG>& h) {
  static_assert(vk_kind<kVK>() == 1 || vk_kind<kVK>() == kVKSmem, "wide rows: 8-bit value indices only");
  const int64_t base = sell_row_base(A.slice_ptr, row);
  h.len = A.row_len[row];
#pragma unroll
  for (int g = 0; g < kG; ++g) {
    if (4 * g < h.len) {
      const int64_t e = sell_entry(base, 4 * g);
      const int4 cc = ld_op<kVK>(reinterpret_cast<const int4*>(A.cols + e));
      h.c[4 * g] = cc.x;
      h.c[4 * g + 1] = cc.y;
      h.c[4 * g + 2] = cc.z;
      h.c[4 * g + 3] = cc.w;
      h.w[g] = ld_op<kVK>(reinterpret_cast<const unsigned int*>(static_cast<const unsigned char*>(A.vidx) + e));
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) h.c[4 * g + k] = -1;
      h.w[g] = 0;
    }
  }
}

template <int kVK>
__device__ __forceinline__ double wide_val(const SellView& A, uint32_t w, int k) {
  const uint32_t i = (w >> (8 * k)) & 255u;
  if constexpr (vk_kind<kVK>() == kVKSmem)
    return s_vtab[i];
  else
    return __ldg(A.table + i);
}

// acc := acc - sum_{c != row} a_rc x_c in stored order, diag := a_rr (row_offdiag's result).
template <int kVK, int kG>
__device__ __forceinline__ void row_wide_offdiag(const SellView& A, const RowWide<kG>& h, int32_t row,
                                                 const double* __restrict__ x, double& acc, double& diag) {
  double xv[4 * kG];
#pragma unroll
  for (int j = 0; j < 4 * kG; ++j) xv[j] = (j < h.len && h.c[j] != row) ? __ldg(x + h.c[j]) : 0.0;
#pragma unroll
  for (int j = 0; j < 4 * kG; ++j) {
    if (j < h.len) {
      const double v = wide_val<kVK>(A, h.w[j >> 2], j & 3);
      if (h.c[j] == row)
        diag = v;
      else
        acc = __dsub_rn(acc, __dmul_rn(v, xv[j]));
    }
  }
}

#ifndef PF_WIDE_MINB
#define PF_WIDE_MINB 2
#endif
template <bool kSor, int kVK, int kG>
__global__ void __launch_bounds__(kBlock, PF_WIDE_MINB) k_color_sweep_wide(SellView A, double* x,
                                                                    const double* __restrict__ b, int32_t row0,
                                                                    int32_t row1, double omega) {
  vtab_stage<kVK>(A);
  const int32_t row = row0 + blockIdx.x * kBlock + threadIdx.x;
  RowWide<kG> hd;
  if (row < row1) row_wide_head<kVK, kG>(A, row, hd);  // operator only: before the wait
  PF_PDL_ENTRY();
  if (row >= row1) return;
  const double bb = b[row];
  const double xo = kSor ? x[row] : 0.0;
  double acc = bb, diag = 0.0;
  row_wide_offdiag<kVK, kG>(A, hd, row, x, acc, diag);
  if (kSor)
    x[row] = __dadd_rn(__dmul_rn(1.0 - omega, xo), __ddiv_rn(__dmul_rn(omega, acc), diag));
  else
    x[row] = __ddiv_rn(acc, diag);
}

// k_jacobi with wide rows (identity block schedule).
template <int kVK, int kG>
__global__ void __launch_bounds__(kBlock, PF_WIDE_MINB) k_jacobi_wide(SellView A, const double* __restrict__ x_old,
                                                               double* __restrict__ x_new,
                                                               const double* __restrict__ b, int32_t n_own,
                                                               int32_t n, double omega) {
  vtab_stage<kVK>(A);
  const int32_t row = blockIdx.x * kBlock + threadIdx.x;
  RowWide<kG> hd;
  if (row < n_own) row_wide_head<kVK, kG>(A, row, hd);
  PF_PDL_ENTRY();
  if (row >= n) return;
  const double xo = x_old[row];
  if (row >= n_own) {
    x_new[row] = xo;
    return;
  }
  double acc = b[row], diag = 0.0;
  row_wide_offdiag<kVK, kG>(A, hd, row, x_old, acc, diag);
  x_new[row] = __dadd_rn(__dmul_rn(1.0 - omega, xo), __ddiv_rn(__dmul_rn(omega, acc), diag));
}

// Residual of the cycle (multigrid.cpp:166-167): y = A x (spmv order, acc from 0), r = b - y,
// on rows [0, n).
template <int kVK>
__global__ void __launch_bounds__(kBlock, minb_for<kVK>(PF_ROW_MINB)) k_residual(SellView A, const double* __restrict__ x,
                                                     const double* __restrict__ b,
                                                     double* __restrict__ r, int32_t n, int32_t n_own,
                                                     RowMap map) {
  vtab_stage<kVK>(A);
  const int32_t row = map_row(map, blockIdx.x, threadIdx.x, n_own);
  RowHead hd;
  if constexpr (head_early<kVK>())
    if (row >= 0 && row < n) row_head<kVK, kPrefetch>(A, row, hd);
  PF_PDL_ENTRY();
  if (row < 0 || row >= n) return;
  if constexpr (head_early<kVK>())
    r[row] = __dsub_rn(b[row], row_dot_from<false, true, kVK>(A, hd, x, 0.0));
  else
    r[row] = __dsub_rn(b[row], row_dot<false, true, kVK>(A, row, x, 0.0));
}

// y = A x on every row (linalg.cpp:45-57).
template <int kVK>
__global__ void __launch_bounds__(kBlock, minb_for<kVK>(PF_ROW_MINB)) k_spmv(SellView A, const double* __restrict__ x,
                                                 double* __restrict__ y, int32_t n) {
  PF_PDL_ENTRY();
  const int32_t row = blockIdx.x * kBlock + threadIdx.x;
  if (row >= n) return;
  y[row] = row_dot<false, true, kVK>(A, row, x, 0.0);
}

// Deterministic block sum: fixed shuffle tree inside each warp, then warp 0 sums the
// per-warp values in warp order.  No floating-point atomics anywhere.
__device__ __forceinline__ double block_sum(double v, double* smem /* kBlock/32 */) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) smem[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (warp == 0) {
    s = lane < (kBlock / 32) ? smem[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
  }
  return s;  // valid in thread 0
}

// sum_{r < n_own} (b_r - A_r x)^2 (residual_norm's local part, linalg.cpp:64-73).  Every
// block writes its partial; the last block to finish (ticket counter, integer atomic
// only) sums the partials in index order, stores the rank sum in *sumsq and, when
// `norm_out` is set (single-subdomain case: the ascending-rank allreduce of one value
// is 0.0 + s, transport.cpp:139-149), sqrt of it.  The ticket is reset for the next use.
template <int kVK>
__global__ void __launch_bounds__(kBlock, minb_for<kVK>(PF_ROW_MINB)) k_resnorm(SellView A, const double* __restrict__ x,
                                                    const double* __restrict__ b, int32_t n_own,
                                                    double* __restrict__ partials,
                                                    unsigned int* ticket, double* sumsq,
                                                    double* norm_out) {
  vtab_stage<kVK>(A);
  PF_PDL_ENTRY();
  __shared__ double smem[kBlock / 32];
  __shared__ bool last;
  const int32_t row = blockIdx.x * kBlock + threadIdx.x;
  double sq = 0.0;
  if (row < n_own) {
    const double acc = row_dot<true, true, kVK>(A, row, x, b[row]);
    sq = __dmul_rn(acc, acc);
  }
  const double s = block_sum(sq, smem);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = 0.0;
  for (unsigned int i = threadIdx.x; i < gridDim.x; i += kBlock) t = __dadd_rn(t, partials[i]);
  __syncthreads();
  t = block_sum(t, smem);
  if (threadIdx.x == 0) {
    *sumsq = t;
    if (norm_out) *norm_out = sqrt(__dadd_rn(0.0, t));
    *ticket = 0u;
  }
}

// k_jacobi that also returns the residual norm of its input iterate: each own row's
// b - A x_old is accumulated alongside the sweep from the same loaded entries (in the
// reference's order, so each row's residual is bit-identical), so solve_outer's convergence
// test of the previous cycle (multigrid.cpp:230) costs no extra pass over the matrix.
// Deterministic block sums + last-block finish exactly as k_resnorm; *sumsq gets this
// subdomain's sum of squares.
template <int kVK>
__global__ void __launch_bounds__(kBlock, minb_for<kVK>(PF_ROW_MINB)) k_jacobi_norm(SellView A, const double* __restrict__ x_old,
                                                        double* __restrict__ x_new,
                                                        const double* __restrict__ b, int32_t n_own,
                                                        int32_t n, double omega,
                                                        double* __restrict__ partials,
                                                        unsigned int* ticket, double* sumsq) {
  vtab_stage<kVK>(A);
  PF_PDL_ENTRY();
  __shared__ double smem[kBlock / 32];
  __shared__ bool last;
  const int32_t row = blockIdx.x * kBlock + threadIdx.x;
  double sq = 0.0;
  if (row < n) {
    const double xo = x_old[row];
    if (row >= n_own) {
      x_new[row] = xo;
    } else {
      double acc = b[row], diag = 0.0, res = b[row];
      row_offdiag<true, true, kVK, kChunkGroups, kPrefetch>(A, row, x_old, acc, diag, &res, xo);
      sq = __dmul_rn(res, res);
      x_new[row] = __dadd_rn(__dmul_rn(1.0 - omega, xo), __ddiv_rn(__dmul_rn(omega, acc), diag));
    }
  }
  const double s = block_sum(sq, smem);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = 0.0;
  for (unsigned int i = threadIdx.x; i < gridDim.x; i += kBlock) t = __dadd_rn(t, partials[i]);
  __syncthreads();
  t = block_sum(t, smem);
  if (threadIdx.x == 0) {
    *sumsq = t;
    *ticket = 0u;
  }
}

// Ordered allreduce of per-subdomain sums: out = sqrt(((0 + s_0) + s_1) + ...)
// (ascending rank, transport.cpp:139-149), optionally without the sqrt.
static __global__ void k_ordered_sum(const double* __restrict__ parts, int n, double* out, int take_sqrt) {
  PF_PDL_ENTRY();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0;
  for (int i = 0; i < n; ++i) s = __dadd_rn(s, parts[i]);
  *out = take_sqrt ? sqrt(s) : s;
}

// x_f += P x_c over every local fine dof (multigrid.cpp:121-129 + :183-184): the
// correction is accumulated from 0 in P's entry order, then added.
#ifndef PF_PROLONG_MINB
#define PF_PROLONG_MINB PF_ROW_MINB
#endif
#ifndef PF_RESTRICT_MINB
#define PF_RESTRICT_MINB PF_ROW_MINB
#endif
template <int kVK>
__global__ void __launch_bounds__(kBlock, minb_for<kVK>(PF_PROLONG_MINB)) k_prolong_add(SellView P, const double* __restrict__ xc,
                                                        double* __restrict__ xf, int32_t n_f, int add) {
  vtab_stage<kVK>(P);
  const int32_t row = blockIdx.x * kBlock + threadIdx.x;
  RowHead hd;
  if constexpr (head_early<kVK>())
    if (row < n_f) row_head<kVK, kPrefetch>(P, row, hd);
  PF_PDL_ENTRY();
  if (row >= n_f) return;
  double acc;
  if constexpr (head_early<kVK>())
    acc = row_dot_from<false, true, kVK>(P, hd, xc, 0.0);
  else
    acc = row_dot<false, true, kVK>(P, row, xc, 0.0);
  xf[row] = add ? __dadd_rn(xf[row], acc) : acc;
}

// k_prolong_add for prolongations of at most 8 entries per row (trilinear Q1: 1, 2, 4 or 8)
// with 8-bit weights: both groups of a row's columns and weight indices issued at once, then
// all of its coarse gathers at once — two dependent round trips after the row start instead
// of one per group.  Same sum, in the same order, as k_prolong_add.
template <int kVK>
__global__ void __launch_bounds__(kBlock, minb_for<kVK>(PF_PROLONG_MINB)) k_prolong_add8(SellView P, const double* __restrict__ xc,
                                                                       double* __restrict__ xf, int32_t n_f, int add) {
  static_assert(vk_kind<kVK>() == 1 || vk_kind<kVK>() == kVKSmem, "8-bit weights");
  vtab_stage<kVK>(P);
  PF_PDL_ENTRY();
  const int32_t row = blockIdx.x * kBlock + threadIdx.x;
  if (row >= n_f) return;
  const int64_t base = sell_row_base(P.slice_ptr, row);
  const int len = P.row_len[row];
  const double xo = add ? xf[row] : 0.0;
  int4 c0 = make_int4(0, 0, 0, 0), c1 = make_int4(0, 0, 0, 0);
  unsigned int w0 = 0, w1 = 0;
  if (len > 0) {
    c0 = ld_op<kVK>(reinterpret_cast<const int4*>(P.cols + base));
    w0 = ld_op<kVK>(reinterpret_cast<const unsigned int*>(static_cast<const unsigned char*>(P.vidx) + base));
  }
  if (len > 4) {
    c1 = ld_op<kVK>(reinterpret_cast<const int4*>(P.cols + base + 128));
    w1 = ld_op<kVK>(reinterpret_cast<const unsigned int*>(static_cast<const unsigned char*>(P.vidx) + base + 128));
  }
  const int32_t c[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
  double xv[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) xv[j] = j < len ? __ldg(xc + c[j]) : 0.0;
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (j < len) acc = __dadd_rn(acc, __dmul_rn(wide_val<kVK>(P, j < 4 ? w0 : w1, j & 3), xv[j]));
  xf[row] = add ? __dadd_rn(xo, acc) : acc;
}

// rc = R r_f with R = P^T restricted to owns_row fine rows (multigrid.cpp:131-146), as a
// gather: each coarse row sums its fine contributions in ascending fine host index,
// i.e. exactly the order of the reference's scatter-add.  Fused epilogue of the cycle
// (multigrid.cpp:172-179): Dirichlet coarse entries of b become 0 and the coarse x is
// zeroed.  (Zeroing before the master/slave accumulate is equivalent: Dirichlet
// carriers are Dirichlet on every rank, so they only ever accumulate zeros.)
template <int kVK>
__global__ void __launch_bounds__(kBlock, minb_for<kVK>(PF_RESTRICT_MINB)) k_restrict(SellView R, const double* __restrict__ rf,
                                                     double* __restrict__ bc,
                                                     double* __restrict__ xc,
                                                     const uint8_t* __restrict__ is_dir_c,
                                                     int32_t n_c, int zero_dirichlet) {
  vtab_stage<kVK>(R);
  const int32_t row = blockIdx.x * kBlock + threadIdx.x;
  RowHead hd;
  if constexpr (head_early<kVK>())
    if (row < n_c) row_head<kVK, kPrefetch>(R, row, hd);
  PF_PDL_ENTRY();
  if (row >= n_c) return;
  double acc;
  if constexpr (head_early<kVK>())
    acc = row_dot_from<false, true, kVK>(R, hd, rf, 0.0);
  else
    acc = row_dot<false, true, kVK>(R, row, rf, 0.0);
  bc[row] = (zero_dirichlet && is_dir_c[row]) ? 0.0 : acc;
  if (xc) xc[row] = 0.0;
}

// Cycle residual + restriction of a small level in one launch (multigrid.cpp:166-176): one
// warp per coarse row; lane j forms the residual of the row's j-th fine entry exactly as
// k_residual does (b_f - A_f x, products summed from 0 in stored order), scales it by the
// entry's weight, and lane 0 adds the products in R's stored order from 0 — k_restrict's
// sum — then the Dirichlet zeroing and the coarse x = 0.  A fine residual shared by several
// coarse rows is formed once per row (identical bits every time); on the latency-bound
// small levels that redundancy is cheaper than a second launch.  R rows of <= 32 entries.
template <int kVK>
__global__ void __launch_bounds__(kBlock) k_residual_restrict(SellView A, SellView R, const double* __restrict__ x,
                                                              const double* __restrict__ b, double* __restrict__ bc,
                                                              double* __restrict__ xc,
                                                              const uint8_t* __restrict__ is_dir_c, int32_t n_c,
                                                              int zero_dirichlet) {
  vtab_stage<kVK>(A);
  PF_PDL_ENTRY();
  const int32_t row = static_cast<int32_t>((static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n_c) return;  // whole warps exit together
  const int len = R.row_len[row];
  double p = 0.0;
  if (lane < len) {
    const int64_t e = sell_entry(sell_row_base(R.slice_ptr, row), lane);
    const int32_t f = R.cols[e];
    const double r = __dsub_rn(b[f], row_dot<false, true, kVK>(A, f, x, 0.0));
    p = __dmul_rn(sell_val<-1>(R, e), r);
  }
  double acc = 0.0;
  for (int j = 0; j < len; ++j) {
    const double pj = __shfl_sync(0xffffffffu, p, j);
    acc = __dadd_rn(acc, pj);
  }
  if (lane == 0) {
    bc[row] = (zero_dirichlet && is_dir_c[row]) ? 0.0 : acc;
    if (xc) xc[row] = 0.0;
  }
}

// Sequential coarse solve (solvers.cpp:70-92) of every subdomain held on this device:
// per iteration, in-place Gauss-Seidel over each subdomain's own rows in the
// reference's host order (host_of_own[i] = device row of host own dof i), then the
// communicating part of smooth() — update_master_slave(Scatter) and update_halo1
// (solvers.cpp:65-66) as level-global index copies — then residual_norm with the
// ascending-rank sum; stop at <= tol * r0 or max_iter.  One thread: the coarse level of
// the n_coarse=2 hierarchies holds one unknown, and a sequential sweep is the only way
// to keep the reference's exact ordering.  stats: [iterations, converged, r0, final].
static __device__ void coarse_gs_body(const CoarseSub* __restrict__ subs, int n_sub, double* x,
                               const double* __restrict__ b, const int32_t* __restrict__ ms_dst,
                               const int32_t* __restrict__ ms_src, int32_t ms_n,
                               const int32_t* __restrict__ h1_dst, const int32_t* __restrict__ h1_src,
                               int32_t h1_n, double tol, int32_t max_iter, double* stats) {
  auto norm = [&]() {
    double total = 0.0;
    for (int s = 0; s < n_sub; ++s) {
      const CoarseSub& S = subs[s];
      const double* xs = x + S.offset;
      const double* bs = b + S.offset;
      double local = 0.0;
      for (int32_t i = 0; i < S.n_own; ++i) {
        const int32_t d = S.host_of_own[i];
        const int64_t base = sell_row_base(S.A.slice_ptr, d);
        double acc = bs[d];
        for (int j = 0; j < S.A.row_len[d]; ++j) {
          const int64_t e = sell_entry(base, j);
          acc = __dsub_rn(acc, __dmul_rn(sell_val<-1>(S.A, e), xs[S.A.cols[e]]));
        }
        local = __dadd_rn(local, __dmul_rn(acc, acc));
      }
      total = __dadd_rn(total, local);
    }
    return sqrt(total);
  };
  const double r0 = norm();
  stats[0] = 0;
  stats[1] = 1;
  stats[2] = r0;
  stats[3] = r0;
  if (r0 == 0.0) return;
  const double target = __dmul_rn(tol, r0);
  int it = 0;
  while (it < max_iter) {
    for (int s = 0; s < n_sub; ++s) {
      const CoarseSub& S = subs[s];
      double* xs = x + S.offset;
      const double* bs = b + S.offset;
      for (int32_t i = 0; i < S.n_own; ++i) {
        const int32_t d = S.host_of_own[i];
        const int64_t base = sell_row_base(S.A.slice_ptr, d);
        double acc = bs[d], diag = 0.0;
        for (int j = 0; j < S.A.row_len[d]; ++j) {
          const int64_t e = sell_entry(base, j);
          const int32_t c = S.A.cols[e];
          if (c == d)
            diag = sell_val<-1>(S.A, e);
          else
            acc = __dsub_rn(acc, __dmul_rn(sell_val<-1>(S.A, e), xs[c]));
        }
        xs[d] = __ddiv_rn(acc, diag);
      }
    }
    for (int32_t i = 0; i < ms_n; ++i) x[ms_dst[i]] = x[ms_src[i]];
    for (int32_t i = 0; i < h1_n; ++i) x[h1_dst[i]] = x[h1_src[i]];
    ++it;
    const double fr = norm();
    stats[0] = it;
    stats[3] = fr;
    if (fr <= target) return;
  }
  stats[1] = 0;
}

// coarse_gs_body on a block: all threads stage the packed level in shared memory (one
// round of parallel loads); the residual norm takes one row per thread (squares summed
// by thread 0 in row order); the Gauss-Seidel sweep visits the rows in order with warp 0:
// its lanes form the row's products a_e x_c from the current x, lane 0 subtracts them in
// stored order.  Same operations in the same order as coarse_gs_body.
static __device__ void coarse_gs_smem(const CoarsePack& P, double* x, const double* __restrict__ b, double tol,
                               int32_t max_iter, double* stats, unsigned char* smem) {
  double* sx = reinterpret_cast<double*>(smem);
  double* sb = sx + P.n_total;
  double* sv = sb + P.n_rows;
  double* ssq = sv + P.nnz;
  double* sp = ssq + P.n_rows;
  double* stot = sp + (P.max_row > P.n_rows ? P.max_row : P.n_rows);
  int32_t* srp = reinterpret_cast<int32_t*>(stot + 1);
  int32_t* srd = srp + P.n_rows + 1;
  int32_t* sc = srd + P.n_rows;
  int32_t* ssr = sc + P.nnz;
  int32_t* smd = ssr + P.n_sub + 1;
  int32_t* sms = smd + P.ms_n;
  int32_t* shd = sms + P.ms_n;
  int32_t* shs = shd + P.h1_n;
  int32_t* sdg = shs + P.h1_n;
  for (int i = threadIdx.x; i < P.n_total; i += blockDim.x) sx[i] = x[i];
  for (int i = threadIdx.x; i < P.n_rows; i += blockDim.x) {
    srd[i] = P.rowdev[i];
    sb[i] = b[P.rowdev[i]];
  }
  for (int i = threadIdx.x; i <= P.n_rows; i += blockDim.x) srp[i] = P.rowptr[i];
  for (int i = threadIdx.x; i < P.nnz; i += blockDim.x) {
    sv[i] = P.vals[i];
    sc[i] = P.cols[i];
  }
  for (int i = threadIdx.x; i <= P.n_sub; i += blockDim.x) ssr[i] = P.sub_rows[i];
  for (int i = threadIdx.x; i < P.ms_n; i += blockDim.x) {
    smd[i] = P.ms_dst[i];
    sms[i] = P.ms_src[i];
  }
  for (int i = threadIdx.x; i < P.h1_n; i += blockDim.x) {
    shd[i] = P.h1_dst[i];
    shs[i] = P.h1_src[i];
  }
  __syncthreads();
  // position of each row's diagonal entry (the last one, as the sequential scan keeps)
  for (int i = threadIdx.x; i < P.n_rows; i += blockDim.x) {
    int32_t dpos = -1;
    for (int32_t e = srp[i]; e < srp[i + 1]; ++e)
      if (sc[e] == srd[i]) dpos = e;
    sdg[i] = dpos;
  }
  auto norm = [&]() {
    __syncthreads();
    for (int i = threadIdx.x; i < P.n_rows; i += blockDim.x) {
      double acc = sb[i];
      for (int32_t e = srp[i]; e < srp[i + 1]; ++e) acc = __dsub_rn(acc, __dmul_rn(sv[e], sx[sc[e]]));
      ssq[i] = __dmul_rn(acc, acc);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double total = 0.0;
      for (int s = 0; s < P.n_sub; ++s) {
        double local = 0.0;
        for (int32_t i = ssr[s]; i < ssr[s + 1]; ++i) local = __dadd_rn(local, ssq[i]);
        total = __dadd_rn(total, local);
      }
      stot[0] = sqrt(total);
    }
    __syncthreads();
    return stot[0];
  };
  const double r0 = norm();
  if (threadIdx.x == 0) {
    stats[0] = 0;
    stats[1] = 1;
    stats[2] = r0;
    stats[3] = r0;
  }
  if (P.inv && r0 != 0.0) {
    // direct: r = b - A_o,rest x_rest (stored order), x_own = inv r (ascending columns)
    for (int i = threadIdx.x; i < P.n_rows; i += blockDim.x) {
      double acc = sb[i];
      for (int32_t e = srp[i]; e < srp[i + 1]; ++e)
        if (sc[e] >= P.n_own_dev) acc = __dsub_rn(acc, __dmul_rn(sv[e], sx[sc[e]]));
      sp[i] = acc;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < P.n_rows; i += blockDim.x) {
      double acc = 0.0;
      const double* row = P.inv + static_cast<int64_t>(i) * P.n_rows;
      for (int32_t j = 0; j < P.n_rows; ++j) acc = __dadd_rn(acc, __dmul_rn(__ldg(row + j), sp[j]));
      sx[srd[i]] = acc;
    }
    const double fr = norm();
    if (threadIdx.x == 0) {
      stats[0] = 1;
      stats[1] = fr <= __dmul_rn(tol, r0) ? 1 : 0;
      stats[3] = fr;
    }
  } else if (r0 != 0.0) {
    const double target = __dmul_rn(tol, r0);
    const int lane = threadIdx.x & 31;
    int it = 0;
    bool conv = false;
    while (it < max_iter) {
      if (threadIdx.x < 32) {
        for (int32_t i = 0; i < P.n_rows; ++i) {
          const int32_t r0e = srp[i], r1e = srp[i + 1];
          for (int32_t e = r0e + lane; e < r1e; e += 32) sp[e - r0e] = __dmul_rn(sv[e], sx[sc[e]]);
          __syncwarp();
          if (lane == 0) {
            const int32_t de = sdg[i];
            double acc = sb[i], diag = 0.0;
            for (int32_t e = r0e; e < r1e; ++e) {
              if (e == de)
                diag = sv[e];
              else
                acc = __dsub_rn(acc, sp[e - r0e]);
            }
            sx[srd[i]] = __ddiv_rn(acc, diag);
          }
          __syncwarp();
        }
        if (lane == 0) {
          for (int32_t i = 0; i < P.ms_n; ++i) sx[smd[i]] = sx[sms[i]];
          for (int32_t i = 0; i < P.h1_n; ++i) sx[shd[i]] = sx[shs[i]];
        }
      }
      ++it;
      const double fr = norm();
      if (threadIdx.x == 0) {
        stats[0] = it;
        stats[3] = fr;
      }
      if (fr <= target) {
        conv = true;
        break;
      }
    }
    if (!conv && threadIdx.x == 0) stats[1] = 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < P.n_total; i += blockDim.x) x[i] = sx[i];
}

static __global__ void k_coarse_smem(CoarsePack P, double* x, const double* __restrict__ b, double tol,
                              int32_t max_iter, double* stats) {
  PF_PDL_ENTRY();
  extern __shared__ __align__(16) unsigned char smem_c[];
  coarse_gs_smem(P, x, b, tol, max_iter, stats, smem_c);
}

static __global__ void k_coarse_gs(const CoarseSub* __restrict__ subs, int n_sub, double* x,
                            const double* __restrict__ b, const int32_t* __restrict__ ms_dst,
                            const int32_t* __restrict__ ms_src, int32_t ms_n,
                            const int32_t* __restrict__ h1_dst, const int32_t* __restrict__ h1_src,
                            int32_t h1_n, double tol, int32_t max_iter, double* stats) {
  PF_PDL_ENTRY();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  coarse_gs_body(subs, n_sub, x, b, ms_dst, ms_src, ms_n, h1_dst, h1_src, h1_n, tol, max_iter, stats);
}

// ------------------------------------------------------------- vector utilities --

// Host order -> device order: dev[perm[i]] = host[i].
static __global__ void k_scatter_perm(const double* __restrict__ host, const int32_t* __restrict__ perm,
                               double* __restrict__ dev, int32_t n) {
  PF_PDL_ENTRY();
  const int32_t i = blockIdx.x * kBlock + threadIdx.x;
  if (i < n) dev[perm[i]] = host[i];
}
// Device order -> host order: host[i] = dev[perm[i]].
static __global__ void k_gather_perm(const double* __restrict__ dev, const int32_t* __restrict__ perm,
                              double* __restrict__ host, int32_t n) {
  PF_PDL_ENTRY();
  const int32_t i = blockIdx.x * kBlock + threadIdx.x;
  if (i < n) host[i] = dev[perm[i]];
}
static __global__ void k_fill(double* __restrict__ v, double value, int64_t n) {
  PF_PDL_ENTRY();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x;
  if (i < n) v[i] = value;
}
static __global__ void k_copy(const double* __restrict__ src, double* __restrict__ dst, int64_t n) {
  PF_PDL_ENTRY();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x;
  if (i < n) dst[i] = src[i];
}

// ------------------------------------------------------------- exchange kernels --
// A channel plan flattens every (peer, entry) of one exchange of one subdomain.

// Local transport of one scatter: v[dst[i]] = v[src[i]] (pack + send + recv + unpack of
// fecomm.cpp:25-39 when every peer lives on this device).
static __global__ void k_copy_idx(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                           double* v, int32_t n) {
  PF_PDL_ENTRY();
  const int32_t i = blockIdx.x * kBlock + threadIdx.x;
  if (i < n) v[dst[i]] = v[src[i]];
}
// Pack: buf[i] = v[idx[i]] (send side of scatter, fecomm.cpp:28-32).
static __global__ void k_pack(const double* __restrict__ v, const int32_t* __restrict__ idx,
                       double* __restrict__ buf, int32_t n) {
  PF_PDL_ENTRY();
  const int32_t i = blockIdx.x * kBlock + threadIdx.x;
  if (i < n) buf[i] = v[idx[i]];
}
// Unpack: v[idx[i]] = buf[i] (receive side of scatter, fecomm.cpp:33-38).
static __global__ void k_unpack(const double* __restrict__ buf, const int32_t* __restrict__ idx,
                         double* __restrict__ v, int32_t n) {
  PF_PDL_ENTRY();
  const int32_t i = blockIdx.x * kBlock + threadIdx.x;
  if (i < n) v[idx[i]] = buf[i];
}
// Accumulate (fecomm.cpp:43-59): master entry m receives its slave partials in ascending
// peer order: v[dst[m]] = ((v + p_a) + p_b) + ...  with the partials' buffer positions
// listed per master in src[acc_off[m] .. acc_off[m+1]).
static __global__ void k_unpack_accumulate(const double* __restrict__ buf,
                                    const int32_t* __restrict__ acc_off,
                                    const int32_t* __restrict__ src,
                                    const int32_t* __restrict__ dst, double* __restrict__ v,
                                    int32_t n_masters) {
  PF_PDL_ENTRY();
  const int32_t m = blockIdx.x * kBlock + threadIdx.x;
  if (m >= n_masters) return;
  double acc = v[dst[m]];
  for (int32_t e = acc_off[m]; e < acc_off[m + 1]; ++e) acc = __dadd_rn(acc, buf[src[e]]);
  v[dst[m]] = acc;
}

}  // namespace pf
