// pf_window.cuh — the row kernels over block windows (WinView, pf_types.hpp).
//
// ncu of the plain finest-level sweep (profiles/r02_ncu_k_jacobi_c2_details.csv): DRAM 52 %,
// L1/TEX 64 %, issue slots 59 %, 15 warp cycles per instruction — every stored entry costs
// a 4-byte column from HBM and an 8-byte x gather that is its own L1 request (42 % L1 hit
// rate, the rest a round trip to L2).  With the device placement the x entries a block of
// 256 consecutive rows reads are a few dozen short runs (a few lattice lines of each other
// colour), so the block copies them into shared memory once, with coalesced 128-byte loads
// (all of them independent: one round trip), and every gather becomes a shared-memory read
// at a 16-bit slot: 2 + 1 instead of 4 + 1 bytes per stored entry from HBM, and no L1/L2
// request per entry.  Rows do the same operations in the same order as the plain kernels
// (row_offdiag / row_dot of pf_kernels.cuh), so results are bit-identical.
//
// Status: opt-in (Options::win, PF_WIN=1), parity-tested, measured SLOWER than the plain
// kernels (C2 finest Jacobi sweep 87.4 vs 74.5 us, SOR 106.5 vs 103.8 us, fp64 values 133 vs
// 112 us): the SM's LSU data pipe is as busy as before (shared-memory gathers, value-table
// lookups and the staging's own loads and stores), see profiles/r02_sweep_experiments.md.
//
// Layout of a block's window in shared memory (WinView, pf_types.hpp): slot t < kBlock is
// private to thread t — its row's diagonal and padding entries point there — and holds
// x_r in the residual-type kernels and a zero of the diagonal's sign in the smoothers, whose
// off-diagonal sum thereby skips the diagonal without a per-entry test (a_rr * (+-0) = +0.0,
// and acc - (+0.0) == acc for every acc, -0.0 and NaN included); the cover chunks of the
// other columns follow in ascending x order.
#pragma once

#include "pf_kernels.cuh"

namespace pf {

// The block's chunk starts into shared memory (operator data: before griddepcontrol.wait),
// padded with a sentinel to the staging loop's batch; win_stage's first barrier publishes them.
constexpr int kWinHalfWarps = kBlock / kWinChunk, kWinBatch = 8;
constexpr int kWinChunkSlots = (kWinChunksCap + kWinHalfWarps * kWinBatch - 1) / (kWinHalfWarps * kWinBatch) *
                               (kWinHalfWarps * kWinBatch);
__device__ __forceinline__ void win_chunks(const WinView& W, int32_t c0, int32_t c1, int32_t* s_ch) {
  for (int32_t i = threadIdx.x; i < kWinChunkSlots; i += kBlock)
    s_ch[i] = c0 + i < c1 ? __ldg(W.chunks + c0 + i) : INT32_MAX - kWinChunk;
}

// Copy the block's cover of x into the window (half-warp per chunk, 8 independent loads in
// flight per thread); ends with a block barrier.
__device__ __forceinline__ void win_stage(const int32_t* s_ch, int32_t nch, const double* __restrict__ x,
                                          int32_t n, double* s_x) {
  const int sub = threadIdx.x / kWinChunk, ln = threadIdx.x % kWinChunk;
  double* dst = s_x + kBlock + sub * kWinChunk + ln;
  __syncthreads();  // s_ch
  for (int32_t i0 = sub; i0 < nch; i0 += kWinHalfWarps * kWinBatch, dst += kWinHalfWarps * kWinBatch * kWinChunk) {
    double v[kWinBatch];
    int32_t g[kWinBatch];
#pragma unroll
    for (int k = 0; k < kWinBatch; ++k) {
      g[k] = s_ch[i0 + k * kWinHalfWarps] + ln;
      if (g[k] < n) v[k] = __ldg(x + g[k]);
    }
#pragma unroll
    for (int k = 0; k < kWinBatch; ++k)
      if (g[k] < n) dst[k * kWinHalfWarps * kWinChunk] = v[k];
  }
  __syncthreads();
}

// One group of 4 stored entries as loaded (window byte offsets packed in 8 bytes, values
// still encoded: a pending group costs 3 registers, not 12), and its decoding.
struct WinRaw {
  uint2 cc;
  uint32_t w0, w1;
  double v[4];
};
template <int kVK>
__device__ __forceinline__ void win_load(const SellView& A, const WinView& W, int64_t e, WinRaw& r) {
  constexpr int K = vk_kind<kVK>();
  r.cc = ld_op<kVK>(reinterpret_cast<const uint2*>(W.cols16 + e));
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
__device__ __forceinline__ void win_decode(const SellView& A, const WinRaw& r, uint32_t o[4], double v[4]) {
  constexpr int K = vk_kind<kVK>();
  o[0] = r.cc.x & 0xffffu;
  o[1] = r.cc.x >> 16;
  o[2] = r.cc.y & 0xffffu;
  o[3] = r.cc.y >> 16;
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
__device__ __forceinline__ double win_x(const double* s_x, uint32_t off) {
  return *reinterpret_cast<const double*>(reinterpret_cast<const char*>(s_x) + off);
}

template <int kVK, int kPf>
__device__ __forceinline__ void win_prefetch(const SellView& A, const WinView& W, int64_t base, int len) {
  if constexpr (kPf > 0 && !vk_cached<kVK>()) {
    const int ng = (len + 3) / 4;
#pragma unroll
    for (int g = 1; g <= kPf; ++g) {
      if (g < ng) {
        const int64_t e = sell_entry(base, 4 * g);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(W.cols16 + e));
        if constexpr (vk_kind<kVK>() == 1 || vk_kind<kVK>() == kVKSmem)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(static_cast<const unsigned char*>(A.vidx) + e));
        else if constexpr (vk_kind<kVK>() == 2)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(static_cast<const unsigned short*>(A.vidx) + e));
        else if constexpr (vk_kind<kVK>() == 0)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(A.vals + e));
      }
    }
  }
}

// The operator-only start of a window row (cf. RowHead / row_head): base, length and the
// first group as loaded; kDiag: also the diagonal value (through WinView::dpos).
struct WinHead {
  int64_t base;
  int len;
  WinRaw g0;
  double diag;
};
template <int kVK, int kPf, bool kDiag>
__device__ __forceinline__ void win_head(const SellView& A, const WinView& W, int32_t row, WinHead& h) {
  h.base = sell_row_base(A.slice_ptr, row);
  h.len = A.row_len[row];
  win_prefetch<kVK, kPf>(A, W, h.base, h.len);
  if (h.len > 0) win_load<kVK>(A, W, h.base, h.g0);
  if constexpr (kDiag) h.diag = sell_val<kVK>(A, sell_entry(h.base, W.dpos[row]));
}

// A row over its window, entries in stored order, a group of 4 at a time with the next
// group's loads issued first; only the last group is predicated (its padding entries).
//   kWinSmooth:  acc -= a x over every entry — the private slot holds the signed zero, so the
//                diagonal term subtracts +0.0 (row_offdiag without the residual)
//   kWinSub/Add: acc -= / += a x over every entry, the private slot holds x_r (row_dot)
//   kWinBoth:    res -= a x over every entry and acc -= a x off the diagonal, the private
//                slot holds x_r (row_offdiag with the residual: k_jacobi_norm)
enum { kWinSmooth = 0, kWinSub = 1, kWinAdd = 2, kWinBoth = 3 };
template <int kMode, int kVK>
__device__ __forceinline__ void win_terms(const SellView& A, const WinRaw& raw, int n, uint32_t self,
                                          const double* s_x, double& acc, double& res) {
  uint32_t o[4];
  double v[4], xv[4];
  win_decode<kVK>(A, raw, o, v);
#pragma unroll
  for (int k = 0; k < 4; ++k) xv[k] = win_x(s_x, o[k]);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k < n) {
      const double p = __dmul_rn(v[k], xv[k]);
      if constexpr (kMode == kWinAdd) {
        acc = __dadd_rn(acc, p);
      } else if constexpr (kMode == kWinBoth) {
        res = __dsub_rn(res, p);
        if (o[k] != self) acc = __dsub_rn(acc, p);
      } else {
        acc = __dsub_rn(acc, p);
      }
    }
  }
}

template <int kMode, int kVK>
__device__ __forceinline__ void win_row(const SellView& A, const WinView& W, const WinHead& h, const double* s_x,
                                        double& acc, double& res) {
  const int len = h.len;
  if (len <= 0) return;
  const uint32_t self = threadIdx.x * 8u;
  WinRaw cur = h.g0;
  int j = 0;
  for (; j + 4 < len; j += 4) {
    WinRaw nxt;
    win_load<kVK>(A, W, sell_entry(h.base, j + 4), nxt);
    win_terms<kMode, kVK>(A, cur, 4, self, s_x, acc, res);
    cur = nxt;
  }
  win_terms<kMode, kVK>(A, cur, len - j, self, s_x, acc, res);
}

#ifndef PF_WIN_MINB
#define PF_WIN_MINB 5
#endif
#ifndef PF_WIN_PREFETCH
#define PF_WIN_PREFETCH 6
#endif
constexpr int kWinPf = PF_WIN_PREFETCH;

// Every kernel below: a block with a window (non-empty chunk range) stages it and its own
// rows read the 16-bit offsets; a block without one (cover over the cap, or past the own
// rows) takes the plain row path of pf_kernels.cuh.  The choice is uniform per block, and
// the two paths are separate branches (each with its own griddepcontrol.wait) so neither
// path's registers stay live through the other.
#define PF_WIN_SHARED()                           \
  extern __shared__ double s_x[];                 \
  __shared__ int32_t s_ch[kWinChunkSlots];        \
  vtab_stage<kVK>(A);                             \
  const int32_t c0 = W.chunk_ptr[blk], c1 = W.chunk_ptr[blk + 1]
// window branch: chunk starts and the row's head before the wait, the cover after it
#define PF_WIN_ENTER(x_vec, kDiag)                                   \
  WinHead wh;                                                        \
  win_chunks(W, c0, c1, s_ch);                                       \
  if (act) win_head<kVK, kPfW, kDiag>(A, W, row, wh);                \
  PF_PDL_ENTRY();                                                    \
  win_stage(s_ch, c1 - c0, x_vec, n, s_x)

// The zero whose product with the diagonal value is +0.0.
__device__ __forceinline__ double win_zero_for(double diag) { return copysign(0.0, diag); }

// k_jacobi over block windows (identity block schedule): own rows relaxed from the staged
// x_old, every other row carried over.
template <int kVK>
__global__ void __launch_bounds__(kBlock, PF_WIN_MINB) k_jacobi_win(SellView A, WinView W,
                                                                    const double* __restrict__ x_old,
                                                                    double* __restrict__ x_new,
                                                                    const double* __restrict__ b, int32_t n_own,
                                                                    int32_t n, double omega) {
  constexpr int kPfW = kWinPf;
  const int32_t blk = blockIdx.x, row = blk * kBlock + threadIdx.x;
  const bool act = row < n_own;
  PF_WIN_SHARED();
  if (c1 > c0) {
    PF_WIN_ENTER(x_old, true);
    if (row >= n) return;
    const double xo = x_old[row];
    if (!act) {
      x_new[row] = xo;
      return;
    }
    double acc = b[row], unused = 0.0;
    s_x[threadIdx.x] = win_zero_for(wh.diag);
    win_row<kWinSmooth, kVK>(A, W, wh, s_x, acc, unused);
    x_new[row] = __dadd_rn(__dmul_rn(1.0 - omega, xo), __ddiv_rn(__dmul_rn(omega, acc), wh.diag));
  } else {
    PF_PDL_ENTRY();
    if (row >= n) return;
    const double xo = x_old[row];
    if (!act) {
      x_new[row] = xo;
      return;
    }
    double acc = b[row], diag = 0.0;
    row_offdiag<true, false, kVK, kChunkGroups, kPrefetch>(A, row, x_old, acc, diag);
    x_new[row] = __dadd_rn(__dmul_rn(1.0 - omega, xo), __ddiv_rn(__dmul_rn(omega, acc), diag));
  }
}

// The deterministic finish of the norm kernels (as k_resnorm / k_jacobi_norm).
__device__ __forceinline__ void win_norm_finish(double sq, double* __restrict__ partials, unsigned int* ticket,
                                                double* sumsq, double* norm_out) {
  __shared__ double smem[kBlock / 32];
  __shared__ bool last;
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

// k_jacobi_norm over block windows.
template <int kVK>
__global__ void __launch_bounds__(kBlock, PF_WIN_MINB) k_jacobi_norm_win(SellView A, WinView W,
                                                                         const double* __restrict__ x_old,
                                                                         double* __restrict__ x_new,
                                                                         const double* __restrict__ b, int32_t n_own,
                                                                         int32_t n, double omega,
                                                                         double* __restrict__ partials,
                                                                         unsigned int* ticket, double* sumsq) {
  constexpr int kPfW = kWinPf;
  const int32_t blk = blockIdx.x, row = blk * kBlock + threadIdx.x;
  const bool act = row < n_own;
  PF_WIN_SHARED();
  double sq = 0.0;
  if (c1 > c0) {
    PF_WIN_ENTER(x_old, true);
    if (row < n) {
      const double xo = x_old[row];
      if (!act) {
        x_new[row] = xo;
      } else {
        double acc = b[row], res = b[row];
        s_x[threadIdx.x] = xo;
        win_row<kWinBoth, kVK>(A, W, wh, s_x, acc, res);
        sq = __dmul_rn(res, res);
        x_new[row] = __dadd_rn(__dmul_rn(1.0 - omega, xo), __ddiv_rn(__dmul_rn(omega, acc), wh.diag));
      }
    }
  } else {
    PF_PDL_ENTRY();
    if (row < n) {
      const double xo = x_old[row];
      if (!act) {
        x_new[row] = xo;
      } else {
        double acc = b[row], diag = 0.0, res = b[row];
        row_offdiag<true, true, kVK, kChunkGroups, kPrefetch>(A, row, x_old, acc, diag, &res, xo);
        sq = __dmul_rn(res, res);
        x_new[row] = __dadd_rn(__dmul_rn(1.0 - omega, xo), __ddiv_rn(__dmul_rn(omega, acc), diag));
      }
    }
  }
  win_norm_finish(sq, partials, ticket, sumsq, nullptr);
}

// k_residual over block windows: r = b - A x on rows [0, n) (the rows past the own ones
// have no window).
template <int kVK>
__global__ void __launch_bounds__(kBlock, PF_WIN_MINB) k_residual_win(SellView A, WinView W,
                                                                      const double* __restrict__ x,
                                                                      const double* __restrict__ b,
                                                                      double* __restrict__ r, int32_t n,
                                                                      int32_t n_own) {
  constexpr int kPfW = kWinPf;
  const int32_t blk = blockIdx.x, row = blk * kBlock + threadIdx.x;
  const bool act = row < n_own;
  PF_WIN_SHARED();
  if (c1 > c0) {
    PF_WIN_ENTER(x, false);
    if (row >= n) return;
    if (!act) {
      r[row] = __dsub_rn(b[row], row_dot<false, true, kVK>(A, row, x, 0.0));
    } else {
      s_x[threadIdx.x] = x[row];
      double acc = 0.0, unused = 0.0;
      win_row<kWinAdd, kVK>(A, W, wh, s_x, acc, unused);
      r[row] = __dsub_rn(b[row], acc);
    }
  } else {
    PF_PDL_ENTRY();
    if (row >= n) return;
    r[row] = __dsub_rn(b[row], row_dot<false, true, kVK>(A, row, x, 0.0));
  }
}

// k_resnorm over block windows (grid over the own rows).
template <int kVK>
__global__ void __launch_bounds__(kBlock, PF_WIN_MINB) k_resnorm_win(SellView A, WinView W,
                                                                     const double* __restrict__ x,
                                                                     const double* __restrict__ b, int32_t n_own,
                                                                     int32_t n, double* __restrict__ partials,
                                                                     unsigned int* ticket, double* sumsq,
                                                                     double* norm_out) {
  constexpr int kPfW = kWinPf;
  const int32_t blk = blockIdx.x, row = blk * kBlock + threadIdx.x;
  const bool act = row < n_own;
  PF_WIN_SHARED();
  double sq = 0.0;
  if (c1 > c0) {
    PF_WIN_ENTER(x, false);
    if (act) {
      double acc = b[row], unused = 0.0;
      s_x[threadIdx.x] = x[row];
      win_row<kWinSub, kVK>(A, W, wh, s_x, acc, unused);
      sq = __dmul_rn(acc, acc);
    }
  } else {
    PF_PDL_ENTRY();
    if (act) {
      const double acc = row_dot<true, true, kVK>(A, row, x, b[row]);
      sq = __dmul_rn(acc, acc);
    }
  }
  win_norm_finish(sq, partials, ticket, sumsq, norm_out);
}

// One colour of multicolour GS / SOR over block windows: the launch covers the window
// blocks block0, block0 + 1, ... that overlap the colour's rows [row0, row1); the rows of
// other colours inside the first and last block stay idle.  A block may stage x entries
// of this colour that other blocks are writing (chunk granularity), but no row reads them:
// a row's columns are its own entry and other colours' rows.
template <bool kSor, int kVK>
__global__ void __launch_bounds__(kBlock, PF_WIN_MINB) k_color_sweep_win(SellView A, WinView W, double* x,
                                                                         const double* __restrict__ b,
                                                                         int32_t block0, int32_t row0, int32_t row1,
                                                                         int32_t n, double omega) {
  constexpr int kPfW = 0;
  const int32_t blk = block0 + blockIdx.x, row = blk * kBlock + threadIdx.x;
  const bool act = row >= row0 && row < row1;
  PF_WIN_SHARED();
  double acc, diag;
  if (c1 > c0) {
    PF_WIN_ENTER(x, true);
    if (!act) return;
    acc = b[row];
    diag = wh.diag;
    double unused = 0.0;
    s_x[threadIdx.x] = win_zero_for(diag);
    win_row<kWinSmooth, kVK>(A, W, wh, s_x, acc, unused);
  } else {
    RowHead hd;
    if (act) row_head<kVK>(A, row, hd);
    PF_PDL_ENTRY();
    if (!act) return;
    acc = b[row];
    diag = 0.0;
    row_offdiag_from<true, false, kVK>(A, hd, row, x, acc, diag);
  }
  if (kSor)
    x[row] = __dadd_rn(__dmul_rn(1.0 - omega, x[row]), __ddiv_rn(__dmul_rn(omega, acc), diag));
  else
    x[row] = __ddiv_rn(acc, diag);
}

#undef PF_WIN_SHARED
#undef PF_WIN_ENTER

}  // namespace pf
