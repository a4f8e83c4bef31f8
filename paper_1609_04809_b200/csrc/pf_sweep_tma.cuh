// pf_sweep_tma.cuh — TMA-staged colour sweep of multicolour Gauss-Seidel / SOR.
//
// Same arithmetic, in the same order, as k_color_sweep (one_local_sweep, solvers.cpp:21-34,
// with the omega blend): only the way the operator reaches the threads changes.
//
// k_color_sweep walks a row's 7 SELL groups with a software pipeline one group deep, so
// every row is a chain of ~8 dependent memory round trips (row length -> columns and
// value indices -> x gathers, group after group); a colour (1/8 of the level) is ~1.7
// waves of such chains and the sweep ran at ~0.5 of HBM bandwidth.  Here a persistent
// block owns chunks of kCS consecutive SELL slices (kCS x 32 rows) of the colour:
//   * one elected thread streams a chunk's row lengths, columns and values (or value
//     indices) into shared memory with bulk asynchronous copies (cp.async.bulk, TMA
//     engine, completion on an mbarrier), double-buffered: chunk i+1 lands while chunk i
//     is computed;
//   * the first two chunks are requested BEFORE griddepcontrol.wait — the level operator
//     is immutable once uploaded, so the matrix stream of colour c+1 overlaps the tail of
//     colour c (programmatic dependent launch) and only the x gathers wait for it;
//   * a thread then issues all of its row's x gathers at once (one L2 round trip instead
//     of seven) and subtracts the products in stored order.
#pragma once

#include <cstdint>

#include "pf_kernels.cuh"

namespace pf {

constexpr int kTmaMaxGroups = 7;  // rows of up to 28 stored entries (Q1: 27, rotated Q1: 11)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Bytes per stored entry of the staged value stream (columns are 4 more).
template <int kVK>
constexpr int tma_vbytes() {
  return vk_kind<kVK>() == 0 ? 8 : vk_kind<kVK>() == 2 ? 2 : 1;
}

// Shared-memory layout of one stage (one SELL slice of width <= w entries): row lengths
// [32 int32], columns [32 w int32], values [32 w x vbytes].
struct TmaStageLayout {
  uint32_t cols_off, vals_off, bytes;
};
__host__ __device__ inline TmaStageLayout tma_layout(int w, int vbytes) {
  TmaStageLayout L;
  L.cols_off = 128u;
  L.vals_off = L.cols_off + static_cast<uint32_t>(4 * 32 * w);
  L.bytes = (L.vals_off + static_cast<uint32_t>(vbytes * 32 * w) + 127u) & ~127u;
  return L;
}

// Rows [row0, row1) of one colour; SELL slices s_lo .. s_hi-1 cover them (the first and
// last may hold rows of neighbouring colours, which are skipped).  width = the widest
// slice of the level (entries, multiple of 4, <= 4 kTmaMaxGroups).  Every warp runs its
// own pipeline over the slices warp_id, warp_id + n_warps, ... (n_warps = all warps of the
// grid): lane 0 keeps kTmaStages slices in flight, each landing on the stage's mbarrier;
// the 32 lanes relax the slice's 32 rows, one row each.
template <bool kSor, int kVK, int kTmaWarps, int kTmaStages>
__global__ void __launch_bounds__(32 * kTmaWarps) k_color_sweep_tma(SellView A, double* x, const double* __restrict__ b,
                                                                     int32_t row0, int32_t row1, double omega,
                                                                     int32_t width) {
  constexpr int VB = tma_vbytes<kVK>();
  extern __shared__ __align__(128) unsigned char tma_smem[];
  __shared__ __align__(8) uint64_t full[kTmaWarps][kTmaStages];
  __shared__ int32_t len_pad[kTmaWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TmaStageLayout lay = tma_layout(width, VB);
  unsigned char* mine = tma_smem + static_cast<size_t>(warp) * kTmaStages * lay.bytes;
  const int32_t s_lo = row0 >> 5, s_hi = ((row1 - 1) >> 5) + 1;
  const int32_t stride = static_cast<int32_t>(gridDim.x) * kTmaWarps;
  const int32_t first = s_lo + static_cast<int32_t>(blockIdx.x) * kTmaWarps + warp;
  (void)len_pad;
  // slice k of this warp = first + k * stride, into stage k % kTmaStages.  Lane 0 keeps
  // the slice pointers of the next slice to issue in registers, loaded one slice ahead, so
  // an issue never waits for them.
  int64_t nx0 = 0, nx1 = 0;
  auto fetch_ptr = [&](int k) {
    const int32_t sl = first + k * stride;
    if (sl < s_hi) {
      nx0 = A.slice_ptr[sl];
      nx1 = A.slice_ptr[sl + 1];
    }
  };
  auto issue = [&](int k) {
    const int32_t sl = first + k * stride;
    if (sl >= s_hi) return;
    const int64_t e0 = nx0;
    const uint32_t ne = static_cast<uint32_t>(nx1 - e0);
    unsigned char* buf = mine + static_cast<size_t>(k % kTmaStages) * lay.bytes;
    uint64_t* bar = &full[warp][k % kTmaStages];
    mbar_expect_tx(bar, 128u + 4u * ne + static_cast<uint32_t>(VB) * ne);
    bulk_g2s(buf, A.row_len + static_cast<int64_t>(sl) * 32, 128u, bar);
    bulk_g2s(buf + lay.cols_off, A.cols + e0, 4u * ne, bar);
    if constexpr (vk_kind<kVK>() == 0)
      bulk_g2s(buf + lay.vals_off, A.vals + e0, 8u * ne, bar);
    else if constexpr (vk_kind<kVK>() == 2)
      bulk_g2s(buf + lay.vals_off, static_cast<const unsigned short*>(A.vidx) + e0, 2u * ne, bar);
    else
      bulk_g2s(buf + lay.vals_off, static_cast<const unsigned char*>(A.vidx) + e0, ne, bar);
  };
  if (lane == 0) {
    for (int st = 0; st < kTmaStages; ++st) mbar_init(&full[warp][st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the level operator never changes after upload: stream it before the predecessor ends
    for (int k = 0; k < kTmaStages; ++k) {
      fetch_ptr(k);
      issue(k);
    }
    fetch_ptr(kTmaStages);
  }
  vtab_stage<kVK>(A);  // (a __syncthreads when the value table goes to shared memory)
  __syncwarp();
  PF_PDL_ENTRY();
  for (int k = 0;; ++k) {
    const int32_t sl = first + k * stride;
    if (sl >= s_hi) break;
    mbar_wait(&full[warp][k % kTmaStages], static_cast<uint32_t>((k / kTmaStages) & 1));
    const unsigned char* buf = mine + static_cast<size_t>(k % kTmaStages) * lay.bytes;
    const int32_t row = sl * 32 + lane;
    if (row >= row0 && row < row1) {
      const int len = reinterpret_cast<const int32_t*>(buf)[lane];
      // entry j of this lane: 128 (j/4) + 4 lane + j%4 inside the slice
      const int32_t soff = 4 * lane;
      const int32_t* scol = reinterpret_cast<const int32_t*>(buf + lay.cols_off) + soff;
      int32_t c[4 * kTmaMaxGroups];
      double xv[4 * kTmaMaxGroups];
#pragma unroll
      for (int g = 0; g < kTmaMaxGroups; ++g) {
        if (4 * g < len) {
          const int4 cc = *reinterpret_cast<const int4*>(scol + 128 * g);
          c[4 * g] = cc.x;
          c[4 * g + 1] = cc.y;
          c[4 * g + 2] = cc.z;
          c[4 * g + 3] = cc.w;
        }
      }
      // every gather of the row in flight at once (other colours are read-only during
      // this launch; the row's own entry is the diagonal and not gathered)
#pragma unroll
      for (int j = 0; j < 4 * kTmaMaxGroups; ++j)
        if (j < len && c[j] != row) xv[j] = __ldg(x + c[j]);
      double acc = b[row], diag = 0.0;
#pragma unroll
      for (int j = 0; j < 4 * kTmaMaxGroups; ++j) {
        if (j < len) {
          const int32_t e = soff + 128 * (j / 4) + (j & 3);
          double v;
          if constexpr (vk_kind<kVK>() == 0)
            v = reinterpret_cast<const double*>(buf + lay.vals_off)[e];
          else if constexpr (vk_kind<kVK>() == 2)
            v = __ldg(A.table + reinterpret_cast<const unsigned short*>(buf + lay.vals_off)[e]);
          else if constexpr (vk_kind<kVK>() == kVKSmem)
            v = s_vtab[(buf + lay.vals_off)[e]];
          else
            v = __ldg(A.table + (buf + lay.vals_off)[e]);
          if (c[j] == row)
            diag = v;
          else
            acc = __dsub_rn(acc, __dmul_rn(v, xv[j]));
        }
      }
      if (kSor)
        x[row] = __dadd_rn(__dmul_rn(1.0 - omega, x[row]), __ddiv_rn(__dmul_rn(omega, acc), diag));
      else
        x[row] = __ddiv_rn(acc, diag);
    }
    __syncwarp();  // the warp is done with this stage
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k + kTmaStages);
      fetch_ptr(k + kTmaStages + 1);
    }
  }
}

}  // namespace pf
