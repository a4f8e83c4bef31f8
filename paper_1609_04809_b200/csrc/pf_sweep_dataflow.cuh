// pf_sweep_dataflow.cuh — multicolour Gauss-Seidel / SOR as ONE dataflow launch.
//
// Same rows, same arithmetic and the same per-row summation order as the per-colour
// k_color_sweep launches (one_local_sweep, solvers.cpp:21-34, with the omega blend), so the
// result is bit-identical; only the schedule changes.
//
// The per-colour schedule runs S sweeps x C colours as S*C dependent launches.  Each colour
// is ~1.7 waves of latency-bound rows with a ramp and a tail, and on a level whose x
// outgrows L2 every colour pass re-reads x from HBM (it gathers from all other colours
// across the whole lattice).  Here the colour passes of a whole smoothing phase form one
// task graph: task (n, k) relaxes chunk k (kBlock consecutive rows) of colour pass n
// (colour n % C of sweep n / C).  Own rows are colour-major and each colour is in lattice
// order, so the neighbours of chunk k of one colour lie within chunks k - W .. k + W of
// every other colour (W measured from the operator at upload).  A task needs the chunks
// [k - W, k + W] of pass n - 1 finished; transitively that finishes every earlier pass's
// neighbours (new values for the lower colours) and every reader of this chunk's old
// values (passes n - 7 .. n - 1 touch it only within the same band), so the order of
// updates equals the per-colour launches'.  Tasks are claimed in the order t = k + (W+1) n
// (a tilted wavefront: every dependency is claimed earlier, so a persistent grid cannot
// deadlock), the resident blocks work on one lattice slab of all colours at once (x stays
// in L2), and completion is signalled through per-task epoch flags (release / acquire at
// GPU scope) instead of grid-wide barriers.
#pragma once

#include <cstdint>

#include "pf_kernels.cuh"

namespace pf {

constexpr int kDfTaskBits = 20;  // task word: pass n << 20 | chunk k
constexpr int kDfMaxColors = 8;

struct DataflowView {
  const int32_t* tasks;    // n_tasks words in claim order
  int32_t n_tasks;
  int32_t n_colors;
  int32_t w;               // neighbour reach in chunks
  int32_t kmax;            // chunks of the largest colour (flag row stride)
  int32_t cs[kDfMaxColors + 1];  // colour starts over the own rows
  int32_t kc[kDfMaxColors];      // chunks per colour
  uint32_t* flags;         // [passes][kmax]: epoch of the launch that finished the task
  uint32_t* ctl;           // [0] next task, [1] epoch, [2] finish ticket
};

__device__ __forceinline__ uint32_t df_ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void df_st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <bool kSor, int kVK>
__global__ void __launch_bounds__(kBlock, PF_SOR_MINB) k_color_sweep_dataflow(SellView A, double* x,
                                                                             const double* __restrict__ b,
                                                                             DataflowView d, double omega) {
  vtab_stage<kVK>(A);
  PF_PDL_ENTRY();
  __shared__ int32_t s_task;
  __shared__ uint32_t s_epoch;
  __shared__ int32_t s_cs[kDfMaxColors + 1], s_kc[kDfMaxColors];  // indexed by colour
  if (threadIdx.x == 0) {
    s_epoch = *reinterpret_cast<volatile uint32_t*>(&d.ctl[1]);
#pragma unroll
    for (int i = 0; i <= kDfMaxColors; ++i) s_cs[i] = d.cs[i];  // constant indices: stays in params
#pragma unroll
    for (int i = 0; i < kDfMaxColors; ++i) s_kc[i] = d.kc[i];
  }
  for (;;) {
    if (threadIdx.x == 0) s_task = static_cast<int32_t>(atomicAdd(&d.ctl[0], 1u));
    __syncthreads();
    const int32_t id = s_task;
    const uint32_t epoch = s_epoch;
    if (id >= d.n_tasks) break;
    const int32_t word = d.tasks[id];
    const int32_t n = word >> kDfTaskBits, k = word & ((1 << kDfTaskBits) - 1);
    const int32_t c = n % d.n_colors;
    if (n > 0 && threadIdx.x < 32) {  // chunks k - w .. k + w of pass n - 1 are done
      const int32_t cp = (n - 1) % d.n_colors;
      const int32_t lo = max(0, k - d.w), hi = min(s_kc[cp] - 1, k + d.w);
      const uint32_t* f = d.flags + static_cast<int64_t>(n - 1) * d.kmax;
      for (int32_t j = lo + static_cast<int32_t>(threadIdx.x); j <= hi; j += 32)
        while (df_ld_acquire(f + j) != epoch) __nanosleep(20);
      __syncwarp();
    }
    __syncthreads();
    const int32_t row = s_cs[c] + k * kBlock + static_cast<int32_t>(threadIdx.x);
    if (row < s_cs[c + 1]) {
      double acc = b[row], diag = 0.0;
      // x is written by other blocks of this launch: coherent loads (no read-only path)
      row_offdiag<false, false, kVK, kSorChunkGroups>(A, row, x, acc, diag);
      if (kSor)
        x[row] = __dadd_rn(__dmul_rn(1.0 - omega, x[row]), __ddiv_rn(__dmul_rn(omega, acc), diag));
      else
        x[row] = __ddiv_rn(acc, diag);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      df_st_release(d.flags + static_cast<int64_t>(n) * d.kmax + k, epoch);
    }
  }
  // the last block out resets the queue and moves to the next epoch (the next launch of
  // this level is stream-ordered after this one)
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&d.ctl[2], 1u) == gridDim.x - 1) {
      d.ctl[0] = 0;
      d.ctl[2] = 0;
      __threadfence();
      atomicAdd(&d.ctl[1], 1u);
    }
  }
}

}  // namespace pf
