// pf_bottom.cuh — the bottom of the V-cycle in one cooperative persistent kernel.
//
// Levels 0..Lc of the hierarchy are tiny: at C2 they hold 27, 125, 729, 4,913 and
// 35,937 dofs.  Run as separate launches, every phase of cycle() on them is one
// latency-bound kernel (launch + a chain of dependent L2 round trips), so the five
// bottom levels cost ~30 % of a V-cycle while holding 1.7 % of the dofs.  k_bottom runs
// the whole of cycle(Lc) (multigrid.cpp:150-190) — pre-smoothing, halo refreshes,
// residual, restriction, master/slave accumulate, the coarse Gauss-Seidel, prolongation,
// post-smoothing — in one launch, with a grid barrier between dependent phases.  Every
// phase runs the same per-row code as the standalone kernels (row_offdiag / row_dot,
// separate rounding, reference entry order), so the result is bit-identical to the
// multi-launch path; only the launch structure changes.
//
// The launch is cooperative (all blocks co-resident), which is what makes the grid
// barrier legal; blocks never wait on another launch.
#pragma once

#include <cooperative_groups.h>

#include "pf_bottom_types.hpp"
#include "pf_kernels.cuh"

namespace pf {

namespace cg = cooperative_groups;

// Latency-oriented row routines for the bottom levels, where each phase is a chain of
// dependent L2 round trips rather than a bandwidth problem: all entries of a row (up to
// kBotChunk) are loaded in one round, then all x gathers in one round.  Same operations
// in the same order as row_offdiag / row_dot, so results are bit-identical.
// (kBotChunk: pf_bottom_types.hpp)

__device__ __forceinline__ void bot_row_offdiag(const SellView& A, int32_t row, const double* x, double& acc,
                                                double& diag) {
  const int64_t base = sell_row_base(A.slice_ptr, row);
  const int len = A.row_len[row];
  if (len > kBotChunk) {  // long rows (never staged): the bandwidth kernel's loop
    row_offdiag<false, false, -1>(A, row, x, acc, diag);
    return;
  }
  int32_t c[kBotChunk];
  double v[kBotChunk], xv[kBotChunk];
  if (A.vkind == 1) {  // 8-bit value index (the staged levels)
    const unsigned char* vi = static_cast<const unsigned char*>(A.vidx);
#pragma unroll
    for (int k = 0; k < kBotChunk; ++k) {
      const int64_t e = sell_entry(base, k < len ? k : 0);
      c[k] = A.cols[e];
      v[k] = A.table[vi[e]];
    }
  } else {  // fp64 (decoded copies of the unstaged levels)
#pragma unroll
    for (int k = 0; k < kBotChunk; ++k) {
      const int64_t e = sell_entry(base, k < len ? k : 0);
      c[k] = A.cols[e];
      v[k] = A.vals[e];
    }
  }
#pragma unroll
  for (int k = 0; k < kBotChunk; ++k) xv[k] = x[c[k]];
#pragma unroll
  for (int k = 0; k < kBotChunk; ++k)
    if (k < len) {
      if (c[k] == row)
        diag = v[k];
      else
        acc = __dsub_rn(acc, __dmul_rn(v[k], xv[k]));
    }
}

// (measured: the 28-wide unrolled form that helps the sweeps makes the residual,
// restriction and prolongation phases 2-3x slower; they keep the bandwidth loop)
// A staged operator (shared memory: generic loads, latency ~30 cycles) takes a plain
// entry loop; the global ones the bandwidth kernel's group loop.
__device__ __forceinline__ double bot_row_dot(const SellView& A, int32_t row, const double* x, double acc) {
  if (!__isShared(A.cols)) return row_dot<false, false, -1>(A, row, x, acc);
  const int64_t base = sell_row_base(A.slice_ptr, row);
  const int len = A.row_len[row];
  if (len == 0) return acc;  // (an empty row may sit in an all-empty slice: no entry to read)
  if (len <= kBotChunk) {  // every load of the row first, then the products in stored order
    int32_t c[kBotChunk];
    double v[kBotChunk], xv[kBotChunk];
    const unsigned char* vi = static_cast<const unsigned char*>(A.vidx);
#pragma unroll
    for (int k = 0; k < kBotChunk; ++k) {
      const int64_t e = sell_entry(base, k < len ? k : 0);
      c[k] = A.cols[e];
      v[k] = A.vkind == 1 ? A.table[vi[e]] : A.vals[e];
    }
#pragma unroll
    for (int k = 0; k < kBotChunk; ++k) xv[k] = x[c[k]];
#pragma unroll
    for (int k = 0; k < kBotChunk; ++k)
      if (k < len) acc = __dadd_rn(acc, __dmul_rn(v[k], xv[k]));
    return acc;
  }
  if (A.vkind == 1) {
    const unsigned char* vi = static_cast<const unsigned char*>(A.vidx);
    for (int j = 0; j < len; ++j) {
      const int64_t e = sell_entry(base, j);
      acc = __dadd_rn(acc, __dmul_rn(A.table[vi[e]], x[A.cols[e]]));
    }
  } else {
    for (int j = 0; j < len; ++j) {
      const int64_t e = sell_entry(base, j);
      acc = __dadd_rn(acc, __dmul_rn(A.vals[e], x[A.cols[e]]));
    }
  }
  return acc;
}

// Point block 0's descriptor copy at the staged arena (pointers into the blob move to the
// arena; the staged levels' vectors get their arena slots).
template <class P>
__device__ __forceinline__ void bot_reloc(P& p, const unsigned char* lo, const unsigned char* hi,
                                          unsigned char* arena) {
  const unsigned char* q = reinterpret_cast<const unsigned char*>(p);
  if (q >= lo && q < hi) p = reinterpret_cast<P>(arena + (q - lo));
}
__device__ __forceinline__ void bot_reloc_view(SellView& A, const unsigned char* lo, const unsigned char* hi,
                                               unsigned char* arena) {
  bot_reloc(A.vals, lo, hi, arena);
  bot_reloc(A.cols, lo, hi, arena);
  bot_reloc(A.slice_ptr, lo, hi, arena);
  bot_reloc(A.row_len, lo, hi, arena);
  bot_reloc(A.vidx, lo, hi, arena);
  bot_reloc(A.table, lo, hi, arena);
}
static __device__ void bot_relocate(BotDesc& D, unsigned char* arena) {
  const unsigned char* lo = D.stage.blob;
  const unsigned char* hi = lo + D.stage.blob_bytes;
  for (int l = 0; l <= D.stage.hs; ++l) {
    BotLevel& L = D.lev[l];
    L.x = reinterpret_cast<double*>(arena + D.stage.vec_off[l][0]);
    L.xa = reinterpret_cast<double*>(arena + D.stage.vec_off[l][1]);
    L.b = reinterpret_cast<double*>(arena + D.stage.vec_off[l][2]);
    L.r = reinterpret_cast<double*>(arena + D.stage.vec_off[l][3]);
    for (BotPlan* pl : {&L.ms, &L.h1, &L.h2}) {
      bot_reloc(pl->dst, lo, hi, arena);
      bot_reloc(pl->src, lo, hi, arena);
    }
    bot_reloc(L.acc_off, lo, hi, arena);
    bot_reloc(L.acc_src, lo, hi, arena);
    bot_reloc(L.acc_dst, lo, hi, arena);
    for (int s = 0; s < D.n_sub; ++s) {
      BotSub& S = D.sub[l][s];
      bot_reloc_view(S.A, lo, hi, arena);
      bot_reloc_view(S.P, lo, hi, arena);
      bot_reloc_view(S.R, lo, hi, arena);
      bot_reloc(S.color_start, lo, hi, arena);
      bot_reloc(S.is_dir, lo, hi, arena);
    }
  }
}

// grid barrier + optional phase timestamp (block 0, thread 0)
__device__ __forceinline__ void bsync(cg::grid_group& g, const BotDesc& D, int& phase) {
  g.sync();
  if (D.stamps && blockIdx.x == 0 && threadIdx.x == 0 && phase < 127) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    D.stamps[++phase] = t;
  }
}

// A team is whoever executes a phase: the whole grid (grid barrier between phases) or,
// for the tiniest levels, block 0 alone (__syncthreads, ~20x cheaper than a grid barrier).
struct GridTeam {
  cg::grid_group g;
  int64_t t, stride;
  __device__ void sync(const BotDesc& D, int& ph) { bsync(g, D, ph); }
};
struct BlockTeam {
  int64_t t, stride;
  __device__ void sync(const BotDesc& D, int& ph) {
    __syncthreads();
    // PF_BOTTOM_PROFILE: block-phase timestamps in stamps[128..254]
    if (D.stamps && t == 0 && ph < 126) {
      unsigned long long ts;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
      D.stamps[128 + ++ph] = ts;
    }
  }
};

__device__ __forceinline__ int bot_find(const BotDesc& D, int l, int32_t row) {
  int s = D.n_sub - 1;
  while (s > 0 && row < D.sub[l][s].off) --s;
  return s;
}

__device__ __forceinline__ void bot_copy_plan(const BotPlan& P, double* v, int64_t t, int64_t stride) {
  for (int64_t i = t; i < P.n; i += stride) v[P.dst[i]] = v[P.src[i]];
}

template <class Team, int kKind = -1>  // kKind: the smoother when known at compile time
__device__ void bot_smooth(const BotDesc& D, int l, const BotCfg& c, int sweeps, Team& T, int& ph) {
  const int kind = kKind >= 0 ? kKind : c.kind;
  const int64_t t = T.t, stride = T.stride;
  const BotLevel& L = D.lev[l];
  double* bufs[2] = {L.x, L.xa};
  int cur = 0;
  for (int sw = 0; sw < sweeps; ++sw) {
    for (int loc = 0; loc < c.local_sweeps; ++loc) {
      if (kind == 0) {  // damped Jacobi, ping-pong (k_jacobi)
        const double* src = bufs[cur];
        double* dst = bufs[cur ^ 1];
        for (int64_t r = t; r < L.total; r += stride) {
          const BotSub& S = D.sub[l][bot_find(D, l, static_cast<int32_t>(r))];
          const int32_t lr = static_cast<int32_t>(r - S.off);
          const double xo = src[r];
          if (lr >= S.n_own) {  // non-own rows (and replica padding) carry over
            dst[r] = xo;
            continue;
          }
          double acc = L.b[r], diag = 0.0;
          bot_row_offdiag(S.A, lr, src + S.off, acc, diag);
          dst[r] = __dadd_rn(__dmul_rn(1.0 - c.omega, xo), __ddiv_rn(__dmul_rn(c.omega, acc), diag));
        }
        cur ^= 1;
        T.sync(D, ph);
      } else {  // coloured GS / SOR, in place (k_color_sweep)
        const bool sor = kind == 2;
        double* x = bufs[cur];
        for (int col = 0; col < L.max_colors; ++col) {
          for (int s = 0; s < D.n_sub; ++s) {
            const BotSub& S = D.sub[l][s];
            if (col >= S.n_colors) continue;
            const int32_t r0 = S.color_start[col], r1 = S.color_start[col + 1];
            double* xs = x + S.off;
            const double* bs = L.b + S.off;
            for (int64_t lr = r0 + t; lr < r1; lr += stride) {
              const int32_t row = static_cast<int32_t>(lr);
              double acc = bs[row], diag = 0.0;
              bot_row_offdiag(S.A, row, xs, acc, diag);
              xs[row] = sor ? __dadd_rn(__dmul_rn(1.0 - c.omega, xs[row]),
                                        __ddiv_rn(__dmul_rn(c.omega, acc), diag))
                            : __ddiv_rn(acc, diag);
            }
          }
          T.sync(D, ph);
          // colour-wise exchange: every copy refreshed before the next colour (the
          // sweep's own exchange follows the last colour of the last local sweep)
          if (c.colorwise && !(loc + 1 == c.local_sweeps && col + 1 == L.max_colors)) {
            if (L.ms.n) {
              bot_copy_plan(L.ms, x, t, stride);
              T.sync(D, ph);
            }
            if (L.h1.n) {
              bot_copy_plan(L.h1, x, t, stride);
              T.sync(D, ph);
            }
          }
        }
      }
    }
    if (L.ms.n) {
      bot_copy_plan(L.ms, bufs[cur], t, stride);
      T.sync(D, ph);
    }
    if (L.h1.n) {
      bot_copy_plan(L.h1, bufs[cur], t, stride);
      T.sync(D, ph);
    }
  }
  if (cur) {
    for (int64_t r = t; r < L.total; r += stride) L.x[r] = L.xa[r];
    T.sync(D, ph);
  }
}

// master/slave AccumulateThenScatter on level l (fecomm.cpp:41-62)
template <class Team>
__device__ void bot_accumulate_scatter(const BotDesc& D, int l, double* v, Team& T, int& ph) {
  const int64_t t = T.t, stride = T.stride;
  const BotLevel& L = D.lev[l];
  if (L.acc_n) {
    for (int64_t m = t; m < L.acc_n; m += stride) {
      double acc = v[L.acc_dst[m]];
      for (int32_t e = L.acc_off[m]; e < L.acc_off[m + 1]; ++e) acc = __dadd_rn(acc, v[L.acc_src[e]]);
      v[L.acc_dst[m]] = acc;
    }
    T.sync(D, ph);
  }
  if (L.ms.n) {
    bot_copy_plan(L.ms, v, t, stride);
    T.sync(D, ph);
  }
}

// Descending half of cycle(l) (multigrid.cpp:160-179): pre-smooth, halo2, residual,
// restriction to l-1 (Dirichlet zeroed, coarse x = 0), master/slave accumulate on l-1.
template <class Team, int kKind = -1>
__device__ void bot_descend(const BotDesc& D, int l, const BotCfg& c, Team& T, int& ph) {
  const int64_t t = T.t, stride = T.stride;
  const BotLevel& L = D.lev[l];
  bot_smooth<Team, kKind>(D, l, c, c.pre, T, ph);
  if (L.h2.n) {
    bot_copy_plan(L.h2, L.x, t, stride);
    T.sync(D, ph);
  }
  for (int64_t r = t; r < L.total; r += stride) {  // r = b - A x on every row (k_residual)
    const BotSub& S = D.sub[l][bot_find(D, l, static_cast<int32_t>(r))];
    const int32_t lr = static_cast<int32_t>(r - S.off);
    if (lr >= S.n) continue;  // padding of a replicated (strided) level
    L.r[r] = __dsub_rn(L.b[r], bot_row_dot(S.A, lr, L.x + S.off, 0.0));
  }
  T.sync(D, ph);
  const BotLevel& C = D.lev[l - 1];
  for (int64_t pr = t; pr < C.total; pr += stride) {  // b_c = R r (k_restrict)
    const int s = bot_find(D, l - 1, static_cast<int32_t>(pr));
    const BotSub& F = D.sub[l][s];
    const BotSub& Sc = D.sub[l - 1][s];
    const int32_t lr = static_cast<int32_t>(pr - Sc.off);
    if (lr >= Sc.n) continue;
    const double acc = bot_row_dot(F.R, lr, L.r + F.off, 0.0);
    C.b[pr] = Sc.is_dir[lr] ? 0.0 : acc;
    C.x[pr] = 0.0;
  }
  T.sync(D, ph);
  bot_accumulate_scatter(D, l - 1, C.b, T, ph);
}

// Ascending half of cycle(l) (multigrid.cpp:183-189): x += P x_c, post-smooth, halo2.
template <class Team, int kKind = -1>
__device__ void bot_ascend(const BotDesc& D, int l, const BotCfg& c, Team& T, int& ph) {
  const int64_t t = T.t, stride = T.stride;
  const BotLevel& L = D.lev[l];
  const BotLevel& C = D.lev[l - 1];
  for (int64_t r = t; r < L.total; r += stride) {
    const int s = bot_find(D, l, static_cast<int32_t>(r));
    const BotSub& S = D.sub[l][s];
    const int32_t lr = static_cast<int32_t>(r - S.off);
    if (lr >= S.n) continue;
    const double acc = bot_row_dot(S.P, lr, C.x + D.sub[l - 1][s].off, 0.0);
    L.x[r] = __dadd_rn(L.x[r], acc);
  }
  T.sync(D, ph);
  bot_smooth<Team, kKind>(D, l, c, c.post, T, ph);
  if (L.h2.n) {
    bot_copy_plan(L.h2, L.x, t, stride);
    T.sync(D, ph);
  }
}

// Level 0: coarse_solve + update_halo2 (multigrid.cpp:153-158).  Block 0 runs the
// shared-memory solve; every thread of the team then meets at the team barrier.
template <class Team>
__device__ void bot_coarse(const BotDesc& D, const BotCfg& c, Team& T, int& ph, unsigned char* smem_coarse) {
  const BotLevel& L0 = D.lev[0];
  if (blockIdx.x == 0)
    coarse_gs_smem(D.coarse, L0.x, L0.b, c.coarse_tol, c.coarse_max_iter, D.coarse_stats, smem_coarse);
  T.sync(D, ph);
  if (L0.h2.n) {
    bot_copy_plan(L0.h2, L0.x, T.t, T.stride);
    T.sync(D, ph);
  }
}

// Block 0 (every thread): copy the staged blob into the arena and point block 0's descriptor
// at it (no-op unless levels 0..bt are staged).  stage_in_vectors then moves the interface
// level bt's b and x in (after griddepcontrol.wait / the grid barrier that produced them),
// stage_out its x back to global memory at the end of the block section.
struct BotIo {
  double* gx;        // level bt's x / b in global memory
  const double* gb;
  int32_t n;
  bool staged, io;   // levels 0..bt staged; bt itself staged (interface copies needed)
};
static __device__ BotIo bot_stage_operators(BotDesc& DB, unsigned char* smem_b, int bt) {
  BotIo io{DB.lev[bt].x, DB.lev[bt].b, DB.lev[bt].total, DB.stage.hs >= 0 && bt == DB.block_top, false};
  io.io = io.staged && DB.stage.hs == bt;
  if (!io.staged) return io;
  unsigned char* arena = smem_b + DB.stage.smem_off;
  __syncthreads();  // everyone has read the global interface pointers
  const int4* src = reinterpret_cast<const int4*>(DB.stage.blob);
  int4* dst = reinterpret_cast<int4*>(arena);
  for (int64_t i = threadIdx.x; i < DB.stage.blob_bytes / 16; i += blockDim.x) dst[i] = src[i];
  if (threadIdx.x == 0) bot_relocate(DB, arena);
  __syncthreads();
  return io;
}
static __device__ void bot_stage_in_vectors(BotDesc& DB, const BotIo& io, int bt) {
  if (!io.io) return;
  for (int32_t i = threadIdx.x; i < io.n; i += blockDim.x) {
    DB.lev[bt].b[i] = io.gb[i];
    DB.lev[bt].x[i] = io.gx[i];
  }
  __syncthreads();
}
static __device__ void bot_stage_out(BotDesc& DB, const BotIo& io, int bt) {
  if (!io.io) return;
  __syncthreads();
  for (int32_t i = threadIdx.x; i < io.n; i += blockDim.x) io.gx[i] = DB.lev[bt].x[i];
}

// cycle(Lc) (multigrid.cpp:150-190) on levels 0..Lc.  On entry lev[Lc].b holds the
// restricted residual (Dirichlet entries zeroed, before the master/slave accumulate when
// `accumulate_top`) and lev[Lc].x is zero.  Levels above block_top run with the whole
// grid; levels 0..block_top (at most a few hundred rows each) run inside block 0.
static __global__ void __launch_bounds__(kBlock, 1) k_bottom(const BotDesc* __restrict__ Dp, BotCfg c,
                                                      int accumulate_top) {
  PF_PDL_ENTRY();
  // The descriptor is read on every row of every phase: keep a per-block copy in
  // shared memory (the grid barrier invalidates L1, so global reads would go to L2).
  extern __shared__ __align__(16) unsigned char smem_b[];
  {
    const uint64_t* src = reinterpret_cast<const uint64_t*>(Dp);
    uint64_t* dst = reinterpret_cast<uint64_t*>(smem_b);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(BotDesc) / 8); i += blockDim.x) dst[i] = src[i];
    __syncthreads();
  }
  const BotDesc& D = *reinterpret_cast<const BotDesc*>(smem_b);
  unsigned char* smem_coarse = smem_b + ((sizeof(BotDesc) + 15) / 16) * 16;
  GridTeam G{cg::this_grid(), static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x,
             static_cast<int64_t>(gridDim.x) * blockDim.x};
  const int top = D.n_levels - 1;
  int ph = 0;
  if (D.stamps && G.t == 0) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    D.stamps[0] = t0;
  }
  for (int i = 0; i < c.calib; ++i) G.sync(D, ph);
  if (accumulate_top) bot_accumulate_scatter(D, top, D.lev[top].b, G, ph);
  const int bt = c.block_top < D.block_top ? c.block_top : D.block_top;
  for (int l = top; l > bt && l >= 1; --l) bot_descend(D, l, c, G, ph);
  if (bt >= 0) {
    if (blockIdx.x == 0) {
      BotDesc& DB = *reinterpret_cast<BotDesc*>(smem_b);  // block 0's own copy
      const BotIo io = bot_stage_operators(DB, smem_b, bt);
      bot_stage_in_vectors(DB, io, bt);
      BlockTeam B{threadIdx.x, blockDim.x};
      int bph = 0;
      if (D.stamps && threadIdx.x == 0) {
        unsigned long long ts;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
        D.stamps[128] = ts;
      }
      for (int l = bt; l >= 1; --l) bot_descend(D, l, c, B, bph);
      bot_coarse(D, c, B, bph, smem_coarse);
      for (int l = 1; l <= bt; ++l) bot_ascend(D, l, c, B, bph);
      bot_stage_out(DB, io, bt);
    }
    G.sync(D, ph);
  } else {
    bot_coarse(D, c, G, ph, smem_coarse);
  }
  for (int l = (bt >= 0 ? bt + 1 : 1); l <= top; ++l) bot_ascend(D, l, c, G, ph);
  if (D.stamps && G.t == 0) D.stamps[255] = static_cast<unsigned long long>(ph);
}

// Every bottom level staged (BotDesc::stage.hs == top == block_top): the whole bottom
// cycle in ONE block, with the smoother known at compile time — a fraction of k_bottom's
// code (no grid-team paths), launched as an ordinary PDL-chained kernel of one block.  The
// descriptor and the staged operators are copied before griddepcontrol.wait (immutable),
// the top level's b and x after it.
#ifndef PF_BOT_BLOCK_THREADS
#define PF_BOT_BLOCK_THREADS 256
#endif
constexpr int kBotBlockThreads = PF_BOT_BLOCK_THREADS;
template <int kKind>
__global__ void __launch_bounds__(kBotBlockThreads, 1) k_bottom_block(const BotDesc* __restrict__ Dp, BotCfg c,
                                                            int accumulate_top) {
  extern __shared__ __align__(16) unsigned char smem_b[];
  {
    const uint64_t* src = reinterpret_cast<const uint64_t*>(Dp);
    uint64_t* dst = reinterpret_cast<uint64_t*>(smem_b);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(BotDesc) / 8); i += blockDim.x) dst[i] = src[i];
    __syncthreads();
  }
  BotDesc& DB = *reinterpret_cast<BotDesc*>(smem_b);
  const int top = DB.n_levels - 1;
  const BotIo io = bot_stage_operators(DB, smem_b, top);
  PF_PDL_ENTRY();
  bot_stage_in_vectors(DB, io, top);
  const BotDesc& D = DB;
  unsigned char* smem_coarse = smem_b + ((sizeof(BotDesc) + 15) / 16) * 16;
  BlockTeam B{threadIdx.x, blockDim.x};
  int ph = 0;
  if (D.stamps && threadIdx.x == 0) {
    unsigned long long ts;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
    D.stamps[128] = ts;
  }
  if (accumulate_top) bot_accumulate_scatter(D, top, D.lev[top].b, B, ph);
  for (int l = top; l >= 1; --l) bot_descend<BlockTeam, kKind>(D, l, c, B, ph);
  bot_coarse(D, c, B, ph, smem_coarse);
  for (int l = 1; l <= top; ++l) bot_ascend<BlockTeam, kKind>(D, l, c, B, ph);
  bot_stage_out(DB, io, top);
}

}  // namespace pf
