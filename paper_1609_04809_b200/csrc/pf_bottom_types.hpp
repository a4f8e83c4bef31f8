// pf_bottom_types.hpp — the bottom kernel's descriptor types (pf_bottom.cuh), shared with
// the host code that fills them (pf_build.cu).
#pragma once

#include <cstdint>

#include "pf_types.hpp"

namespace pf {

constexpr int kBotMaxLevels = 8;
constexpr int kBotMaxSubs = 8;
constexpr int kBotChunk = 28;  // widest row of the bottom's latency-oriented row routines (Q1: 27 entries)

struct BotSub {
  SellView A;
  const int32_t* host_of_own;
  const int32_t* color_start;  // n_colors + 1, subdomain-local device rows
  SellView P;                  // P of this level (rows: this level; cols: parent, local)
  SellView R;                  // R to the parent (rows: parent, local; cols: this level, local)
  const uint8_t* is_dir;
  int32_t n, n_own, n_colors;
  int32_t off;                 // position in the level vectors
};

struct BotPlan {
  const int32_t* dst;
  const int32_t* src;
  int32_t n;
};

struct BotLevel {
  double* x;   // primary
  double* xa;  // Jacobi ping-pong partner
  double* b;
  double* r;
  int32_t total;
  int32_t max_colors;
  BotPlan ms, h1, h2;
  const int32_t* acc_off;
  const int32_t* acc_src;
  const int32_t* acc_dst;
  int32_t acc_n;
};

// Shared-memory staging of the block levels (levels 0..hs <= block_top, which block 0 runs
// alone).  Their operators (SELL-32x4 with 8-bit value indices where the level has at
// most 256 distinct values), colour ranges, Dirichlet flags and exchange plans are copied
// at finalize into one global blob; the descriptor points into the blob.  At the start of
// the block section block 0 copies the blob into shared memory, points its own copy of the
// descriptor at it and gives the level vectors (x, xa, b, r) shared-memory slots, so every
// dependent load of the 70-odd phases of the tiny levels is a shared-memory access instead
// of an L2 round trip.  The blob is an exact copy, so the unstaged path (the same
// descriptor without relocation) computes the same values from global memory.
struct BotStage {
  const unsigned char* blob;
  int64_t blob_bytes;   // multiple of 16
  int64_t arena_bytes;  // blob + the staged levels' vectors
  int64_t smem_off;     // arena offset in the kernel's dynamic shared memory
  int hs;               // staged levels 0..hs (-1: none)
  int64_t vec_off[kBotMaxLevels][4];  // arena offsets of x, xa, b, r
};

struct BotDesc {
  int n_sub;
  int n_levels;   // Lc + 1
  int block_top;  // highest level small enough for block 0 alone (block barriers), -1: none
  unsigned long long* stamps;  // optional (PF_BOTTOM_PROFILE): globaltimer after each phase
  CoarsePack coarse;        // level 0 packed for the shared-memory coarse solve
  double* coarse_stats;
  BotLevel lev[kBotMaxLevels];
  BotSub sub[kBotMaxLevels][kBotMaxSubs];
  BotStage stage;
};

struct BotCfg {
  int kind, pre, post, local_sweeps, coarse_max_iter;
  double omega, coarse_tol;
  int block_top;  // levels 0..block_top inside block 0 (-1: none); chosen per smoother
  int calib;      // PF_BOTTOM_CALIB: empty grid-barrier phases first (profiling aid)
  int colorwise;  // coloured smoothers: master/slave + halo1 scatter after every colour
};

}  // namespace pf
