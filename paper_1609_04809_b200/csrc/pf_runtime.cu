// pf_runtime.cu — launches, CUDA graphs and the core C ABI of the B200 GMG V-cycle hot path
// (the device layout is built by pf_build.cu, the heat / operator / load ABI lives in
// pf_ops.cu; shared declarations in pf_internal.hpp).
//
// Maps the reference's hot-path API onto sm_100a kernels:
//   spmv / residual_norm            linalg.cpp:45-74     -> k_spmv / k_resnorm
//   smooth (Jacobi, GS)             solvers.cpp:17-68    -> k_jacobi / k_color_sweep
//   coarse_solve                    solvers.cpp:70-92    -> k_coarse_gs
//   prolongate / restrict_residual  multigrid.cpp:121-146 -> k_prolong_add / k_restrict
//   v_cycle / solve_outer           multigrid.cpp:150-246 -> one CUDA graph per outer cycle
//   ParFECommunicator updates       fecomm.cpp:25-72     -> exchange plans (device copies
//                                                           or NCCL send/recv)
//   allreduce_sum                   transport.cpp:139-165 -> ordered device sum
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <parallel/algorithm>
#include <unordered_set>
#include <omp.h>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <type_traits>
#include <unordered_map>
#include <sstream>
#include <string>
#include <vector>

#include "pf_bottom.cuh"
#include "pf_kernels.cuh"
#include "pf_nccl.hpp"
#include "pf_sweep_tma.cuh"
#include "pf_window.cuh"
#include "pf_internal.hpp"
#include "pf_runtime.hpp"

using namespace pf;


using namespace pf;

namespace pf {

thread_local std::string g_last_error;
void set_error(const char* m) { g_last_error = m; }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(PF_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

std::atomic<int64_t> g_guard_failures{0};
bool guard_on() {
  static const bool on = [] {
    const char* e = std::getenv("PF_GUARD");
    return e && std::atoi(e) != 0;
  }();
  return on;
}
void guard_check(const void* zone, size_t bytes) {
  unsigned char h[kGuardBytes];
  // (no device-wide synchronisation: in-process peer ranks may have kernels waiting on this
  // thread; the library synchronises its streams before it frees their buffers)
  if (cudaMemcpy(h, zone, kGuardBytes, cudaMemcpyDeviceToHost) != cudaSuccess) {
    (void)cudaGetLastError();
    return;  // a failed device (reported elsewhere), not a guard hit
  }
  size_t first = kGuardBytes;
  for (size_t i = 0; i < kGuardBytes && first == kGuardBytes; ++i)
    if (h[i] != 0xFF) first = i;
  if (first != kGuardBytes) {
    ++g_guard_failures;
    std::fprintf(stderr, "[pf guard] write past the end of a %zu-byte device buffer (first at +%zu)\n", bytes, first);
  }
}

namespace rt {

thread_local int64_t* g_capture_counter = nullptr;

double wall_now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int sm_count(int device) {
  static int cached[64] = {};
  if (device < 0 || device >= 64) device = 0;
  if (!cached[device]) PF_CUDA(cudaDeviceGetAttribute(&cached[device], cudaDevAttrMultiProcessorCount, device));
  return cached[device];
}

[[noreturn]] void invalid(const std::string& m) { throw Error(PF_ERR_INVALID_ARGUMENT, m); }

// PF_TRACE=1: one stderr line per major host step (debugging integrations).
void trace(const char* what, int rank) {
  static const bool on = std::getenv("PF_TRACE") != nullptr;
  if (!on) return;
  if (rank < 0) {
    std::fprintf(stderr, "[pf] %s\n", what);
  } else {
    const double t = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    std::fprintf(stderr, "[pf %.6f r%d] %s\n", t, rank, what);
  }
}
[[noreturn]] void state(const std::string& m) { throw Error(PF_ERR_STATE, m); }


// The option table: name (pf_hierarchy_set_option), environment variable, member, and
// whether it shapes the device layout (fixed by pf_hierarchy_finalize).
struct OptionSpec {
  const char* name;
  const char* env;
  int64_t Options::*field;
  bool build;
};
const OptionSpec kOptions[] = {
    {"value_index", "PF_VALUE_INDEX", &Options::value_index, true},
    {"value_index_min", "PF_VALUE_INDEX_MIN", &Options::value_index_min, true},
    {"vtab_smem", "PF_VTAB_SMEM", &Options::vtab_smem, true},
    {"cached_max_bytes", "PF_CACHED_MAX_BYTES", &Options::cached_max_bytes, true},
    {"interleave_min_bytes", "PF_INTERLEAVE_MIN_BYTES", &Options::interleave_min_bytes, true},
    {"bottom_rows", "PF_BOTTOM_ROWS", &Options::bottom_rows, true},
    {"bottom_block_rows", "PF_BOTTOM_BLOCK_ROWS", &Options::bottom_block_rows, true},
    {"bottom_grid", "PF_BOTTOM_GRID", &Options::bottom_grid, true},
    {"bottom_stage", "PF_BOTTOM_STAGE", &Options::bottom_stage, true},
    {"rep_bottom_rows", "PF_REP_BOTTOM_ROWS", &Options::rep_bottom_rows, true},
    {"bottom_jacobi", "PF_BOTTOM_JACOBI", &Options::bottom_jacobi, false},
    {"bottom_block_kernel", "PF_BOTTOM_BLOCK_KERNEL", &Options::bottom_block_kernel, false},
    {"split_row_len", "PF_SPLIT_ROW_LEN", &Options::split_row_len, false},
    {"split_max_rows", "PF_SPLIT_MAX_ROWS", &Options::split_max_rows, false},
    {"split_rows_max", "PF_SPLIT_ROWS_MAX", &Options::split_rows_max, false},
    {"wide_max_rows", "PF_WIDE_MAX_ROWS", &Options::wide_max_rows, false},
    {"fused_rr_rows", "PF_FUSED_RR_ROWS", &Options::fused_rr_rows, false},
    {"sor_tma", "PF_SOR_TMA", &Options::sor_tma, false},
    {"sor_tma_min_rows", "PF_SOR_TMA_MIN_ROWS", &Options::sor_tma_min_rows, false},
    {"sor_tma_bps", "PF_SOR_TMA_BPS", &Options::sor_tma_bps, false},
    {"sor_tma_cfg", "PF_SOR_TMA_CFG", &Options::sor_tma_cfg, false},
    {"win", "PF_WIN", &Options::win, true},
    {"win_min_rows", "PF_WIN_MIN_ROWS", &Options::win_min_rows, true},
    {"win_max_chunks", "PF_WIN_MAX_CHUNKS", &Options::win_max_chunks, true},
    {"win_kernels", "PF_WIN_KERNELS", &Options::win_kernels, false},
    {"solve_graph_if", "PF_SOLVE_GRAPH_IF", &Options::solve_graph_if, false},
    {"pdl", "PF_PDL", &Options::pdl, false},
    {"solve_mode_host", nullptr, &Options::solve_mode_host, false},  // env: PF_SOLVE_MODE=host
};

const OptionSpec* find_option(const char* name) {
  for (const OptionSpec& o : kOptions)
    if (name && std::strcmp(o.name, name) == 0) return &o;
  return nullptr;
}

Options options_from_env() {
  Options o;
  for (const OptionSpec& s : kOptions)
    if (s.env)
      if (const char* e = std::getenv(s.env)) o.*s.field = std::atoll(e);
  if (const char* e = std::getenv("PF_SOLVE_MODE")) o.solve_mode_host = std::string(e) == "host";
  return o;
}

size_t bottom_kernel_static_smem() {
  cudaFuncAttributes fa{};
  PF_CUDA(cudaFuncGetAttributes(&fa, k_bottom));
  return fa.sharedSizeBytes;
}
void bottom_kernel_caps(int device) {
  int optin = 0;
  PF_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  auto cap = [&](auto kern) {
    cudaFuncAttributes fa{};
    PF_CUDA(cudaFuncGetAttributes(&fa, kern));
    PF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 optin - static_cast<int>(fa.sharedSizeBytes)));
  };
  cap(k_bottom);
  cap(k_bottom_block<0>);
  cap(k_bottom_block<1>);
  cap(k_bottom_block<2>);
}
int bottom_kernel_occupancy(size_t smem) {
  int occ = 0;
  PF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bottom, kBlock, smem));
  return occ;
}

// ------------------------------------------------------------------ enqueue --

void enq_plan(pf_hierarchy* h, ExchangePlan& P, double* v, cudaStream_t st = nullptr);

void enq_scatter(pf_hierarchy* h, int l, int kind, double* v) { enq_plan(h, h->levels[l].scatter[kind], v); }

// Execute one exchange plan on stream st (default: the hierarchy's stream).
void enq_plan(pf_hierarchy* h, ExchangePlan& P, double* v, cudaStream_t st) {
  auto launch = launcher(h, st);
  if (!st) st = h->stream;
  if (h->world == h->n_sub) {
    if (P.n == 0) return;
    // pack, transport and unpack in one device copy: sends and receives of one
    // channel kind touch disjoint entries (masters/owners vs slaves/halos)
    launch(grid_for(P.n), kBlock, k_copy_idx, static_cast<const int32_t*>(P.src.p),
           static_cast<const int32_t*>(P.dst.p), v, static_cast<int32_t>(P.n));
    return;
  }
  // collective on every rank, even one with nothing to move on this channel
  if (!h->xport) state("multi-process hierarchy used before pf_hierarchy_init_nccl");
  if (h->xport->direct()) {  // one kernel: stores into the peers' staging, waits, scatters
    h->xport->run_plan(P, v, false, st);
    return;
  }
  launch(grid_for(P.pack_idx.n), kBlock, k_pack, static_cast<const double*>(v),
         static_cast<const int32_t*>(P.pack_idx.p), P.sendbuf.p, static_cast<int32_t>(P.pack_idx.n));
  h->xport->group_start();
  for (const PeerSeg& s : P.send_segs) h->xport->send(P.sendbuf.p + s.off, s.len, s.peer, st);
  for (const PeerSeg& s : P.recv_segs) h->xport->recv(P.recvbuf.p + s.off, s.len, s.peer, st);
  h->xport->group_end(st);
  launch(grid_for(P.unpack_idx.n), kBlock, k_unpack, static_cast<const double*>(P.recvbuf.p),
         static_cast<const int32_t*>(P.unpack_idx.p), v, static_cast<int32_t>(P.unpack_idx.n));
}

void enq_accumulate(pf_hierarchy* h, int l, double* v) {
  ExchangePlan& A = h->levels[l].accumulate;
  auto launch = launcher(h);
  if (h->world == h->n_sub) {
    if (A.n_masters == 0) return;
    launch(grid_for(A.n_masters), kBlock, k_unpack_accumulate, static_cast<const double*>(v),
           static_cast<const int32_t*>(A.acc_off.p), static_cast<const int32_t*>(A.acc_src.p),
           static_cast<const int32_t*>(A.acc_dst.p), v, A.n_masters);
    return;
  }
  if (!h->xport) state("multi-process hierarchy used before pf_hierarchy_init_nccl");
  if (h->xport->direct()) {  // partials stored into the masters' staging, summed there in peer order
    h->xport->run_plan(A, v, true, h->stream);
    launch(grid_for(A.n_masters), kBlock, k_unpack_accumulate, h->xport->staging(A),
           static_cast<const int32_t*>(A.acc_off.p), static_cast<const int32_t*>(A.acc_src.p),
           static_cast<const int32_t*>(A.acc_dst.p), v, A.n_masters);
    h->xport->ack_plan(A, h->stream);
    return;
  }
  launch(grid_for(A.pack_idx.n), kBlock, k_pack, static_cast<const double*>(v),
         static_cast<const int32_t*>(A.pack_idx.p), A.sendbuf.p, static_cast<int32_t>(A.pack_idx.n));
  h->xport->group_start();
  for (const PeerSeg& s : A.send_segs) h->xport->send(A.sendbuf.p + s.off, s.len, s.peer, h->stream);
  for (const PeerSeg& s : A.recv_segs) h->xport->recv(A.recvbuf.p + s.off, s.len, s.peer, h->stream);
  h->xport->group_end(h->stream);
  launch(grid_for(A.n_masters), kBlock, k_unpack_accumulate, static_cast<const double*>(A.recvbuf.p),
         static_cast<const int32_t*>(A.acc_off.p), static_cast<const int32_t*>(A.acc_src.p),
         static_cast<const int32_t*>(A.acc_dst.p), v, A.n_masters);
}

void enq_update_ms(pf_hierarchy* h, int l, double* v, int mode) {
  if (mode == PF_UPDATE_ACCUMULATE_THEN_SCATTER) enq_accumulate(h, l, v);
  enq_scatter(h, l, PF_CH_MASTER_SLAVE, v);
}

// ascending-rank allreduce of the per-subdomain sums in L.sumsq into L.norm
void enq_allreduce(pf_hierarchy* h, Level& L, bool take_sqrt) {
  auto launch = launcher(h);
  if (h->world == h->n_sub) {
    launch(1, 32, k_ordered_sum, static_cast<const double*>(L.sumsq.p), h->n_sub, L.norm.p,
           take_sqrt ? 1 : 0);
  } else {
    if (!h->xport) state("multi-process hierarchy used before pf_hierarchy_init_nccl");
    h->xport->allgather(L.sumsq.p, L.sumsq.p + 1, 1, h->stream);
    launch(1, 32, k_ordered_sum, static_cast<const double*>(L.sumsq.p + 1), h->world, L.norm.p,
           take_sqrt ? 1 : 0);
  }
}

// Block-window kernels (pf_window.cuh) for the levels that have windows (DevWin).
bool win_on(const pf_hierarchy* h, const DevLevel& D) { return D.W.on && h->opt.win_kernels != 0; }
WinView win_view(const DevLevel& D) { return WinView{D.W.cols16.p, D.W.chunk_ptr.p, D.W.chunks.p, D.W.dpos.p}; }
template <typename K>
size_t win_smem(K kern, const DevLevel& D) {  // the launch's dynamic shared memory, cap raised once
  const size_t smem = D.W.smem();
  static thread_local std::map<const void*, size_t> attr_set;
  auto& have = attr_set[reinterpret_cast<const void*>(kern)];
  if (smem > 48 * 1024 && have < smem) {
    PF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    have = smem;
  }
  return smem;
}

void enq_resnorm(pf_hierarchy* h, int l, const double* x, const double* b) {
  Level& L = h->levels[l];
  auto launch = launcher(h);
  const bool single = h->world == 1;
  for (int s = 0; s < h->n_sub; ++s) {
    DevLevel& D = L.sub[s];
    vk_dispatch_rows(D.A, [&](auto V) {
    constexpr int vk = decltype(V)::value;
    if (win_on(h, D)) {
      auto kern = k_resnorm_win<vk>;
      launch.with_smem(win_smem(kern, D))(static_cast<unsigned>(D.resnorm_blocks), kBlock, kern, view(D.A),
                                          win_view(D), x + D.offset, b + D.offset, D.n_own, D.n, D.partials.p,
                                          D.ticket.p, L.sumsq.p + s, single ? L.norm.p : nullptr);
      return;
    }
    launch(static_cast<unsigned>(D.resnorm_blocks), kBlock, k_resnorm<decltype(V)::value>, view(D.A), x + D.offset,
           b + D.offset, D.n_own, D.partials.p, D.ticket.p, L.sumsq.p + s, single ? L.norm.p : nullptr);
    });
  }
  if (!single) enq_allreduce(h, L, true);
}

// Long rows (longer than Options::split_row_len) on levels of at most
// Options::split_rows_max rows take the slice-split Jacobi / residual (k_rows_split).
bool rows_split_ok(const pf_hierarchy* h, const DevLevel& D) {
  return h->opt.split_row_len > 0 && D.A.max_len > h->opt.split_row_len && D.n <= h->opt.split_rows_max;
}
template <bool kJacobi>
void enq_rows_split(pf_hierarchy* h, DevLevel& D, const double* x, double* out, const double* b, double omega) {
  const int32_t width = (D.A.max_len + 3) / 4 * 4;
  const size_t smem = sizeof(double) * kSlice * static_cast<size_t>(width);
  auto launch = launcher(h);
  vk_dispatch_rows(D.A, [&](auto V) {
    constexpr int vk = decltype(V)::value;
    auto kern = k_rows_split<kJacobi, vk>;
    static thread_local std::map<const void*, size_t> attr_set;
    auto& have = attr_set[reinterpret_cast<const void*>(kern)];
    if (smem > 48 * 1024 && have < smem) {
      PF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      have = smem;
    }
    const unsigned grid = static_cast<unsigned>((static_cast<int64_t>(D.n) + kSlice - 1) / kSlice);
    launch.with_smem(smem)(grid, kSplitBlock, kern, view(D.A), x, out, b, D.n_own, D.n, omega);
  });
}

void enq_residual(pf_hierarchy* h, int l, const double* x, const double* b, double* r) {
  Level& L = h->levels[l];
  auto launch = launcher(h);
  bool split = true;
  for (DevLevel& D : L.sub) split = split && rows_split_ok(h, D);
  if (split) {
    for (DevLevel& D : L.sub) enq_rows_split<false>(h, D, x + D.offset, r + D.offset, b + D.offset, 0.0);
    return;
  }
  for (DevLevel& D : L.sub)
    vk_dispatch_rows(D.A, [&](auto V) {
      constexpr int vk = decltype(V)::value;
      if (win_on(h, D)) {
        auto kern = k_residual_win<vk>;
        launch.with_smem(win_smem(kern, D))(grid_for(D.n), kBlock, kern, view(D.A), win_view(D), x + D.offset,
                                            b + D.offset, r + D.offset, D.n, D.n_own);
        return;
      }
      launch(D.rmap_grid, kBlock, k_residual<decltype(V)::value>, view(D.A), x + D.offset, b + D.offset, r + D.offset, D.n,
             D.n_own, D.rmap);
    });
}

void enq_spmv(pf_hierarchy* h, int l, const double* x, double* y) {
  Level& L = h->levels[l];
  auto launch = launcher(h);
  for (DevLevel& D : L.sub)
    vk_dispatch(D.A.vals.vkind, [&](auto V) {
      launch(grid_for(D.n), kBlock, k_spmv<decltype(V)::value>, view(D.A), x + D.offset, y + D.offset, D.n);
    });
}

void enq_copy(pf_hierarchy* h, const double* src, double* dst, int64_t n) {
  launcher(h)(grid_for(n), kBlock, k_copy, src, dst, n);
}

// Launches of at most Options::wide_max_rows rows (default: one wave of the wide kernels, 2
// blocks of 256 per SM) on operators with 8-bit value indices and rows of <= 28 entries
// take the wide-row kernels (k_color_sweep_wide / k_jacobi_wide: the whole row's operator
// loaded before griddepcontrol.wait, all its x gathers in flight at once after it); 0: never.
constexpr int kWideGroups = 7;
int64_t wide_max_rows(const pf_hierarchy* h) {
  return h->opt.wide_max_rows >= 0 ? h->opt.wide_max_rows : int64_t(PF_WIDE_MINB) * sm_count(h->device) * kBlock;
}
template <int vk>
bool wide_ok(const pf_hierarchy* h, const DevLevel& D, int64_t rows) {
  constexpr int K = vk_kind<vk>();
  return (K == 1 || K == kVKSmem) && D.A.max_len > 0 && D.A.max_len <= 4 * kWideGroups && rows > 0 &&
         rows <= wide_max_rows(h);
}

// One damped-Jacobi sweep of subdomain level D, src -> dst.
void enq_jacobi_sweep(pf_hierarchy* h, DevLevel& D, const double* src, double* dst, const double* b, double omega) {
  if (rows_split_ok(h, D)) {
    enq_rows_split<true>(h, D, src, dst, b, omega);
    return;
  }
  auto launch = launcher(h);
  vk_dispatch_rows(D.A, [&](auto V) {
    constexpr int vk = decltype(V)::value;
    if (win_on(h, D)) {
      auto kern = k_jacobi_win<vk>;
      launch.with_smem(win_smem(kern, D))(grid_for(D.n), kBlock, kern, view(D.A), win_view(D), src, dst, b, D.n_own,
                                          D.n, omega);
      return;
    }
    if constexpr (vk_kind<vk>() == 1 || vk_kind<vk>() == kVKSmem) {
      if (D.rmap.n_col == 0 && wide_ok<vk>(h, D, D.n)) {
        launch(grid_for(D.n), kBlock, k_jacobi_wide<vk, kWideGroups>, view(D.A), src, dst, b, D.n_own, D.n, omega);
        return;
      }
    }
    launch(D.rmap_grid, kBlock, k_jacobi<vk>, view(D.A), src, dst, b, D.n_own, D.n, omega, D.rmap);
  });
}

// Options::sor_tma (default 0, measured slower): colour sweeps of operators with rows of <= 28
// entries (Q1, rotated Q1) take the TMA-staged persistent kernel (pf_sweep_tma.cuh) on
// levels with at least sor_tma_min_rows own rows, sor_tma_bps blocks per SM, warp layout
// sor_tma_cfg (0 = 8 warps x 2 stages, 1 = 4 x 4, 2 = 8 x 3).

// One colour of a coloured sweep.  Levels with long rows (Q2: up to 125 entries; longer
// than Options::split_row_len, default 48) take the slice-split kernel: a colour has few
// rows there (1/27 of the level), so one thread per row leaves most SMs idle while each
// thread walks its 32 groups — on levels up to Options::split_max_rows own rows (default
// 1M): on larger ones the colours are big enough for the row kernel (Q2 at 64^3: 482 vs
// 431 us per sweep).
void enq_color_sweep(pf_hierarchy* h, DevLevel& D, int c, bool sor, double omega, double* x, const double* b) {
  const int32_t r0 = D.color_start[c], r1 = D.color_start[c + 1];
  if (r1 <= r0) return;
  auto launch = launcher(h);
  const int64_t split = h->opt.split_row_len;
  vk_dispatch_rows(D.A, [&](auto V) {
    constexpr int vk = decltype(V)::value;
    if (h->opt.sor_tma && D.A.max_len <= 4 * kTmaMaxGroups && D.A.max_len > 0 && D.n_own >= h->opt.sor_tma_min_rows) {
      const int32_t width = (D.A.max_len + 3) / 4 * 4;
      const TmaStageLayout lay = tma_layout(width, tma_vbytes<vk>());
      auto go = [&](auto W, auto S) {
        constexpr int kw = decltype(W)::value, ks = decltype(S)::value;
        const size_t smem = static_cast<size_t>(kw) * ks * lay.bytes;
        auto kern = sor ? k_color_sweep_tma<true, vk, kw, ks> : k_color_sweep_tma<false, vk, kw, ks>;
        static thread_local std::map<const void*, size_t> attr_set;
        auto& have = attr_set[reinterpret_cast<const void*>(kern)];
        if (smem > 48 * 1024 && have < smem) {
          PF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
          have = smem;
        }
        const int64_t n_slices = ((r1 - 1) >> 5) - (r0 >> 5) + 1;
        const int64_t grid = std::min<int64_t>((n_slices + kw - 1) / kw,
                                               std::max<int64_t>(1, h->opt.sor_tma_bps) * sm_count(h->device));
        launch.with_smem(smem)(static_cast<unsigned>(grid), 32 * kw, kern, view(D.A), x, b, r0, r1, omega, width);
      };
      switch (h->opt.sor_tma_cfg) {
        case 1: go(std::integral_constant<int, 4>{}, std::integral_constant<int, 4>{}); break;
        case 2: go(std::integral_constant<int, 8>{}, std::integral_constant<int, 3>{}); break;
        default: go(std::integral_constant<int, 8>{}, std::integral_constant<int, 2>{}); break;
      }
      return;
    }
    if (win_on(h, D) && h->opt.win_kernels >= 2) {
      const int32_t b0 = r0 / kBlock, b1 = (r1 - 1) / kBlock + 1;
      if (sor) {
        auto kern = k_color_sweep_win<true, vk>;
        launch.with_smem(win_smem(kern, D))(static_cast<unsigned>(b1 - b0), kBlock, kern, view(D.A), win_view(D), x, b,
                                            b0, r0, r1, D.n, omega);
      } else {
        auto kern = k_color_sweep_win<false, vk>;
        launch.with_smem(win_smem(kern, D))(static_cast<unsigned>(b1 - b0), kBlock, kern, view(D.A), win_view(D), x, b,
                                            b0, r0, r1, D.n, 1.0);
      }
      return;
    }
    if constexpr (vk_kind<vk>() == 1 || vk_kind<vk>() == kVKSmem) {
      if (wide_ok<vk>(h, D, r1 - r0)) {
        if (sor)
          launch(grid_for(r1 - r0), kBlock, k_color_sweep_wide<true, vk, kWideGroups>, view(D.A), x, b, r0, r1, omega);
        else
          launch(grid_for(r1 - r0), kBlock, k_color_sweep_wide<false, vk, kWideGroups>, view(D.A), x, b, r0, r1, 1.0);
        return;
      }
    }
    if (split > 0 && D.A.max_len > split && D.n_own <= h->opt.split_max_rows) {
      const int32_t width = (D.A.max_len + 3) / 4 * 4;
      const size_t smem = sizeof(double) * kSlice * static_cast<size_t>(width);
      auto kern = sor ? k_color_sweep_split<true, vk> : k_color_sweep_split<false, vk>;
      static thread_local const void* attr_set[2][16] = {};
      if (smem > 48 * 1024 && attr_set[sor][vk + 1] != reinterpret_cast<const void*>(smem)) {
        PF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        attr_set[sor][vk + 1] = reinterpret_cast<const void*>(smem);
      }
      const unsigned grid = static_cast<unsigned>(((r1 - 1) >> 5) - (r0 >> 5) + 1);
      launch.with_smem(smem)(grid, kSplitBlock, kern, view(D.A), x, b, r0, r1, omega, width);
    } else if (sor) {
      launch(grid_for(r1 - r0), kBlock, k_color_sweep<true, vk>, view(D.A), x, b, r0, r1, omega);
    } else {
      launch(grid_for(r1 - r0), kBlock, k_color_sweep<false, vk>, view(D.A), x, b, r0, r1, 1.0);
    }
  });
}

// smooth (solvers.cpp:56-68) on x (primary buffer) with b.
// first_done: the first Jacobi sweep already ran (k_jacobi_norm in the solve graph).
// Returns true when the halo2 scatter that follows a smoothing phase in the cycle was
// already done (fused into the last sweep's exchange).
bool enq_smooth(pf_hierarchy* h, int l, pf_vector* xv, const double* b, const pf_smoother_config& sc,
                bool first_done = false, bool then_h2 = false) {
  Level& L = h->levels[l];
  auto launch = launcher(h);
  double* bufs[2] = {xv->cur(), xv->alt()};
  int cur = 0;
  bool exchanged = false;
  for (int sweep = 0; sweep < sc.sweeps; ++sweep) {
    for (int local = 0; local < sc.local_sweeps; ++local) {
      const bool overlap = h->fused && h->world > h->n_sub && h->xport && h->xport->overlap_ok() &&
                           sc.kind == PF_SMOOTHER_JACOBI &&
                           local + 1 == sc.local_sweeps && !(first_done && sweep == 0 && local == 0);
      if (overlap) {
        // boundary rows (+ the non-own carry-over) first, then the exchange on the side
        // stream overlapped with the interior rows
        const DevLevel& D = L.sub[0];
        const bool last = sweep + 1 == sc.sweeps;
        vk_dispatch_rows(D.A, [&](auto V) {
          constexpr int vk = decltype(V)::value;
          launch(std::max<unsigned>(grid_for(D.n_brows), 1u) + grid_for(D.n - D.n_own), kBlock, k_jacobi_boundary<vk>,
                 view(D.A), static_cast<const int32_t*>(D.brows.p), D.n_brows,
                 static_cast<const double*>(bufs[cur] + D.offset), bufs[cur ^ 1] + D.offset, b + D.offset,
                 D.n_own, D.n, sc.damping);
        });
        PF_CUDA(cudaEventRecord(h->ev_fork, h->stream));
        PF_CUDA(cudaStreamWaitEvent(h->comm_stream, h->ev_fork, 0));
        enq_plan(h, last && then_h2 ? L.fused_all : L.fused_ms_h1, bufs[cur ^ 1], h->comm_stream);
        vk_dispatch_rows(D.A, [&](auto V) {
          constexpr int vk = decltype(V)::value;
          launch(grid_for(D.n_own), kBlock, k_jacobi_interior<vk>, view(D.A),
                 static_cast<const uint8_t*>(D.is_brow.p), static_cast<const double*>(bufs[cur] + D.offset),
                 bufs[cur ^ 1] + D.offset, b + D.offset, D.n_own, sc.damping);
        });
        PF_CUDA(cudaEventRecord(h->ev_join, h->comm_stream));
        PF_CUDA(cudaStreamWaitEvent(h->stream, h->ev_join, 0));
        cur ^= 1;
        exchanged = true;
        continue;
      }
      const bool overlap_c = h->fused && h->world > h->n_sub && h->xport && h->xport->overlap_ok() &&
                             sc.kind != PF_SMOOTHER_JACOBI && !h->colorwise && local + 1 == sc.local_sweeps &&
                             L.sub[0].n_cpre >= 0 && L.sub[0].n_colors >= 1;
      if (overlap_c) {
        // coloured sweep: every colour but the last as usual; the last colour's rows that
        // send or read a non-own copy first, then the exchange on the side stream overlapped
        // with the rest of the last colour (they touch neither the sent rows nor the copies
        // the exchange rewrites, so the result is the reference order's bit for bit)
        DevLevel& D = L.sub[0];
        const bool sor = sc.kind == PF_SMOOTHER_MULTICOLOR_SOR;
        const double om = sor ? sc.damping : 1.0;
        double* x = bufs[cur] + D.offset;
        const double* bb = b + D.offset;
        for (int c = 0; c + 1 < D.n_colors; ++c) enq_color_sweep(h, D, c, sor, om, x, bb);
        const int32_t c0 = D.color_start[D.n_colors - 1], c1 = D.color_start[D.n_colors];
        vk_dispatch_rows(D.A, [&](auto V) {
          constexpr int vk = decltype(V)::value;
          if (D.n_cpre > 0) {
            if (sor)
              launch(grid_for(D.n_cpre), kBlock, k_color_sweep_list<true, vk>, view(D.A), x, bb,
                     static_cast<const int32_t*>(D.cpre.p), D.n_cpre, om);
            else
              launch(grid_for(D.n_cpre), kBlock, k_color_sweep_list<false, vk>, view(D.A), x, bb,
                     static_cast<const int32_t*>(D.cpre.p), D.n_cpre, om);
          }
        });
        const bool last = sweep + 1 == sc.sweeps;
        PF_CUDA(cudaEventRecord(h->ev_fork, h->stream));
        PF_CUDA(cudaStreamWaitEvent(h->comm_stream, h->ev_fork, 0));
        enq_plan(h, last && then_h2 ? L.fused_all : L.fused_ms_h1, bufs[cur], h->comm_stream);
        vk_dispatch_rows(D.A, [&](auto V) {
          constexpr int vk = decltype(V)::value;
          if (c1 > c0) {
            if (sor)
              launch(grid_for(c1 - c0), kBlock, k_color_sweep_skip<true, vk>, view(D.A), x, bb, c0, c1,
                     static_cast<const uint8_t*>(D.is_cpre.p), om);
            else
              launch(grid_for(c1 - c0), kBlock, k_color_sweep_skip<false, vk>, view(D.A), x, bb, c0, c1,
                     static_cast<const uint8_t*>(D.is_cpre.p), om);
          }
        });
        PF_CUDA(cudaEventRecord(h->ev_join, h->comm_stream));
        PF_CUDA(cudaStreamWaitEvent(h->stream, h->ev_join, 0));
        exchanged = true;
        continue;
      }
      if (sc.kind == PF_SMOOTHER_JACOBI) {
        if (!(first_done && sweep == 0 && local == 0))
          for (DevLevel& D : L.sub)
            enq_jacobi_sweep(h, D, bufs[cur] + D.offset, bufs[cur ^ 1] + D.offset, b + D.offset, sc.damping);
        cur ^= 1;
      } else {
        const bool sor = sc.kind == PF_SMOOTHER_MULTICOLOR_SOR;
        int max_colors = 0;
        for (DevLevel& D : L.sub) max_colors = std::max(max_colors, D.n_colors);
        for (int c = 0; c < max_colors; ++c) {
          for (DevLevel& D : L.sub) {
            if (c >= D.n_colors) continue;
            enq_color_sweep(h, D, c, sor, sor ? sc.damping : 1.0, bufs[cur] + D.offset, b + D.offset);
          }
          // colour-wise exchange: every copy is refreshed before the next colour, so a
          // partitioned sweep relaxes like the single-domain coloured sweep (the sweep's
          // own exchange below follows the last colour of the last local sweep)
          if (h->colorwise && !(local + 1 == sc.local_sweeps && c + 1 == max_colors)) {
            if (h->fused) {
              enq_plan(h, L.fused_ms_h1, bufs[cur]);
            } else {
              enq_update_ms(h, l, bufs[cur], PF_UPDATE_SCATTER);
              enq_scatter(h, l, PF_CH_HALO1, bufs[cur]);
            }
          }
        }
      }
    }
    if (exchanged) {
      exchanged = false;  // done by the overlapped sweep
    } else if (h->fused) {
      const bool last = sweep + 1 == sc.sweeps;
      enq_plan(h, last && then_h2 ? L.fused_all : L.fused_ms_h1, bufs[cur]);
    } else {
      enq_update_ms(h, l, bufs[cur], PF_UPDATE_SCATTER);
      enq_scatter(h, l, PF_CH_HALO1, bufs[cur]);
    }
  }
  if (cur) enq_copy(h, bufs[1], bufs[0], L.total);
  return h->fused && then_h2 && sc.sweeps > 0;
}

void enq_prolong(pf_hierarchy* h, int fine, const double* xc, double* xf, int add) {
  Level& F = h->levels[fine];
  Level& Cl = h->levels[fine - 1];
  auto launch = launcher(h);
  for (int s = 0; s < h->n_sub; ++s) {
    DevLevel& D = F.sub[s];
    vk_dispatch_rows(D.P, [&](auto V) {
      constexpr int vk = decltype(V)::value;
      // trilinear P (<= 8 entries per row, 8-bit weights): k_prolong_add8 (prolongation
      // 31.7 -> 29.7 us at C2's finest level)
      if constexpr (vk_kind<vk>() == 1 || vk_kind<vk>() == kVKSmem) {
        if (D.P.max_len <= 8) {
          launch(grid_for(D.n), kBlock, k_prolong_add8<vk>, view(D.P), xc + Cl.sub[s].offset, xf + D.offset, D.n, add);
          return;
        }
      }
      launch(grid_for(D.n), kBlock, k_prolong_add<vk>, view(D.P), xc + Cl.sub[s].offset, xf + D.offset, D.n, add);
    });
  }
}

// Options::fused_rr_rows (default 8192; 0 = off): levels up to that many rows form the cycle
// residual and its restriction in one launch (k_residual_restrict).  Measured at C2:
// levels 1-3 fused, Jacobi solve 5.86 -> 5.78 ms; level 4 (36k rows) too, 5.82 ms (its
// redundant fine-residual work outweighs the saved launch).
bool fused_rr_for(pf_hierarchy* h, int fine) {
  const int64_t limit = h->opt.fused_rr_rows;
  for (const DevLevel& D : h->levels[fine].sub)
    if (D.n > limit || D.R.max_len > 32) return false;
  return true;
}

void enq_residual_restrict(pf_hierarchy* h, int fine, const double* x, const double* b, double* bc, double* xc) {
  Level& F = h->levels[fine];
  Level& Cl = h->levels[fine - 1];
  auto launch = launcher(h);
  for (int s = 0; s < h->n_sub; ++s) {
    DevLevel& D = F.sub[s];
    DevLevel& DC = Cl.sub[s];
    vk_dispatch_rows(D.A, [&](auto V) {
      launch(grid_for(static_cast<int64_t>(DC.n) * 32), kBlock, k_residual_restrict<decltype(V)::value>, view(D.A),
             view(D.R), x + D.offset, b + D.offset, bc + DC.offset, xc ? xc + DC.offset : nullptr,
             static_cast<const uint8_t*>(DC.d_is_dir.p), DC.n, 1);
    });
  }
}

// rc = R rf over owns_row rows; optional zeroing of Dirichlet b and of the coarse x.
void enq_restrict(pf_hierarchy* h, int fine, const double* rf, double* bc, double* xc, int zero_dir) {
  Level& F = h->levels[fine];
  Level& Cl = h->levels[fine - 1];
  auto launch = launcher(h);
  for (int s = 0; s < h->n_sub; ++s) {
    DevLevel& D = F.sub[s];
    DevLevel& DC = Cl.sub[s];
    vk_dispatch_rows(D.R, [&](auto V) {
      constexpr int vk = decltype(V)::value;
      launch(grid_for(DC.n), kBlock, k_restrict<vk>, view(D.R), rf + D.offset, bc + DC.offset,
             xc ? xc + DC.offset : nullptr, static_cast<const uint8_t*>(DC.d_is_dir.p), DC.n, zero_dir);
    });
  }
}

// Inverse by Gauss-Jordan elimination with partial pivoting (the first row of maximal
// |pivot|), pivot rows scaled by division; oracle/gmg_oracle.c restates it.
void gauss_jordan_inverse(int n, std::vector<double> M, std::vector<double>& inv) {
  inv.assign(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i) inv[static_cast<size_t>(i) * n + i] = 1.0;
  auto at = [n](std::vector<double>& v, int i, int j) -> double& { return v[static_cast<size_t>(i) * n + j]; };
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = std::fabs(at(M, k, k));
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(at(M, i, k)) > best) {
        best = std::fabs(at(M, i, k));
        p = i;
      }
    if (best == 0.0) throw Error(PF_ERR_SINGULAR_DIAGONAL, "singular coarse matrix");
    if (p != k)
      for (int j = 0; j < n; ++j) {
        std::swap(at(M, p, j), at(M, k, j));
        std::swap(at(inv, p, j), at(inv, k, j));
      }
    const double piv = at(M, k, k);
    for (int j = 0; j < n; ++j) {
      at(M, k, j) = at(M, k, j) / piv;
      at(inv, k, j) = at(inv, k, j) / piv;
    }
    for (int i = 0; i < n; ++i) {
      if (i == k) continue;
      const double f = at(M, i, k);
      if (f == 0.0) continue;
      for (int j = 0; j < n; ++j) {
        at(M, i, j) = at(M, i, j) - f * at(M, k, j);
        at(inv, i, j) = at(inv, i, j) - f * at(inv, k, j);
      }
    }
  }
}

void drop_graphs(pf_hierarchy* h) {
  PF_CUDA(cudaStreamSynchronize(h->stream));
  for (auto& [k, e] : h->graphs) {
    if (e.exec) cudaGraphExecDestroy(e.exec);
    if (e.state) cudaFree(e.state);
    if (e.host_state) cudaFreeHost(e.host_state);
  }
  h->graphs.clear();
}

void enq_coarse_smem(pf_hierarchy* h, const CoarsePack& P, double* x, const double* b, double tol,
                     int max_iter, double* stats) {
  const size_t bytes = coarse_pack_smem(P);
  if (bytes > 48 * 1024)
    PF_CUDA(cudaFuncSetAttribute(k_coarse_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(bytes)));
  k_coarse_smem<<<1, kBlock, bytes, h->stream>>>(P, x, b, tol, max_iter, stats);
  PF_CUDA(cudaGetLastError());
  ++*(g_capture_counter ? g_capture_counter : &h->launches);
}

// coarse_solve on level l.  cycle_mode: x enters as zero and update_halo2 follows
// (multigrid.cpp:153-158); returns true when that halo update was already done.
bool enq_coarse(pf_hierarchy* h, int l, double* x, const double* b, double tol, int max_iter,
                bool cycle_mode) {
  Level& L = h->levels[l];
  auto launch = launcher(h);
  if (h->world == h->n_sub && l == 0 && coarse_pack_smem(L.cpack) <= kCoarseSmemMax) {
    enq_coarse_smem(h, L.cpack, x, b, tol, max_iter, L.coarse_stats.p);
    return false;
  }
  if (h->world == h->n_sub) {
    const ExchangePlan& ms = L.scatter[PF_CH_MASTER_SLAVE];
    const ExchangePlan& h1 = L.scatter[PF_CH_HALO1];
    launch(1, 32, k_coarse_gs, static_cast<const CoarseSub*>(L.coarse_subs.p), h->n_sub, x, b,
           static_cast<const int32_t*>(ms.dst.p), static_cast<const int32_t*>(ms.src.p),
           static_cast<int32_t>(ms.n), static_cast<const int32_t*>(h1.dst.p),
           static_cast<const int32_t*>(h1.src.p), static_cast<int32_t>(h1.n), tol, max_iter,
           L.coarse_stats.p);
    return false;
  }
  if (l != 0) state("multi-process coarse solve runs on level 0 only");
  auto& R = h->rep;
  auto& R0 = R.lv[0];
  const DevLevel& D = L.sub[0];
  if (!h->xport) state("multi-process hierarchy used before pf_hierarchy_init_nccl");
  // every rank's coarse rhs (and start vector) on every GPU: one allgather each
  enq_copy(h, b, R.send.p, D.n);
  h->xport->allgather(R.send.p, R0.b.p, R0.stride, h->stream);
  if (cycle_mode) {
    PF_CUDA(cudaMemsetAsync(R0.x.p, 0, sizeof(double) * R0.stride * h->world, h->stream));
  } else {
    enq_copy(h, x, R.send.p, D.n);
    h->xport->allgather(R.send.p, R0.x.p, R0.stride, h->stream);
  }
  const ExchangePlan& ms = R0.scatter[PF_CH_MASTER_SLAVE];
  const ExchangePlan& h1 = R0.scatter[PF_CH_HALO1];
  const ExchangePlan& h2 = R0.scatter[PF_CH_HALO2];
  if (coarse_pack_smem(R.cpack) <= kCoarseSmemMax)
    enq_coarse_smem(h, R.cpack, R0.x.p, R0.b.p, tol, max_iter, L.coarse_stats.p);
  else
    launch(1, 32, k_coarse_gs, static_cast<const CoarseSub*>(R.subs.p), h->world, R0.x.p,
           static_cast<const double*>(R0.b.p), static_cast<const int32_t*>(ms.dst.p),
           static_cast<const int32_t*>(ms.src.p), static_cast<int32_t>(ms.n),
           static_cast<const int32_t*>(h1.dst.p), static_cast<const int32_t*>(h1.src.p),
           static_cast<int32_t>(h1.n), tol, max_iter, L.coarse_stats.p);
  if (cycle_mode && h2.n > 0)
    launch(grid_for(h2.n), kBlock, k_copy_idx, static_cast<const int32_t*>(h2.src.p),
           static_cast<const int32_t*>(h2.dst.p), R0.x.p, static_cast<int32_t>(h2.n));
  enq_copy(h, R0.x.p + h->rank_base * R0.stride, x, D.n);
  return cycle_mode;
}

// cycle(bot.top) in one cooperative launch; lev[top].b holds the restricted residual
// (before the master/slave accumulate when accumulate_top) and lev[top].x is zero.
// (Options::bottom_block_kernel, default 1: a bottom whose levels are all staged runs as the
// one-block k_bottom_block instead of the cooperative k_bottom.)

void enq_bottom(pf_hierarchy* h, const pf_hierarchy::Bottom& bot, const pf_multigrid_config& cfg,
                int accumulate_top) {
  static const int calib0 = std::getenv("PF_BOTTOM_CALIB") ? std::atoi(std::getenv("PF_BOTTOM_CALIB")) : 0;
  if (bot.staged_all && h->opt.bottom_block_kernel && calib0 == 0) {
    const BotCfg c{cfg.smoother.kind, cfg.pre_smooth, cfg.post_smooth, cfg.smoother.local_sweeps,
                   cfg.coarse_max_iter, cfg.smoother.damping, cfg.coarse_tol, 1 << 20, 0,
                   h->colorwise && cfg.smoother.kind != PF_SMOOTHER_JACOBI ? 1 : 0};
    auto launch = launcher(h);
    const BotDesc* d = static_cast<const BotDesc*>(bot.desc);
    switch (cfg.smoother.kind) {
      case PF_SMOOTHER_JACOBI: launch.with_smem(bot.smem)(1, kBotBlockThreads, k_bottom_block<0>, d, c, accumulate_top); break;
      case PF_SMOOTHER_MULTICOLOR_SOR: launch.with_smem(bot.smem)(1, kBotBlockThreads, k_bottom_block<2>, d, c, accumulate_top); break;
      default: launch.with_smem(bot.smem)(1, kBotBlockThreads, k_bottom_block<1>, d, c, accumulate_top); break;
    }
    return;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(static_cast<unsigned>(bot.grid));
  lc.blockDim = dim3(kBlock);
  lc.dynamicSmemBytes = bot.smem;
  lc.stream = h->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  // measured at C2: the coloured smoothers (8 barriers per sweep) gain from running the
  // tiny levels inside one block (V-cycle 1.83 -> 1.75 ms); Jacobi (1 barrier per sweep)
  // loses parallelism there and keeps the whole grid
  // (with every bottom level staged in shared memory, both smoothers run them in block 0)
  const int block_top = cfg.smoother.kind == PF_SMOOTHER_JACOBI && !bot.staged_all ? -1 : 1 << 20;
  static const int calib = std::getenv("PF_BOTTOM_CALIB") ? std::atoi(std::getenv("PF_BOTTOM_CALIB")) : 0;
  const BotCfg c{cfg.smoother.kind, cfg.pre_smooth, cfg.post_smooth, cfg.smoother.local_sweeps,
                 cfg.coarse_max_iter, cfg.smoother.damping, cfg.coarse_tol, block_top, calib,
                 h->colorwise && cfg.smoother.kind != PF_SMOOTHER_JACOBI ? 1 : 0};
  PF_CUDA(cudaLaunchKernelEx(&lc, k_bottom, static_cast<const BotDesc*>(bot.desc), c, accumulate_top));
  ++*(g_capture_counter ? g_capture_counter : &h->launches);
}

// cycle (multigrid.cpp:150-190)
void enq_cycle(pf_hierarchy* h, int l, pf_vector* xv, const double* b, const pf_multigrid_config& cfg,
               bool first_done = false) {
  Level& L = h->levels[l];
  double* x = xv->cur();
  if (l == 0) {
    if (!enq_coarse(h, 0, x, b, cfg.coarse_tol, cfg.coarse_max_iter, true))
      enq_scatter(h, 0, PF_CH_HALO2, x);
    return;
  }
  pf_smoother_config pre = cfg.smoother;
  pre.sweeps = cfg.pre_smooth;
  if (!enq_smooth(h, l, xv, b, pre, first_done && cfg.pre_smooth > 0, true)) enq_scatter(h, l, PF_CH_HALO2, x);
  Level& Cl = h->levels[l - 1];
  if (fused_rr_for(h, l)) {
    enq_residual_restrict(h, l, x, b, Cl.b->cur(), Cl.x->cur());
  } else {
    enq_residual(h, l, x, b, L.r.p);
    enq_restrict(h, l, L.r.p, Cl.b->cur(), Cl.x->cur(), 1);
  }
  if (h->bot.active && l - 1 == h->bot.top && bottom_for(h, cfg)) {
    enq_bottom(h, h->bot, cfg, 1);  // accumulate, cycle(top) ... down to the coarse solve and back
  } else if (h->rep.bot.active && l - 1 == h->rep.bot.top) {
    // multi-process: the restricted partial sums of every rank in one allgather, then the
    // bottom V-cycle of ALL ranks replayed on this GPU (accumulate included), then this
    // rank's part of the result (halo2 already consistent) back into the local level
    auto& RL = h->rep.lv[static_cast<size_t>(l - 1)];
    const DevLevel& D = Cl.sub[0];
    if (!h->xport) state("multi-process hierarchy used before pf_hierarchy_init_nccl");
    enq_copy(h, Cl.b->cur(), h->rep.send.p, D.n);
    h->xport->allgather(h->rep.send.p, RL.b.p, RL.stride, h->stream);
    PF_CUDA(cudaMemsetAsync(RL.x.p, 0, sizeof(double) * RL.stride * h->world, h->stream));
    enq_bottom(h, h->rep.bot, cfg, 1);
    enq_copy(h, RL.x.p + h->rank_base * RL.stride, Cl.x->cur(), D.n);
  } else {
    enq_update_ms(h, l - 1, Cl.b->cur(), PF_UPDATE_ACCUMULATE_THEN_SCATTER);
    enq_cycle(h, l - 1, Cl.x, Cl.b->cur(), cfg);
  }
  enq_prolong(h, l, Cl.x->cur(), x, 1);
  pf_smoother_config post = cfg.smoother;
  post.sweeps = cfg.post_smooth;
  if (!enq_smooth(h, l, xv, b, post, false, true)) enq_scatter(h, l, PF_CH_HALO2, x);
}

// v_cycle (multigrid.cpp:194-208)
void enq_vcycle(pf_hierarchy* h, pf_vector* x, const double* b, const pf_multigrid_config& cfg) {
  const int top = h->n_levels - 1;
  enq_scatter(h, top, PF_CH_HALO2, x->cur());
  enq_cycle(h, top, x, b, cfg);
}

// The norm-producing head of one outer iteration of the device-driven solve: for damped
// Jacobi the first pre-smoothing sweep of the next cycle (k_jacobi_norm), otherwise a
// k_resnorm pass; per-subdomain squares land in L.sumsq for k_decide.
bool fused_head(const pf_multigrid_config& cfg) {
  return cfg.smoother.kind == PF_SMOOTHER_JACOBI && cfg.pre_smooth > 0 && cfg.smoother.local_sweeps >= 1;
}

void enq_norm_head(pf_hierarchy* h, pf_vector* x, const double* b, const pf_multigrid_config& cfg) {
  const int top = h->n_levels - 1;
  Level& L = h->levels[top];
  auto launch = launcher(h);
  for (int s = 0; s < h->n_sub; ++s) {
    DevLevel& D = L.sub[s];
    vk_dispatch_rows(D.A, [&](auto V) {
      constexpr int vk = decltype(V)::value;
      if (win_on(h, D)) {
        if (fused_head(cfg)) {
          auto kern = k_jacobi_norm_win<vk>;
          launch.with_smem(win_smem(kern, D))(grid_for(D.n), kBlock, kern, view(D.A), win_view(D),
                                              static_cast<const double*>(x->cur() + D.offset), x->alt() + D.offset,
                                              b + D.offset, D.n_own, D.n, cfg.smoother.damping, D.partials.p,
                                              D.ticket.p, L.sumsq.p + s);
        } else {
          auto kern = k_resnorm_win<vk>;
          launch.with_smem(win_smem(kern, D))(static_cast<unsigned>(D.resnorm_blocks), kBlock, kern, view(D.A),
                                              win_view(D), static_cast<const double*>(x->cur() + D.offset),
                                              b + D.offset, D.n_own, D.n, D.partials.p, D.ticket.p, L.sumsq.p + s,
                                              static_cast<double*>(nullptr));
        }
        return;
      }
      if (fused_head(cfg))
        launch(grid_for(D.n), kBlock, k_jacobi_norm<vk>, view(D.A), static_cast<const double*>(x->cur() + D.offset),
               x->alt() + D.offset, b + D.offset, D.n_own, D.n, cfg.smoother.damping, D.partials.p,
               D.ticket.p, L.sumsq.p + s);
      else
        launch(static_cast<unsigned>(D.resnorm_blocks), kBlock, k_resnorm<vk>, view(D.A),
               static_cast<const double*>(x->cur() + D.offset), b + D.offset, D.n_own, D.partials.p,
               D.ticket.p, L.sumsq.p + s, static_cast<double*>(nullptr));
    });
  }
}

void sync(pf_hierarchy* h);
std::string graph_key(const char* tag, const pf_vector* x, const pf_vector* b, const pf_multigrid_config& c);
void prune_graphs(pf_hierarchy* h);

cudaGraphNode_t single_leaf(cudaGraph_t g) {
  size_t n = 0;
  PF_CUDA(cudaGraphGetNodes(g, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  PF_CUDA(cudaGraphGetNodes(g, nodes.data(), &n));
  cudaGraphNode_t leaf = nullptr;
  for (cudaGraphNode_t v : nodes) {
    size_t nd = 0;
    PF_CUDA(cudaGraphNodeGetDependentNodes(v, nullptr, &nd));
    if (nd == 0) {
      if (leaf) state("solve graph head has several leaves");
      leaf = v;
    }
  }
  return leaf;
}

// solve_outer as ONE graph launch, no host round trip between cycles; the solve state is
// copied to pinned host memory at the end.  Two shapes (Options::solve_graph_if):
//   0 (default)  head; WHILE(continue) { rest of the V-cycle(s); head }
//   1            WHILE(continue) { head; IF(continue) { rest of the V-cycle(s) } }
// with head = halo2(x), the norm head and k_decide.  Both run the same kernels in the same
// order; the first evaluates one conditional node per outer iteration instead of two and
// keeps the programmatic-launch chain from the cycle's last kernel into the next head.
pf_hierarchy::GraphEntry& solve_graph(pf_hierarchy* h, pf_vector* x, const pf_vector* b,
                                      const pf_multigrid_config& cfg) {
  const std::string key = graph_key(h->opt.solve_graph_if ? "solve_if" : "solve", x, b, cfg);
  auto it = h->graphs.find(key);
  if (it != h->graphs.end()) return it->second;
  trace("solve graph: build");
  prune_graphs(h);
  pf_hierarchy::GraphEntry e;
  e.x_uid = x->uid;
  e.b_uid = b->uid;
  const int top = h->n_levels - 1;
  const size_t state_bytes = sizeof(SolveState) + sizeof(double) * static_cast<size_t>(cfg.outer_max_cycles);
  PF_CUDA(cudaMalloc(&e.state, state_bytes));
  PF_CUDA(cudaMallocHost(&e.host_state, state_bytes));
  e.state_bytes = state_bytes;
  cudaGraph_t G = nullptr;
  PF_CUDA(cudaGraphCreate(&G, 0));
  // capture `what` into graph g after nodes `deps`, counting its kernels into *count;
  // returns the capture's leaf nodes
  auto capture = [&](cudaGraph_t g, const std::vector<cudaGraphNode_t>& deps, int64_t* count, auto&& what) {
    std::vector<cudaGraphNode_t> tail;
    PF_CUDA(cudaStreamBeginCaptureToGraph(h->stream, g, deps.empty() ? nullptr : deps.data(), nullptr, deps.size(),
                                          cudaStreamCaptureModeThreadLocal));
    g_capture_counter = count;
    try {
      what();
      cudaStreamCaptureStatus status;
      const cudaGraphNode_t* d = nullptr;
      size_t nd = 0;
      PF_CUDA(cudaStreamGetCaptureInfo(h->stream, &status, nullptr, nullptr, &d, &nd));
      tail.assign(d, d + nd);
    } catch (...) {
      g_capture_counter = nullptr;
      cudaGraph_t dummy = nullptr;
      cudaStreamEndCapture(h->stream, &dummy);
      throw;
    }
    g_capture_counter = nullptr;
    cudaGraph_t same = nullptr;
    PF_CUDA(cudaStreamEndCapture(h->stream, &same));
    return tail;
  };
  try {
    cudaGraphConditionalHandle hw, hi;
    PF_CUDA(cudaGraphConditionalHandleCreate(&hw, G, 1, cudaGraphCondAssignDefault));
    cudaGraphNode_t reset = nullptr;
    cudaMemsetParams mp = {};
    mp.dst = e.state;
    mp.value = 0;
    mp.elementSize = 1;
    mp.width = state_bytes;
    mp.height = 1;
    PF_CUDA(cudaGraphAddMemsetNode(&reset, G, nullptr, 0, &mp));
    int64_t head = 0, rest = 0, head_again = 0;
    auto enq_head = [&](cudaGraphConditionalHandle h_if) {
      enq_scatter(h, top, PF_CH_HALO2, x->cur());
      enq_norm_head(h, x, b->cur(), cfg);
      launcher(h)(1, 32, k_decide, static_cast<const double*>(h->levels[top].sumsq.p), h->n_sub,
                  cfg.outer_tol, cfg.outer_max_cycles, static_cast<SolveState*>(e.state), hw, h_if);
    };
    auto enq_rest = [&] {
      enq_cycle(h, top, x, b->cur(), cfg, fused_head(cfg));
      for (int j = 1; j < cfg.cycles; ++j) enq_vcycle(h, x, b->cur(), cfg);
    };
    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = hw;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wnode = nullptr;
    if (!h->opt.solve_graph_if) {
      std::vector<cudaGraphNode_t> tail = capture(G, {reset}, &head, [&] { enq_head(hw); });
      trace("solve graph: head captured");
      if (tail.empty()) tail.push_back(reset);
      PF_CUDA(cudaGraphAddNode(&wnode, G, tail.data(), tail.size(), &wp));
      cudaGraph_t body = wp.conditional.phGraph_out[0];
      capture(body, {}, &rest, [&] {
        enq_rest();
        g_capture_counter = &head_again;  // the head again, right behind the cycle
        enq_head(hw);
      });
      if (head_again != head) state("solve graph: the two captures of the head differ");
    } else {
      PF_CUDA(cudaGraphAddNode(&wnode, G, &reset, 1, &wp));
      cudaGraph_t body = wp.conditional.phGraph_out[0];
      PF_CUDA(cudaGraphConditionalHandleCreate(&hi, body, 0, cudaGraphCondAssignDefault));
      capture(body, {}, &head, [&] { enq_head(hi); });
      trace("solve graph: head captured");
      cudaGraphNode_t leaf = single_leaf(body);
      cudaGraphNodeParams ip = {};
      ip.type = cudaGraphNodeTypeConditional;
      ip.conditional.handle = hi;
      ip.conditional.type = cudaGraphCondTypeIf;
      ip.conditional.size = 1;
      cudaGraphNode_t inode = nullptr;
      PF_CUDA(cudaGraphAddNode(&inode, body, &leaf, 1, &ip));
      capture(ip.conditional.phGraph_out[0], {}, &rest, enq_rest);
    }
    trace("solve graph: body captured");
    cudaGraphNode_t copy = nullptr;
    PF_CUDA(cudaGraphAddMemcpyNode1D(&copy, G, &wnode, 1, e.host_state, e.state, state_bytes,
                                     cudaMemcpyDeviceToHost));
    PF_CUDA(cudaGraphInstantiate(&e.exec, G, 0));
    trace("solve graph: instantiated");
    e.head_kernels = head;
    e.kernels = rest;
  } catch (...) {
    cudaGraphDestroy(G);
    throw;
  }
  PF_CUDA(cudaGraphDestroy(G));
  return h->graphs.emplace(key, e).first->second;
}

void sync(pf_hierarchy* h) {
  const double limit = h->xport ? h->xport->watchdog_seconds() : 0.0;
  if (limit <= 0.0) {
    PF_CUDA(cudaStreamSynchronize(h->stream));
    if (h->xport) h->xport->check_async();
    return;
  }
  // multi-process: poll, so that a peer that never arrives (or an NCCL error) surfaces as
  // TransportError after the watchdog period instead of a hang (transport.cpp:54-60)
  const auto t0 = std::chrono::steady_clock::now();
  for (int spin = 0;; ++spin) {
    const cudaError_t r = cudaStreamQuery(h->stream);
    if (r == cudaSuccess) break;
    if (r != cudaErrorNotReady) PF_CUDA(r);
    h->xport->check_async();
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) {
      h->xport->abort();
      throw Error(PF_ERR_TRANSPORT, "watchdog: the exchange did not complete within " + std::to_string(limit) +
                                        " s (a peer rank never arrived); communicator aborted");
    }
    if (spin > 1000) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  h->xport->check_async();
}

double read_norm(pf_hierarchy* h, int l) {
  PF_CUDA(cudaMemcpyAsync(h->pinned, h->levels[l].norm.p, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  sync(h);
  return h->pinned[0];
}

void validate_cfg(const pf_multigrid_config& c) {
  if (c.cycles < 1) invalid("cycles must be >= 1");
  if (c.pre_smooth < 0 || c.post_smooth < 0) invalid("smoothing steps must be >= 0");
  if (c.smoother.local_sweeps < 1) invalid("local_sweeps must be >= 1");
  if (c.smoother.kind < 0 || c.smoother.kind > 2) invalid("unknown smoother kind");
  if (c.outer_max_cycles < 1) invalid("outer_max_cycles must be >= 1");
}

// Cache key of a captured graph: the vectors by id and every config field exactly (doubles
// by their bit patterns: 1e-6 and 1e-10, or 2/3 and 0.666667, are different graphs).
std::string graph_key(const char* tag, const pf_vector* x, const pf_vector* b, const pf_multigrid_config& c) {
  auto bits = [](double d) {
    uint64_t u;
    std::memcpy(&u, &d, sizeof u);
    return u;
  };
  std::ostringstream os;
  os << tag << ':' << x->uid << ':' << b->uid << ':' << c.cycles << ':' << c.smoother.kind << ':'
     << c.smoother.local_sweeps << ':' << std::hex << bits(c.smoother.damping) << std::dec << ':' << c.pre_smooth
     << ':' << c.post_smooth << ':' << std::hex << bits(c.coarse_tol) << std::dec << ':' << c.coarse_max_iter << ':'
     << c.outer_max_cycles << ':' << std::hex << bits(c.outer_tol);
  return os.str();
}

// Drop the cached graphs that use a destroyed vector (their captured device pointers are
// dangling); called before a new graph is captured.
void prune_graphs(pf_hierarchy* h) {
  bool synced = false;
  for (auto it = h->graphs.begin(); it != h->graphs.end();) {
    const auto& e = it->second;
    if (h->vectors->alive(e.x_uid) && h->vectors->alive(e.b_uid)) {
      ++it;
      continue;
    }
    if (!synced) {
      PF_CUDA(cudaStreamSynchronize(h->stream));
      synced = true;
    }
    if (e.exec) cudaGraphExecDestroy(e.exec);
    if (e.state) cudaFree(e.state);
    if (e.host_state) cudaFreeHost(e.host_state);
    it = h->graphs.erase(it);
  }
}

// One outer iteration of solve_outer as a graph: cfg.cycles V-cycles, the finest
// residual norm, and its copy into pinned host memory.
pf_hierarchy::GraphEntry& outer_graph(pf_hierarchy* h, pf_vector* x, const pf_vector* b,
                                      const pf_multigrid_config& cfg, bool with_norm) {
  const std::string key = graph_key(with_norm ? "outer" : "vcycle", x, b, cfg);
  auto it = h->graphs.find(key);
  if (it != h->graphs.end()) return it->second;
  prune_graphs(h);
  pf_hierarchy::GraphEntry e;
  e.x_uid = x->uid;
  e.b_uid = b->uid;
  cudaGraph_t g = nullptr;
  trace("outer graph: capture", h->rank_base);
  PF_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  g_capture_counter = &e.kernels;
  try {
    for (int j = 0; j < cfg.cycles; ++j) enq_vcycle(h, x, b->cur(), cfg);
    if (with_norm) {
      const int top = h->n_levels - 1;
      enq_resnorm(h, top, x->cur(), b->cur());
      PF_CUDA(cudaMemcpyAsync(h->pinned, h->levels[top].norm.p, sizeof(double),
                              cudaMemcpyDeviceToHost, h->stream));
    }
  } catch (...) {
    g_capture_counter = nullptr;
    cudaStreamEndCapture(h->stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  g_capture_counter = nullptr;
  PF_CUDA(cudaStreamEndCapture(h->stream, &g));
  trace("outer graph: captured", h->rank_base);
  PF_CUDA(cudaGraphInstantiate(&e.exec, g, 0));
  trace("outer graph: instantiated", h->rank_base);
  PF_CUDA(cudaGraphDestroy(g));
  return h->graphs.emplace(key, e).first->second;
}

void graph_launch(pf_hierarchy* h, pf_hierarchy::GraphEntry& e) {
  PF_CUDA(cudaGraphLaunch(e.exec, h->stream));
  h->launches += e.kernels;
}

void solve_outer_dev(pf_hierarchy* h, pf_vector* x, const pf_vector* b, const pf_multigrid_config& cfg,
                     pf_solve_stats* st, double* residuals, int max_res) {
  trace("solve_outer_dev");
  validate_cfg(cfg);
  const int top = h->n_levels - 1;
  const double t0 = wall_now();
  pf_solve_stats s{};
  if (h->world == h->n_sub && !h->opt.solve_mode_host) {
    auto& g = solve_graph(h, x, b, cfg);
    trace("solve graph: launch");
    PF_CUDA(cudaGraphLaunch(g.exec, h->stream));
    sync(h);
    trace("solve graph: done");
    const auto* ss = static_cast<const SolveState*>(g.host_state);
    const int m = ss->launches - 1;  // cycles completed
    h->launches += g.head_kernels * ss->launches + g.kernels * m;
    s.initial_residual = ss->r0;
    s.iterations = m;
    s.final_residual = ss->last;
    s.converged = ss->converged;
    for (int i = 0; i < m && residuals && i < max_res; ++i) residuals[i] = ss->hist[i];
    s.solve_seconds = wall_now() - t0;
    if (st) *st = s;
    if (!s.converged) {
      std::ostringstream os;
      os << "multigrid stalled at relative residual " << s.final_residual / s.initial_residual;
      throw Error(PF_ERR_NO_CONVERGENCE, os.str());
    }
    return;
  }
  trace("solve: initial norm", h->rank_base);
  enq_resnorm(h, top, x->cur(), b->cur());
  const double r0 = read_norm(h, top);
  trace("solve: initial norm read", h->rank_base);
  s.initial_residual = r0;
  s.final_residual = r0;
  s.converged = 1;
  if (r0 != 0.0) {
    s.converged = 0;
    const bool eager = h->xport && !h->xport->capturable();
    pf_hierarchy::GraphEntry* g = eager ? nullptr : &outer_graph(h, x, b, cfg, true);
    for (int outer = 1; outer <= cfg.outer_max_cycles; ++outer) {
      if (g) {
        trace("solve: cycle graph launch", h->rank_base);
        graph_launch(h, *g);
      } else {
        for (int j = 0; j < cfg.cycles; ++j) enq_vcycle(h, x, b->cur(), cfg);
        enq_resnorm(h, top, x->cur(), b->cur());
        PF_CUDA(cudaMemcpyAsync(h->pinned, h->levels[top].norm.p, sizeof(double),
                                cudaMemcpyDeviceToHost, h->stream));
      }
      sync(h);
      trace("solve: cycle done", h->rank_base);
      const double r = h->pinned[0];
      s.iterations = outer;
      if (residuals && outer <= max_res) residuals[outer - 1] = r;
      s.final_residual = r;
      if (r <= cfg.outer_tol * r0) {
        s.converged = 1;
        break;
      }
    }
  }
  s.solve_seconds = wall_now() - t0;
  if (st) *st = s;
  if (!s.converged) {
    std::ostringstream os;
    os << "multigrid stalled at relative residual " << s.final_residual / r0;
    throw Error(PF_ERR_NO_CONVERGENCE, os.str());
  }
}

void upload_vec(pf_hierarchy* h, pf_vector* v, int s, const double* host, int64_t n) {
  DevLevel& D = h->levels[v->level].sub[s];
  if (n != D.n)
    invalid("vector length " + std::to_string(n) + " does not match mapper dof count " + std::to_string(D.n));
  PF_CUDA(cudaMemcpyAsync(h->staging.p, host, sizeof(double) * n, cudaMemcpyHostToDevice, h->stream));
  launcher(h)(grid_for(n), kBlock, k_scatter_perm, static_cast<const double*>(h->staging.p),
              static_cast<const int32_t*>(D.d_perm.p), v->cur() + D.offset, D.n);
}

void download_vec(pf_hierarchy* h, const pf_vector* v, int s, double* host, int64_t n) {
  DevLevel& D = h->levels[v->level].sub[s];
  if (n != D.n)
    invalid("vector length " + std::to_string(n) + " does not match mapper dof count " + std::to_string(D.n));
  launcher(h)(grid_for(n), kBlock, k_gather_perm, static_cast<const double*>(v->cur() + D.offset),
              static_cast<const int32_t*>(D.d_perm.p), h->staging.p, D.n);
  PF_CUDA(cudaMemcpyAsync(host, h->staging.p, sizeof(double) * n, cudaMemcpyDeviceToHost, h->stream));
}

pf_vector* new_vector(pf_hierarchy* h, int level) {
  static std::atomic<uint64_t> next_uid{1};
  auto* v = new pf_vector;
  v->uid = next_uid++;
  v->registry = h->vectors;
  {
    std::lock_guard<std::mutex> g(h->vectors->mu);
    h->vectors->live.insert(v->uid);
  }
  v->h = h;
  v->device = h->device;
  v->level = level;
  v->total = h->levels[level].total;
  v->data.alloc(2 * std::max<int64_t>(v->total, 1));
  PF_CUDA(cudaMemsetAsync(v->data.p, 0, sizeof(double) * 2 * std::max<int64_t>(v->total, 1), h->stream));
  return v;
}

}  // namespace rt

// Kernel-launch accounting and the PDL switch for launches made outside this file
// (pf_peer.cu).
int64_t* launch_counter(pf_hierarchy* h) { return rt::g_capture_counter ? rt::g_capture_counter : &h->launches; }
bool pdl_on(const pf_hierarchy* h) { return h->opt.pdl != 0; }
// pf_peer.cu
int64_t peer_export(pf_hierarchy* h, void* buf, int64_t cap);
void peer_import(pf_hierarchy* h, const void* blobs, int64_t stride);

}  // namespace pf

using namespace pf::rt;

pf_hierarchy::~pf_hierarchy() {
  cudaSetDevice(device);
  for (auto& [k, e] : graphs) {
    if (e.exec) cudaGraphExecDestroy(e.exec);
    if (e.state) cudaFree(e.state);
    if (e.host_state) cudaFreeHost(e.host_state);
  }
  for (pf::Level& L : levels) {
    delete L.x;
    delete L.b;
  }
  levels.clear();
  xport.reset();
  if (pinned) cudaFreeHost(pinned);
  if (ev0) cudaEventDestroy(ev0);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (comm_stream) cudaStreamDestroy(comm_stream);
  if (ev1) cudaEventDestroy(ev1);
  if (stream) cudaStreamDestroy(stream);
}

extern "C" {

const char* pf_last_error(void) { return pf::g_last_error.c_str(); }

const char* pf_version(void) {
  return "paper_1609_04809_b200 pf_gpu 0.2 (sm_100a; SELL-32x4 fp64 operators, 8/16-bit lossless value index)";
}

pf_status pf_set_host_threads(int n, int* out) {
  PF_API_BEGIN
  omp_set_num_threads(n > 0 ? n : omp_get_num_procs());
  if (out) *out = omp_get_max_threads();
  PF_API_END
}

pf_status pf_device_count(int* out) {
  PF_API_BEGIN
  if (!out) invalid("null output");
  PF_CUDA(cudaGetDeviceCount(out));
  PF_API_END
}

void pf_default_smoother_config(pf_smoother_config* o) {
  o->kind = PF_SMOOTHER_GAUSS_SEIDEL;  // solvers.hpp:10
  o->sweeps = 3;
  o->local_sweeps = 1;
  o->damping = 0.8;
}

void pf_default_multigrid_config(pf_multigrid_config* o) {
  o->cycles = 1;  // multigrid.hpp:53-62
  pf_default_smoother_config(&o->smoother);
  o->pre_smooth = 3;
  o->post_smooth = 3;
  o->coarse_tol = 1e-12;
  o->coarse_max_iter = 20000;
  o->outer_tol = 1e-9;
  o->outer_max_cycles = 100;
}

pf_status pf_hierarchy_create(int device, int n_levels, int n_subdomains, int rank_base,
                              int world_size, pf_hierarchy** out) {
  PF_API_BEGIN
  if (!out) invalid("null output");
  if (n_levels < 1) invalid("hierarchy needs at least one level");
  if (n_subdomains < 1 || world_size < n_subdomains || rank_base < 0 ||
      rank_base + n_subdomains > world_size)
    invalid("bad subdomain / rank layout");
  if (n_subdomains != world_size && n_subdomains != 1)
    invalid("several subdomains per device are only supported when all ranks are local");
  PF_CUDA(cudaSetDevice(device));
  auto h = std::make_unique<pf_hierarchy>();
  h->device = device;
  h->n_levels = n_levels;
  h->n_sub = n_subdomains;
  h->rank_base = rank_base;
  h->world = world_size;
  h->opt = options_from_env();
  h->levels.resize(static_cast<size_t>(n_levels));
  for (auto& L : h->levels) L.host.resize(static_cast<size_t>(n_subdomains));
  PF_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  PF_CUDA(cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking));
  PF_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  PF_CUDA(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  PF_CUDA(cudaEventCreate(&h->ev0));
  PF_CUDA(cudaEventCreate(&h->ev1));
  PF_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h->pinned), 64 * sizeof(double)));
  *out = h.release();
  PF_API_END
}

pf_status pf_hierarchy_set_option(pf_hierarchy* h, const char* name, int64_t value) {
  PF_API_BEGIN
  if (!h) invalid("null hierarchy");
  const OptionSpec* o = find_option(name);
  if (!o) invalid(std::string("unknown option ") + (name ? name : "(null)"));
  if (o->build && h->finalized) state(std::string("option ") + o->name + " shapes the device layout: set it before pf_hierarchy_finalize");
  if (h->opt.*o->field != value) {
    h->opt.*o->field = value;
    if (h->finalized) drop_graphs(h);  // captured launches may depend on it
  }
  PF_API_END
}

pf_status pf_hierarchy_get_option(const pf_hierarchy* h, const char* name, int64_t* out) {
  PF_API_BEGIN
  if (!h || !out) invalid("null argument");
  const OptionSpec* o = find_option(name);
  if (!o) invalid(std::string("unknown option ") + (name ? name : "(null)"));
  *out = h->opt.*o->field;
  PF_API_END
}

pf_status pf_debug_guard_failures(int64_t* out) {
  PF_API_BEGIN
  if (!out) invalid("null output");
  *out = g_guard_failures.load();
  PF_API_END
}

pf_status pf_debug_guard_selftest(int device, int* detected) {
  PF_API_BEGIN
  if (!detected) invalid("null output");
  PF_CUDA(cudaSetDevice(device));
  const int64_t before = g_guard_failures.load();
  {
    DevBuf<double> v;
    v.alloc(100, true);
    k_fill<<<1, kBlock>>>(v.p, 1.0, 101);  // one element past the end
    PF_CUDA(cudaGetLastError());
  }
  *detected = static_cast<int>(g_guard_failures.load() - before);
  g_guard_failures = before;  // the planted hit is not a failure of the run
  PF_API_END
}

pf_status pf_option_names(char* buf, int64_t capacity) {
  PF_API_BEGIN
  std::string all;
  for (const OptionSpec& o : kOptions) {
    if (!all.empty()) all += ' ';
    all += o.name;
    all += o.build ? ":build" : ":launch";
  }
  if (!buf || capacity < static_cast<int64_t>(all.size()) + 1) invalid("buffer too small for the option names");
  std::memcpy(buf, all.c_str(), all.size() + 1);
  PF_API_END
}

pf_status pf_hierarchy_set_level(pf_hierarchy* h, int level, int sub, const pf_level_desc* d) {
  PF_API_BEGIN
  if (!h || !d) invalid("null argument");
  if (h->finalized) state("hierarchy already finalized");
  if (level < 0 || level >= h->n_levels) invalid("level out of range");
  if (sub < 0 || sub >= h->n_sub) invalid("subdomain out of range");
  h->levels[level].host[sub] = parse_desc(*d, h->rank_base + sub, h->world, level > 0);
  PF_API_END
}

pf_status pf_hierarchy_set_level_from_setup(pf_hierarchy* h, int level, int sub, pf_setup* s) {
  PF_API_BEGIN
  if (!h) invalid("null hierarchy");
  if (h->finalized) state("hierarchy already finalized");
  if (level < 0 || level >= h->n_levels) invalid("level out of range");
  if (sub < 0 || sub >= h->n_sub) invalid("subdomain out of range");
  pf::adopt_setup_level(s, level, h->levels[level].host[sub]);
  PF_API_END
}

pf_status pf_hierarchy_set_replica_level(pf_hierarchy* h, int level, int rank, const pf_level_desc* d) {
  PF_API_BEGIN
  if (!h || !d) invalid("null argument");
  if (h->finalized) state("hierarchy already finalized");
  if (rank < 0 || rank >= h->world) invalid("rank out of range");
  if (level < 0 || level >= h->n_levels) invalid("level out of range");
  auto& R = h->rep;
  if (R.lv.size() <= static_cast<size_t>(level)) R.lv.resize(static_cast<size_t>(level) + 1);
  auto& RL = R.lv[static_cast<size_t>(level)];
  if (RL.host.empty()) RL.host.resize(static_cast<size_t>(h->world));
  RL.host[rank] = parse_desc(*d, rank, h->world, level > 0);
  PF_API_END
}

pf_status pf_hierarchy_set_coarse_replica(pf_hierarchy* h, int rank, const pf_level_desc* d) {
  return pf_hierarchy_set_replica_level(h, 0, rank, d);
}

pf_status pf_hierarchy_finalize(pf_hierarchy* h) {
  PF_API_BEGIN
  if (!h) invalid("null hierarchy");
  if (h->finalized) state("hierarchy already finalized");
  PF_CUDA(cudaSetDevice(h->device));
  int64_t max_total = 1;
  for (int l = 0; l < h->n_levels; ++l) {
    Level& L = h->levels[l];
    L.sub.resize(static_cast<size_t>(h->n_sub));
    int64_t off = 0;
    for (int s = 0; s < h->n_sub; ++s) {
      if (!L.host[s].set)
        state("level " + std::to_string(l) + " subdomain " + std::to_string(s) + " not set");
      build_dev_level(L.host[s], L.sub[s], l, h->opt);
      if (h->world != h->n_sub) {  // the own rows reading a non-own copy (build_fused_plans)
        const HostLevel& H = L.host[s];
        DevLevel& D = L.sub[s];
        D.reads_nonown.assign(static_cast<size_t>(D.n), 0);
#pragma omp parallel for schedule(static)
        for (int32_t i = 0; i < H.n_own; ++i) {
          bool p = false;
          for (int64_t k = H.rowptr[i]; k < H.rowptr[i + 1] && !p; ++k) p = H.cols[k] >= H.n_own;
          D.reads_nonown[static_cast<size_t>(D.perm[i])] = p ? 1 : 0;
        }
      }
      if (l > 0) {  // the operator is on the device; level 0 keeps its CSR for the coarse pack
        std::vector<int32_t>().swap(L.host[s].cols);
        std::vector<double>().swap(L.host[s].vals);
      }
      L.sub[s].offset = off;
      off += L.sub[s].n;
      max_total = std::max<int64_t>(max_total, L.sub[s].n);
    }
    L.total = off;
    if (off >= (int64_t(1) << 31)) invalid("level too large for int32 device indices");
    PhaseTimer tm;
    if (l > 0)
      for (int s = 0; s < h->n_sub; ++s)
        build_transfer(L.host[s], L.sub[s], h->levels[l - 1].host[s], h->levels[l - 1].sub[s], h->opt);
    tm("transfer", l);
    build_plans(h, l);
    tm("plans", l);
    if (l > 0)  // the prolongation is on the device too
      for (HostLevel& H : L.host) {
        std::vector<int32_t>().swap(H.p_col);
        std::vector<double>().swap(H.p_w);
      }
    L.r.alloc(std::max<int64_t>(off, 1));
    L.sumsq.alloc(1 + std::max(h->world, h->n_sub));
    L.norm.alloc(1);
    L.coarse_stats.alloc(4);
    PF_CUDA(cudaMemset(L.coarse_stats.p, 0, 4 * sizeof(double)));
    if (l == 0) {
      std::vector<CoarseSub> cs;
      for (DevLevel& D : L.sub) cs.push_back(CoarseSub{view(D.A), D.d_perm.p, D.n_own, D.offset});
      L.coarse_subs.upload(cs);
      if (h->world == h->n_sub)
        L.cpack = make_coarse_pack(L.host, L.sub, L.scatter, L.cp_sub_rows, L.cp_rowptr, L.cp_rowdev,
                                   L.cp_cols, L.cp_vals);
    }
  }
  // load policy of the operators: the levels below the finest that fit the L2 budget are
  // read with the caching policy (vk_dispatch_rows)
  for (int l = 0; l + 1 < h->n_levels; ++l)
    for (DevLevel& D : h->levels[l].sub)
      for (DevSell* S : {&D.A, &D.P, &D.R})
        S->keep_l2 = S->vals.bytes() + S->cols.bytes() + S->row_len.bytes() + S->slice_ptr.bytes() <=
                     h->opt.cached_max_bytes;
  if (h->world != h->n_sub) build_replica(h);
  h->staging.alloc(max_total);
  for (int l = 0; l < h->n_levels; ++l) {
    h->levels[l].x = new_vector(h, l);
    h->levels[l].b = new_vector(h, l);
  }
  build_bottom(h);
  if (h->world != h->n_sub) build_rep_bottom(h);
  // the host copies go; one subdomain keeps level 0 (pf_hierarchy_set_coarse_direct)
  for (int l = 0; l < h->n_levels; ++l)
    if (l > 0 || h->world != 1 || h->n_sub != 1) h->levels[l].host.clear();
  for (auto& RL : h->rep.lv) RL.host.clear();
  PF_CUDA(cudaStreamSynchronize(h->stream));
  h->finalized = true;
  PF_API_END
}

pf_status pf_nccl_unique_id(void* out, int nbytes) {
  PF_API_BEGIN
  pf::nccl_unique_id(out, nbytes);
  PF_API_END
}

pf_status pf_nccl_selftest(int device, int* ok) {
  PF_API_BEGIN
  if (!ok) invalid("null output");
  *ok = 0;
  PF_CUDA(cudaSetDevice(device));
  unsigned char id[128];
  pf::nccl_unique_id(id, 128);
  auto comm = pf::nccl_init(0, 1, id, 128);
  cudaStream_t st;
  PF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  DevBuf<double> buf;
  buf.alloc(8);
  const double host[4] = {1.5, -2.25, 3.0, 0.0};
  PF_CUDA(cudaMemcpy(buf.p, host, sizeof host, cudaMemcpyHostToDevice));
  comm->group_start();
  comm->send(buf.p, 2, 0, st);      // [1.5, -2.25] to itself
  comm->recv(buf.p + 4, 2, 0, st);  // into [4, 6)
  comm->group_end(st);
  comm->allgather(buf.p + 2, buf.p + 6, 1, st);  // one rank: [3.0] -> [6]
  PF_CUDA(cudaStreamSynchronize(st));
  comm->check_async();
  double out[8];
  PF_CUDA(cudaMemcpy(out, buf.p, sizeof out, cudaMemcpyDeviceToHost));
  PF_CUDA(cudaStreamDestroy(st));
  *ok = out[4] == 1.5 && out[5] == -2.25 && out[6] == 3.0;
  PF_API_END
}

pf_status pf_hierarchy_set_fused_exchanges(pf_hierarchy* h, int on) {
  PF_API_BEGIN
  if (!h) invalid("null hierarchy");
  if (h->finalized) state("set fused exchanges before pf_hierarchy_finalize");
  h->fused = on != 0;
  PF_API_END
}

pf_status pf_hierarchy_set_colorwise_exchange(pf_hierarchy* h, int on) {
  PF_API_BEGIN
  if (!h) invalid("null hierarchy");
  h->colorwise = on != 0;
  if (h->finalized) drop_graphs(h);  // captured smoothing phases change
  PF_API_END
}

pf_status pf_hierarchy_set_coarse_direct(pf_hierarchy* h, int on) {
  PF_API_BEGIN
  if (!h) invalid("null hierarchy");
  if (!h->finalized) state("set the direct coarse solve after pf_hierarchy_finalize");
  if (h->world != 1 || h->n_sub != 1) invalid("the direct coarse solve needs one subdomain in one process");
  PF_CUDA(cudaSetDevice(h->device));
  Level& L = h->levels[0];
  if (on) {
    if (coarse_pack_smem(L.cpack) > kCoarseSmemMax) invalid("coarse level too large for the direct solve");
    if (L.host.empty() || L.host[0].rowptr.empty()) state("level 0 host data not kept");
    const HostLevel& H = L.host[0];
    const int n = H.n_own;
    std::vector<double> A(static_cast<size_t>(n) * n, 0.0), inv(static_cast<size_t>(n) * n, 0.0);
    for (int i = 0; i < n; ++i)
      for (int64_t k = H.rowptr[i]; k < H.rowptr[i + 1]; ++k)
        if (H.cols[k] < n) A[static_cast<size_t>(i) * n + H.cols[k]] = H.vals[k];
    gauss_jordan_inverse(n, A, inv);
    h->coarse_inv.upload(inv);
    L.cpack.inv = h->coarse_inv.p;
    L.cpack.n_own_dev = n;
  } else {
    L.cpack.inv = nullptr;
  }
  if (h->bot.active)
    PF_CUDA(cudaMemcpy(static_cast<char*>(h->bot.desc) + offsetof(BotDesc, coarse), &L.cpack, sizeof(CoarsePack),
                       cudaMemcpyHostToDevice));
  drop_graphs(h);  // captured launches carry the old pack
  PF_API_END
}

pf_status pf_hierarchy_init_nccl(pf_hierarchy* h, const void* id, int nbytes) {
  PF_API_BEGIN
  if (!h) invalid("null hierarchy");
  if (h->world == h->n_sub) state("NCCL is only used when ranks live in separate processes");
  PF_CUDA(cudaSetDevice(h->device));
  if (h->xport) state("transport already initialized");
  {
    auto nc = pf::nccl_init(h->rank_base, h->world, id, nbytes);
    if (const char* e = std::getenv("PF_WATCHDOG_S")) nc->watchdog = std::atof(e);
    h->xport = std::move(nc);
  }
  PF_API_END
}

pf_status pf_hierarchy_peer_export(pf_hierarchy* h, void* blob, int64_t capacity, int64_t* size) {
  PF_API_BEGIN
  if (!h || !size) invalid("null argument");
  if (!h->finalized) state("export the peer arena after pf_hierarchy_finalize");
  if (h->world == h->n_sub) state("the peer transport is only used when ranks live in separate hierarchies");
  PF_CUDA(cudaSetDevice(h->device));
  *size = pf::peer_export(h, blob, capacity);
  PF_API_END
}

pf_status pf_hierarchy_init_peer(pf_hierarchy* h, const void* blobs, int64_t stride) {
  PF_API_BEGIN
  if (!h || !blobs) invalid("null argument");
  if (stride <= 0) invalid("blob stride must be positive");
  PF_CUDA(cudaSetDevice(h->device));
  pf::peer_import(h, blobs, stride);
  drop_graphs(h);
  PF_API_END
}

pf_status pf_hierarchy_drop_transport(pf_hierarchy* h) {
  PF_API_BEGIN
  if (!h) invalid("null hierarchy");
  PF_CUDA(cudaSetDevice(h->device));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  drop_graphs(h);  // captured exchanges use the old transport
  h->xport.reset();
  PF_API_END
}

pf_status pf_loopback_create(int world_size, void** hub) {
  PF_API_BEGIN
  if (!hub || world_size < 1) invalid("bad argument");
  *hub = new pf::LoopbackHub(world_size);
  PF_API_END
}

pf_status pf_loopback_destroy(void* hub) {
  PF_API_BEGIN
  delete static_cast<pf::LoopbackHub*>(hub);
  PF_API_END
}

pf_status pf_hierarchy_init_loopback(pf_hierarchy* h, void* hub) {
  PF_API_BEGIN
  if (!h || !hub) invalid("null argument");
  if (h->world == h->n_sub) state("loopback is only used when ranks live in separate hierarchies");
  if (h->xport) state("transport already initialized");
  auto* H = static_cast<pf::LoopbackHub*>(hub);
  if (H->world != h->world) invalid("loopback hub size differs from the world size");
  auto t = std::make_unique<pf::Loopback>();
  t->hub = H;
  t->rank = h->rank_base;
  h->xport = std::move(t);
  PF_API_END
}

pf_status pf_hierarchy_destroy(pf_hierarchy* h) {
  PF_API_BEGIN
  delete h;
  PF_API_END
}

pf_status pf_hierarchy_device_bytes(const pf_hierarchy* h, int64_t* out) {
  PF_API_BEGIN
  if (!h || !out) invalid("null argument");
  int64_t b = 0;
  for (const Level& L : h->levels) {
    for (const DevLevel& D : L.sub)
      b += D.A.vals.bytes() + D.A.cols.bytes() + D.A.slice_ptr.bytes() + D.A.row_len.bytes() +
           D.P.vals.bytes() + D.P.cols.bytes() + D.P.slice_ptr.bytes() + D.P.row_len.bytes() +
           D.R.vals.bytes() + D.R.cols.bytes() + D.R.slice_ptr.bytes() + D.R.row_len.bytes() +
           D.d_perm.bytes() + D.d_is_dir.bytes();
    b += L.r.bytes() + (L.x ? L.x->data.bytes() : 0) + (L.b ? L.b->data.bytes() : 0);
  }
  *out = b;
  PF_API_END
}

pf_status pf_vector_create(pf_hierarchy* h, int level, pf_vector** out) {
  PF_API_BEGIN
  check_level(h, level);
  if (!out) invalid("null output");
  PF_CUDA(cudaSetDevice(h->device));
  *out = new_vector(h, level);
  PF_CUDA(cudaStreamSynchronize(h->stream));
  PF_API_END
}

pf_status pf_vector_destroy(pf_vector* v) {
  PF_API_BEGIN
  if (v) {
    cudaSetDevice(v->device);
    if (auto reg = v->registry.lock()) {  // the hierarchy is alive: its graphs on v go stale
      std::lock_guard<std::mutex> g(reg->mu);
      reg->live.erase(v->uid);
    }
  }
  delete v;
  PF_API_END
}

pf_status pf_vector_upload(pf_vector* v, int sub, const double* host, int64_t n) {
  PF_API_BEGIN
  if (!v || !host) invalid("null argument");
  pf_hierarchy* h = v->h;
  if (sub < 0 || sub >= h->n_sub) invalid("subdomain out of range");
  PF_CUDA(cudaSetDevice(h->device));
  upload_vec(h, v, sub, host, n);
  sync(h);
  PF_API_END
}

pf_status pf_vector_download(const pf_vector* v, int sub, double* host, int64_t n) {
  PF_API_BEGIN
  if (!v || !host) invalid("null argument");
  pf_hierarchy* h = v->h;
  if (sub < 0 || sub >= h->n_sub) invalid("subdomain out of range");
  PF_CUDA(cudaSetDevice(h->device));
  download_vec(h, v, sub, host, n);
  sync(h);
  PF_API_END
}

pf_status pf_vector_fill(pf_vector* v, double value) {
  PF_API_BEGIN
  if (!v) invalid("null vector");
  PF_CUDA(cudaSetDevice(v->h->device));
  launcher(v->h)(grid_for(2 * v->total), kBlock, k_fill, v->data.p, value, 2 * v->total);
  sync(v->h);
  PF_API_END
}

pf_status pf_vector_copy(const pf_vector* src, pf_vector* dst) {
  PF_API_BEGIN
  if (!src || !dst) invalid("null vector");
  if (src->h != dst->h || src->level != dst->level) invalid("vectors of different levels");
  PF_CUDA(cudaSetDevice(src->h->device));
  enq_copy(src->h, src->cur(), dst->cur(), src->total);
  sync(src->h);
  PF_API_END
}

pf_status pf_host_alloc(void** out, int64_t bytes) {
  PF_API_BEGIN
  if (!out || bytes < 0) invalid("bad argument");
  PF_CUDA(cudaMallocHost(out, static_cast<size_t>(std::max<int64_t>(bytes, 8))));
  PF_API_END
}

pf_status pf_host_free(void* p) {
  PF_API_BEGIN
  if (p) PF_CUDA(cudaFreeHost(p));
  PF_API_END
}

pf_status pf_spmv(pf_hierarchy* h, int level, const pf_vector* x, pf_vector* y) {
  PF_API_BEGIN
  check_level(h, level);
  check_vec(h, x, level, "x");
  check_vec(h, y, level, "y");
  PF_CUDA(cudaSetDevice(h->device));
  enq_spmv(h, level, x->cur(), y->cur());
  sync(h);
  PF_API_END
}

pf_status pf_residual_norm(pf_hierarchy* h, int level, const pf_vector* x, const pf_vector* b, double* out) {
  PF_API_BEGIN
  check_level(h, level);
  check_vec(h, x, level, "x");
  check_vec(h, b, level, "b");
  if (!out) invalid("null output");
  PF_CUDA(cudaSetDevice(h->device));
  enq_resnorm(h, level, x->cur(), b->cur());
  *out = read_norm(h, level);
  PF_API_END
}

pf_status pf_smooth(pf_hierarchy* h, int level, pf_vector* x, const pf_vector* b, const pf_smoother_config* cfg) {
  PF_API_BEGIN
  check_level(h, level);
  check_vec(h, x, level, "x");
  check_vec(h, b, level, "b");
  if (!cfg) invalid("null config");
  if (cfg->kind < 0 || cfg->kind > 2) invalid("unknown smoother kind");
  if (cfg->sweeps < 0 || cfg->local_sweeps < 0) invalid("negative sweep count");
  PF_CUDA(cudaSetDevice(h->device));
  enq_smooth(h, level, x, b->cur(), *cfg);
  sync(h);
  PF_API_END
}

pf_status pf_coarse_solve(pf_hierarchy* h, int level, pf_vector* x, const pf_vector* b, double tol,
                          int max_iter, pf_solve_stats* stats) {
  PF_API_BEGIN
  check_level(h, level);
  check_vec(h, x, level, "x");
  check_vec(h, b, level, "b");
  PF_CUDA(cudaSetDevice(h->device));
  const double t0 = wall_now();
  enq_coarse(h, level, x->cur(), b->cur(), tol, max_iter, false);
  double st[4];
  PF_CUDA(cudaMemcpyAsync(h->pinned, h->levels[level].coarse_stats.p, 4 * sizeof(double),
                          cudaMemcpyDeviceToHost, h->stream));
  sync(h);
  std::memcpy(st, h->pinned, sizeof st);
  if (stats) {
    stats->iterations = static_cast<int32_t>(st[0]);
    stats->converged = static_cast<int32_t>(st[1]);
    stats->initial_residual = st[2];
    stats->final_residual = st[3];
    stats->solve_seconds = wall_now() - t0;
    stats->comm_seconds = 0;
  }
  PF_API_END
}

pf_status pf_prolongate(pf_hierarchy* h, int fine, const pf_vector* coarse, pf_vector* out) {
  PF_API_BEGIN
  check_level(h, fine);
  if (fine == 0) invalid("level 0 has no parent");
  check_vec(h, coarse, fine - 1, "coarse");
  check_vec(h, out, fine, "out");
  PF_CUDA(cudaSetDevice(h->device));
  enq_prolong(h, fine, coarse->cur(), out->cur(), 0);
  sync(h);
  PF_API_END
}

pf_status pf_restrict_residual(pf_hierarchy* h, int fine, const pf_vector* r, pf_vector* rc) {
  PF_API_BEGIN
  check_level(h, fine);
  if (fine == 0) invalid("level 0 has no parent");
  check_vec(h, r, fine, "r");
  check_vec(h, rc, fine - 1, "rc");
  PF_CUDA(cudaSetDevice(h->device));
  enq_restrict(h, fine, r->cur(), rc->cur(), nullptr, 0);
  enq_update_ms(h, fine - 1, rc->cur(), PF_UPDATE_ACCUMULATE_THEN_SCATTER);
  sync(h);
  PF_API_END
}

pf_status pf_update_master_slave(pf_hierarchy* h, int level, pf_vector* v, int mode) {
  PF_API_BEGIN
  check_level(h, level);
  check_vec(h, v, level, "v");
  if (mode != PF_UPDATE_SCATTER && mode != PF_UPDATE_ACCUMULATE_THEN_SCATTER) invalid("bad update mode");
  PF_CUDA(cudaSetDevice(h->device));
  enq_update_ms(h, level, v->cur(), mode);
  sync(h);
  PF_API_END
}

pf_status pf_update_halo1(pf_hierarchy* h, int level, pf_vector* v) {
  PF_API_BEGIN
  check_level(h, level);
  check_vec(h, v, level, "v");
  PF_CUDA(cudaSetDevice(h->device));
  enq_scatter(h, level, PF_CH_HALO1, v->cur());
  sync(h);
  PF_API_END
}

pf_status pf_update_halo2(pf_hierarchy* h, int level, pf_vector* v) {
  PF_API_BEGIN
  check_level(h, level);
  check_vec(h, v, level, "v");
  PF_CUDA(cudaSetDevice(h->device));
  enq_scatter(h, level, PF_CH_HALO2, v->cur());
  sync(h);
  PF_API_END
}

pf_status pf_allreduce_sum(pf_hierarchy* h, const double* per_sub, double* out) {
  PF_API_BEGIN
  check_level(h, 0);
  if (!per_sub || !out) invalid("null argument");
  PF_CUDA(cudaSetDevice(h->device));
  Level& L = h->levels[0];
  PF_CUDA(cudaMemcpyAsync(L.sumsq.p, per_sub, sizeof(double) * h->n_sub, cudaMemcpyHostToDevice, h->stream));
  enq_allreduce(h, L, false);
  *out = read_norm(h, 0);
  PF_API_END
}

pf_status pf_v_cycle(pf_hierarchy* h, pf_vector* x, const pf_vector* b, const pf_multigrid_config* cfg,
                     pf_solve_stats* stats) {
  PF_API_BEGIN
  check_level(h, h ? h->n_levels - 1 : 0);
  check_vec(h, x, h->n_levels - 1, "x");
  check_vec(h, b, h->n_levels - 1, "b");
  if (!cfg) invalid("null config");
  validate_cfg(*cfg);
  PF_CUDA(cudaSetDevice(h->device));
  const double t0 = wall_now();
  enq_vcycle(h, x, b->cur(), *cfg);
  PF_CUDA(cudaMemcpyAsync(h->pinned, h->levels[0].coarse_stats.p, 4 * sizeof(double),
                          cudaMemcpyDeviceToHost, h->stream));
  sync(h);
  if (stats) {
    stats->iterations = static_cast<int32_t>(h->pinned[0]);
    stats->converged = static_cast<int32_t>(h->pinned[1]);
    stats->initial_residual = h->pinned[2];
    stats->final_residual = h->pinned[3];
    stats->solve_seconds = wall_now() - t0;
    stats->comm_seconds = 0;
  }
  PF_API_END
}

pf_status pf_solve_outer(pf_hierarchy* h, pf_vector* x, const pf_vector* b, const pf_multigrid_config* cfg,
                         pf_solve_stats* stats, double* residuals, int max_residuals) {
  trace("pf_solve_outer");
  PF_API_BEGIN
  check_level(h, h ? h->n_levels - 1 : 0);
  check_vec(h, x, h->n_levels - 1, "x");
  check_vec(h, b, h->n_levels - 1, "b");
  if (!cfg) invalid("null config");
  PF_CUDA(cudaSetDevice(h->device));
  solve_outer_dev(h, x, b, *cfg, stats, residuals, max_residuals);
  PF_API_END
}

pf_status pf_solve_outer_host(pf_hierarchy* h, double* const* x_host, const double* const* b_host,
                              const pf_multigrid_config* cfg, pf_solve_stats* stats, double* residuals,
                              int max_residuals) {
  PF_API_BEGIN
  check_level(h, h ? h->n_levels - 1 : 0);
  if (!x_host || !b_host || !cfg) invalid("null argument");
  PF_CUDA(cudaSetDevice(h->device));
  const int top = h->n_levels - 1;
  Level& T = h->levels[top];
  // the finest level's own scratch vectors carry the user's x and b
  for (int s = 0; s < h->n_sub; ++s) {
    upload_vec(h, T.x, s, x_host[s], T.sub[s].n);
    upload_vec(h, T.b, s, b_host[s], T.sub[s].n);
  }
  pf_status rc = PF_OK;
  std::string msg;
  try {
    solve_outer_dev(h, T.x, T.b, *cfg, stats, residuals, max_residuals);
  } catch (const pf::Error& e) {
    if (e.code != PF_ERR_NO_CONVERGENCE) throw;
    rc = e.code;
    msg = e.what();
  }
  for (int s = 0; s < h->n_sub; ++s) {
    download_vec(h, T.x, s, x_host[s], T.sub[s].n);
    sync(h);  // staging buffer is shared between subdomains
  }
  if (rc != PF_OK) throw pf::Error(rc, msg);
  PF_API_END
}

pf_status pf_launch_count(const pf_hierarchy* h, int64_t* out) {
  PF_API_BEGIN
  if (!h || !out) invalid("null argument");
  *out = h->launches;
  PF_API_END
}

pf_status pf_hierarchy_graph_count(const pf_hierarchy* h, int64_t* out) {
  PF_API_BEGIN
  if (!h || !out) invalid("null argument");
  *out = static_cast<int64_t>(h->graphs.size());
  PF_API_END
}

pf_status pf_reset_launch_count(pf_hierarchy* h) {
  PF_API_BEGIN
  if (!h) invalid("null hierarchy");
  h->launches = 0;
  PF_API_END
}

pf_status pf_time_sweep(pf_hierarchy* h, int level, int kind, int iters, double* mean_ms, double* bytes) {
  PF_API_BEGIN
  check_level(h, level);
  if (iters < 1) invalid("iters must be >= 1");
  PF_CUDA(cudaSetDevice(h->device));
  Level& L = h->levels[level];
  DevLevel& D = L.sub[0];
  pf_vector* x = L.x;
  const double* b = L.b->cur();
  auto launch = launcher(h);
  auto one = [&](int i) {
    if (kind == PF_SMOOTHER_JACOBI) {
      const double* src = (i & 1) ? x->alt() : x->cur();
      double* dst = (i & 1) ? x->cur() : x->alt();
      enq_jacobi_sweep(h, D, src, dst, b, 0.8);
    } else {
      for (int c = 0; c < D.n_colors; ++c)
        enq_color_sweep(h, D, c, true, kind == PF_SMOOTHER_MULTICOLOR_SOR ? 1.2 : 1.0, x->cur(), b);
    }
  };
  for (int i = 0; i < 3; ++i) one(i);  // warm-up
  PF_CUDA(cudaEventRecord(h->ev0, h->stream));
  for (int i = 0; i < iters; ++i) one(i);
  PF_CUDA(cudaEventRecord(h->ev1, h->stream));
  sync(h);
  float ms = 0;
  PF_CUDA(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  if (mean_ms) *mean_ms = ms / iters;
  // B = 12 z + 4 n + 8 m + 8 n (b) + 8 n (out), n = own rows,
  // z = own nnz, m = distinct columns the own rows touch — with the stored value width
  // (8 B fp64, or a 1/2 B table index) in place of the 8 of the 12.
  if (bytes)
    *bytes = (4.0 + D.A.vals.value_bytes()) * D.A.own_nnz + 4.0 * D.n_own + 8.0 * D.own_cols_touched +
             16.0 * D.n_own;
  PF_API_END
}

pf_status pf_time_vcycle(pf_hierarchy* h, pf_vector* x, const pf_vector* b, const pf_multigrid_config* cfg,
                         int iters, double* mean_ms) {
  PF_API_BEGIN
  check_level(h, h ? h->n_levels - 1 : 0);
  check_vec(h, x, h->n_levels - 1, "x");
  check_vec(h, b, h->n_levels - 1, "b");
  if (!cfg || iters < 1) invalid("bad argument");
  validate_cfg(*cfg);
  PF_CUDA(cudaSetDevice(h->device));
  pf_multigrid_config one = *cfg;
  one.cycles = 1;
  auto& g = outer_graph(h, x, b, one, false);
  graph_launch(h, g);
  PF_CUDA(cudaEventRecord(h->ev0, h->stream));
  for (int i = 0; i < iters; ++i) graph_launch(h, g);
  PF_CUDA(cudaEventRecord(h->ev1, h->stream));
  sync(h);
  float ms = 0;
  PF_CUDA(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  *mean_ms = ms / iters;
  if (h->bot.stamps) {  // PF_BOTTOM_PROFILE: per-phase times of the last bottom launch
    unsigned long long st[256];
    PF_CUDA(cudaMemcpy(st, h->bot.stamps, sizeof st, cudaMemcpyDeviceToHost));
    const int n = static_cast<int>(st[255]) < 127 ? static_cast<int>(st[255]) : 127;
    std::fprintf(stderr, "[pf] bottom: %d phases, total %.2f us:", n, (st[n] - st[0]) / 1e3);
    for (int i = 1; i <= n; ++i) std::fprintf(stderr, " %.2f", (st[i] - st[i - 1]) / 1e3);
    std::fprintf(stderr, "\n");
    int nb = 0;
    while (nb < 126 && st[129 + nb] > 0) ++nb;
    if (nb > 0) {
      std::fprintf(stderr, "[pf] bottom block 0: %d phases, total %.2f us:", nb, (st[128 + nb] - st[128]) / 1e3);
      for (int i = 1; i <= nb; ++i) std::fprintf(stderr, " %.2f", (st[128 + i] - st[128 + i - 1]) / 1e3);
      std::fprintf(stderr, "\n");
    }
  }
  PF_API_END
}

pf_status pf_hierarchy_stream(const pf_hierarchy* h, void** stream) {
  PF_API_BEGIN
  if (!h || !stream) invalid("null argument");
  *stream = static_cast<void*>(h->stream);
  PF_API_END
}

pf_status pf_level_info(const pf_hierarchy* h, int level, int sub, int64_t* n_dofs, int64_t* n_own,
                        int64_t* nnz, int64_t* n_colors) {
  PF_API_BEGIN
  check_level(h, level);
  if (sub < 0 || sub >= h->n_sub) invalid("subdomain out of range");
  const DevLevel& D = h->levels[level].sub[sub];
  if (n_dofs) *n_dofs = D.n;
  if (n_own) *n_own = D.n_own;
  if (nnz) *nnz = D.A.nnz;
  if (n_colors) *n_colors = D.n_colors;
  PF_API_END
}

}  // extern "C"

