// pf_runtime.hpp — host-side runtime of the B200 GMG hot path (internal).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <unordered_set>
#include <stdexcept>
#include <string>
#include <vector>

#include "pf_gpu.h"
#include "pf_fe.h"
#include "pf_types.hpp"

namespace pf {

struct Error : std::runtime_error {
  pf_status code;
  Error(pf_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what);
#define PF_CUDA(x) ::pf::cuda_check((x), #x)

// Guard zones (PF_GUARD=1; memory checking in the tests, compute-sanitizer being closed on
// the GPU pool): every DevBuf is followed by kGuardBytes of 0xFF — NaN as a double, -1 as an
// index, so a kernel reading past an array feeds NaN or a wild index into a bit-exact
// comparison with the oracle — and the zone is verified when the buffer is freed: a write
// past the end is counted (pf_debug_guard_failures) and reported on stderr.
constexpr size_t kGuardBytes = 4096;
bool guard_on();
void guard_check(const void* zone, size_t bytes);

// Owning device buffer.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  int64_t n = 0;
  bool guarded = false;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), guarded(o.guarded) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { reset(); p = o.p; n = o.n; guarded = o.guarded; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { reset(); }
  void reset() {
    if (p) {
      if (guarded) guard_check(reinterpret_cast<const char*>(p) + bytes(), static_cast<size_t>(bytes()));
      cudaFree(p);
    }
    p = nullptr;
    n = 0;
  }
  void alloc(int64_t count, bool force_guard = false) {
    reset();
    n = count;
    guarded = force_guard || guard_on();
    if (count > 0) {
      const size_t b = sizeof(T) * static_cast<size_t>(count);
      PF_CUDA(cudaMalloc(&p, b + (guarded ? kGuardBytes : 0)));
      if (guarded) PF_CUDA(cudaMemset(reinterpret_cast<char*>(p) + b, 0xFF, kGuardBytes));
    }
  }
  void upload(const std::vector<T>& v) {
    alloc(static_cast<int64_t>(v.size()));
    if (!v.empty()) PF_CUDA(cudaMemcpy(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  }
  int64_t bytes() const { return n * static_cast<int64_t>(sizeof(T)); }
};

struct HostChannel {
  int kind = 0, peer = 0;
  std::vector<int32_t> send, recv;
};

// Deep copy of one pf_level_desc.
struct HostLevel {
  bool set = false;
  int32_t n = 0, n_own = 0;
  std::vector<int64_t> rowptr;
  std::vector<int32_t> cols;
  std::vector<double> vals;
  std::vector<uint8_t> owns_row, is_dir;
  std::vector<int32_t> color;
  std::vector<int64_t> order;  // optional device placement hint (pf_level_desc::row_order)
  std::vector<HostChannel> channels;
  std::vector<int64_t> p_off;
  std::vector<int32_t> p_col;
  std::vector<double> p_w;
};

// The stored values of a SELL-32 operator: fp64, or indices into a table of the distinct
// values (SellView::vkind).
struct DevVals {
  int vkind = 0;
  DevBuf<double> vals;
  DevBuf<uint8_t> vi8;
  DevBuf<uint16_t> vi16;
  DevBuf<double> table;
  int64_t bytes() const { return vals.bytes() + vi8.bytes() + vi16.bytes() + table.bytes(); }
  int value_bytes() const { return vkind == 1 ? 1 : vkind == 2 ? 2 : 8; }
};

// SELL-32 operator on the device.
struct DevSell {
  DevVals vals;
  DevBuf<int32_t> cols;
  DevBuf<int64_t> slice_ptr;
  DevBuf<int32_t> row_len;
  int64_t nnz = 0, own_nnz = 0, stored = 0;
  int32_t max_len = 0;  // longest row
  bool keep_l2 = false;  // read with the caching policy (kVKCached): coarse levels that fit L2
  bool smem_table = true;  // an 8-bit table is staged in shared memory by the row kernels (Options::vtab_smem)
};

// Block windows of a level operator (WinView, pf_types.hpp).
struct DevWin {
  bool on = false;
  DevBuf<uint16_t> cols16;
  DevBuf<int32_t> chunk_ptr, chunks;
  DevBuf<uint8_t> dpos;
  int32_t max_chunks = 0;  // largest block cover: the launches' dynamic shared memory
  size_t smem() const { return sizeof(double) * (kBlock + kWinChunk * static_cast<size_t>(max_chunks)); }
};

// One subdomain of one level on the device.
struct DevLevel {
  int32_t n = 0, n_own = 0;
  int64_t offset = 0;  // position of this subdomain inside the level's vectors
  int n_colors = 0;
  std::vector<int32_t> color_start;  // device rows, n_colors + 1 (own rows only)
  RowMap rmap{};                     // block schedule of the full-level Jacobi / residual passes
  unsigned rmap_grid = 0;            // their grid under rmap
  std::vector<int32_t> perm;         // host index -> device index
  DevBuf<int32_t> d_perm;
  DevSell A;
  DevWin W;  // block windows of A's own rows (Options::win)
  // host copies to place further value sets on A's pattern (pf_operator_set_values)
  std::vector<int64_t> csr_rowptr;   // the level desc's row offsets (host order)
  std::vector<int64_t> sell_ptr;     // A.slice_ptr
  DevBuf<uint8_t> d_is_dir;
  int64_t own_cols_touched = 0;  // distinct columns referenced by own rows
  // prolongation from the parent level (rows: this level's device rows; columns: parent
  // device rows of the same subdomain), SELL-32 like the operator
  DevSell P;
  // restriction to the parent level (rows: parent device rows; columns: this level's
  // device rows), entries in ascending fine host index
  DevSell R;
  // multi-process fused exchanges: own rows whose values are sent (boundary), as a list and
  // as a per-row mask (the interior sweep skips them)
  DevBuf<int32_t> brows;
  DevBuf<uint8_t> is_brow;
  int32_t n_brows = 0;
  // ... and for the coloured smoothers: the rows of the LAST colour that must run before the
  // exchange (boundary rows, and rows reading a non-own copy the exchange rewrites), as a
  // list and a mask; every other row of that colour runs concurrently with the exchange
  DevBuf<int32_t> cpre;
  DevBuf<uint8_t> is_cpre;
  int32_t n_cpre = -1;  // -1: not built
  std::vector<uint8_t> reads_nonown;  // host, multi-process finalize only: own row (device order) reads a copy
  // residual-norm scratch
  int resnorm_blocks = 0;
  DevBuf<double> partials;
  DevBuf<unsigned int> ticket;
};

struct PeerSeg {
  int peer = 0;
  int64_t off = 0, len = 0;
};

// One exchange (scatter of one channel kind, or the master/slave accumulate) on one
// level.  Indices are level-global device indices (subdomain offset included).
struct ExchangePlan {
  int64_t n = 0;  // entries moved
  // local transport (all peers on this device): v[dst[i]] = v[src[i]]
  DevBuf<int32_t> dst, src;
  // accumulate: per master m: v[acc_dst[m]] += sum over acc_src[acc_off[m]..acc_off[m+1])
  int32_t n_masters = 0;
  DevBuf<int32_t> acc_off, acc_src, acc_dst;
  // remote transport (NCCL; one subdomain per process)
  DevBuf<int32_t> pack_idx, unpack_idx;
  std::vector<PeerSeg> send_segs, recv_segs;
  DevBuf<double> sendbuf, recvbuf;
  int peer_id = -1;  // index among the hierarchy's remote plans (PeerTransport)
};

struct Level {
  std::vector<HostLevel> host;  // per local subdomain (freed after finalize)
  std::vector<DevLevel> sub;    // per local subdomain
  int64_t total = 0;            // sum of subdomain sizes
  std::array<ExchangePlan, PF_NUM_CHANNEL_KINDS> scatter;
  ExchangePlan accumulate;
  ExchangePlan fused_ms_h1, fused_all;  // pf_hierarchy_set_fused_exchanges
  DevBuf<double> r;             // residual scratch
  DevBuf<double> sumsq;         // per-subdomain sums of squares
  DevBuf<double> norm;          // allreduced norm
  DevBuf<double> coarse_stats;  // [iterations, converged, r0, final]
  DevBuf<CoarseSub> coarse_subs;  // level 0 only
  // level 0 packed for the shared-memory coarse solve (k_coarse_smem / k_bottom)
  DevBuf<int32_t> cp_sub_rows, cp_rowptr, cp_rowdev, cp_cols;
  DevBuf<double> cp_vals;
  CoarsePack cpack{};
  pf_vector* x = nullptr;       // MultigridLevel::x, b (cycle scratch)
  pf_vector* b = nullptr;
};

struct Transport;  // pf_nccl.hpp

}  // namespace pf

struct pf_setup;
namespace pf {
void adopt_setup_level(pf_setup* s, int level, HostLevel& H);  // pf_setup.cpp
}  // namespace pf

namespace pf {
// Ids of a hierarchy's live vectors: cached graphs are keyed by vector id (never by
// address, which the allocator reuses) and are dropped once a vector they use is gone.
struct VecRegistry {
  std::mutex mu;
  std::unordered_set<uint64_t> live;
  bool alive(uint64_t id) {
    std::lock_guard<std::mutex> g(mu);
    return live.count(id) != 0;
  }
};
}  // namespace pf

struct pf_vector {
  pf_hierarchy* h = nullptr;
  int device = 0;  // kept here so destruction never reads the hierarchy
  int level = 0;
  uint64_t uid = 0;                        // unique for the process lifetime
  std::weak_ptr<pf::VecRegistry> registry;  // the hierarchy's (expired once it is destroyed)
  pf::DevBuf<double> data;  // [2 * total]: primary then Jacobi ping-pong partner
  double* cur() const { return data.p; }
  double* alt() const { return data.p + total; }
  int64_t total = 0;
};

namespace pf {
// Tuning options of one hierarchy (DESIGN.md §6 "Knobs").  Each starts at its measured-best
// default, is overridden by the PF_* environment variable of the same name (upper case)
// when the hierarchy is created, and can then be set with pf_hierarchy_set_option.  Build
// options shape the device layout and are fixed by pf_hierarchy_finalize; launch options
// steer the enqueue (a change drops the cached graphs).
struct Options {
  // build
  int64_t value_index = 1;            // index-encode operator values (8/16-bit)
  // smallest operator (stored entries) encoded; measured at C2: encoding only the >= 2M-entry
  // operators, Jacobi solve 6.08 ms; all of them, 5.86 ms (the smaller levels' operators take
  // less L2 space and fewer L1 requests too)
  int64_t value_index_min = 0;
  int64_t vtab_smem = 1;              // 8-bit value table staged in shared memory (0: through L1)
  // operators of the levels below the finest up to this size (about 40 % of the 126 MB L2)
  // are read with the caching load policy and stay L2-resident across a cycle's sweeps; the
  // finest level, and larger ones, stream evict-first
  int64_t cached_max_bytes = int64_t(48) << 20;
  // levels whose x is at least this large run their full-level Jacobi / residual passes with
  // the colour-interleaved block schedule (0: every level with 2-8 colours)
  int64_t interleave_min_bytes = int64_t(64) << 20;
  int64_t bottom_rows = 1024;         // bottom kernel: levels up to this many rows
  int64_t bottom_block_rows = 1024;   // ... of which block 0 runs those up to this many rows
  int64_t bottom_grid = 0;            // bottom kernel grid (0: automatic)
  int64_t bottom_stage = 1;           // stage the block levels in shared memory
  int64_t rep_bottom_rows = 65536;    // multi-process replicated bottom levels
  // launch
  int64_t bottom_jacobi = 0;          // damped Jacobi through the bottom kernel too
  int64_t bottom_block_kernel = 1;    // fully staged bottom as the one-block kernel
  int64_t split_row_len = 48;         // slice-split colour sweep for rows longer than this
  int64_t split_max_rows = int64_t(1) << 20;  // ... on levels up to this many own rows
  int64_t split_rows_max = 65536;     // slice-split Jacobi / residual for long rows up to this many rows
  int64_t wide_max_rows = -1;         // wide-row kernels for launches up to this many rows (-1: one wave)
  int64_t fused_rr_rows = 8192;       // residual + restriction in one launch up to this many rows
  int64_t sor_tma = 0, sor_tma_min_rows = 65536, sor_tma_bps = 2, sor_tma_cfg = 0;  // opt-in TMA colour sweep
  // opt-in (measured slower, profiles/r02_sweep_experiments.md): block windows (pf_window.cuh)
  // for the own rows of levels with at least win_min_rows rows; a block's cover fits
  // win_max_chunks chunks of 16 doubles or the block takes the plain path
  int64_t win = 0, win_min_rows = 100000, win_max_chunks = kWinChunksCap;
  // launch: window kernels where a level has windows (1: Jacobi / residual / norm, 2: the
  // colour sweeps too)
  int64_t win_kernels = 1;
  int64_t solve_graph_if = 0;         // device solve graph with an IF node inside the WHILE body (the older shape)
  int64_t pdl = 1;                    // programmatic dependent launch
  int64_t solve_mode_host = 0;        // host-driven outer loop instead of the device WHILE graph
};
}  // namespace pf

struct pf_hierarchy {
  int device = 0;
  pf::Options opt;
  int n_levels = 0, n_sub = 1, rank_base = 0, world = 1;
  bool finalized = false;
  bool fused = false;  // master/slave + halo scatters as one message group (direct halo lists)
  bool colorwise = false;  // coloured smoothers exchange after every colour (pf_hierarchy_set_colorwise_exchange)
  pf::DevBuf<double> coarse_inv;  // pf_hierarchy_set_coarse_direct: inverse of level 0's own block
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaStream_t comm_stream = nullptr;  // exchanges overlapped with interior sweeps
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::vector<pf::Level> levels;
  pf::DevBuf<double> staging;  // host-order staging for uploads/downloads
  double* pinned = nullptr;    // pinned host slots for scalars read back each cycle
  int64_t launches = 0;
  std::unique_ptr<pf::Transport> xport;  // multi-process exchanges (NCCL or loopback)
  // graph cache of one outer cycle (cycles x V-cycle + finest residual norm)
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    int64_t kernels = 0;       // kernels per replay (solve graph: per executed IF body)
    int64_t head_kernels = 0;  // solve graph: kernels per WHILE iteration head
    void* state = nullptr;      // solve graph: device SolveState
    void* host_state = nullptr; // pinned copy written at the end of the graph
    size_t state_bytes = 0;
    uint64_t x_uid = 0, b_uid = 0;  // the vectors the graph reads and writes
  };
  std::shared_ptr<pf::VecRegistry> vectors = std::make_shared<pf::VecRegistry>();
  std::map<std::string, GraphEntry> graphs;
  // Levels 0..top of the V-cycle run in one cooperative kernel (pf_bottom.cuh).
  struct Bottom {
    bool active = false;
    bool staged_all = false;  // levels 0..top all staged in block 0's shared memory
    int top = -1;
    int grid = 0;
    size_t smem = 0;       // dynamic shared memory: descriptor copy + coarse pack
    void* desc = nullptr;  // device BotDesc
    void* stamps = nullptr;  // PF_BOTTOM_PROFILE phase timestamps
    std::vector<pf::DevBuf<int32_t>> color_bufs;
    std::vector<pf::DevBuf<double>> val_bufs;  // fp64 copies of index-encoded operators
    pf::DevBuf<unsigned char> stage_blob;       // the staged block levels (BotStage)
    Bottom() = default;
    Bottom(const Bottom&) = delete;
    Bottom& operator=(const Bottom&) = delete;
    ~Bottom() {
      if (desc) cudaFree(desc);
      if (stamps) cudaFree(stamps);
    }
  } bot;
  // Multi-process runs: the bottom levels 0..top of EVERY rank, replicated on each GPU.
  // One allgather of the restricted residual feeds a redundant bottom V-cycle (or, with
  // only level 0 replicated, the coarse solve), instead of the per-sweep and
  // per-coarse-iteration exchanges the reference does on those latency-bound levels.
  struct RepLevel {
    std::vector<pf::HostLevel> host;  // per world rank
    std::vector<pf::DevLevel> sub;
    int64_t stride = 0;               // rank r's entries at [r * stride, r * stride + n_r)
    std::array<pf::ExchangePlan, PF_NUM_CHANNEL_KINDS> scatter;
    pf::ExchangePlan acc;
    pf::DevBuf<double> x, b, r;       // x holds [2 * world * stride] (Jacobi ping-pong)
  };
  struct Replica {
    bool active = false;
    std::vector<RepLevel> lv;         // levels 0..top
    pf::DevBuf<pf::CoarseSub> subs;   // level 0, sequential coarse solve fallback
    pf::DevBuf<int32_t> cp_sub_rows, cp_rowptr, cp_rowdev, cp_cols;
    pf::DevBuf<double> cp_vals;
    pf::CoarsePack cpack{};
    pf::DevBuf<double> send;          // max stride
    pf::DevBuf<double> coarse_stats;
    Bottom bot;                       // bottom kernel over the replicated levels
  } rep;
  ~pf_hierarchy();
};
