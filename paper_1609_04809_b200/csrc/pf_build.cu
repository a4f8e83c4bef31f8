// pf_build.cu — host level data (pf_level_desc, the product setup) -> the device layout of
// the GMG V-cycle: SELL-32x4 operators with lossless value-index tables, device row
// placement (colour-major, lattice order inside a colour), R = P^T as a gather, the
// exchange plans of ParFECommunicator (fecomm.cpp:25-72), the coarse pack of the coarse
// solve, the replicated bottom levels of multi-process runs, and the bottom kernel's
// descriptor with its shared-memory staging (pf_bottom_types.hpp).
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <omp.h>
#include <parallel/algorithm>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "pf_internal.hpp"

using namespace pf;

namespace pf {
namespace rt {



// Stored values (SELL order, padding included) -> device: an 8/16-bit index into the table
// of distinct values (distinguished by bit pattern, so -0.0 and 0.0 stay apart) when there
// are at most 65,536 of them, else fp64.
void encode_values(const std::vector<double>& sv, DevVals& out, const Options& o) {
  out = DevVals{};
  if (o.value_index && !sv.empty() && static_cast<int64_t>(sv.size()) >= o.value_index_min) {
    // pass 1: the distinct values in first-seen order, giving up past 65,536.  Each chunk
    // collects its own first-seen list; merging the lists in chunk order gives the
    // sequential first-seen order.
    const int64_t n = static_cast<int64_t>(sv.size());
    const int nchunk = std::max(1, std::min<int>(omp_get_max_threads(), static_cast<int>(n / (1 << 20)) + 1));
    std::vector<std::vector<uint64_t>> firsts(static_cast<size_t>(nchunk));
    std::vector<int> overflow(static_cast<size_t>(nchunk), 0);
#pragma omp parallel for schedule(static, 1)
    for (int c = 0; c < nchunk; ++c) {
      std::unordered_set<uint64_t> seen;
      const int64_t lo = n * c / nchunk, hi = n * (c + 1) / nchunk;
      for (int64_t i = lo; i < hi; ++i) {
        uint64_t bits;
        std::memcpy(&bits, &sv[static_cast<size_t>(i)], sizeof bits);
        if (seen.insert(bits).second) {
          firsts[static_cast<size_t>(c)].push_back(bits);
          if (seen.size() > 65536) {
            overflow[static_cast<size_t>(c)] = 1;
            break;
          }
        }
      }
    }
    std::unordered_map<uint64_t, uint32_t> ids;
    std::vector<double> table;
    bool fits = std::find(overflow.begin(), overflow.end(), 1) == overflow.end();
    for (int c = 0; c < nchunk && fits; ++c)
      for (uint64_t bits : firsts[static_cast<size_t>(c)]) {
        if (ids.find(bits) != ids.end()) continue;
        if (table.size() == 65536) {
          fits = false;
          break;
        }
        ids.emplace(bits, static_cast<uint32_t>(table.size()));
        double v;
        std::memcpy(&v, &bits, sizeof v);
        table.push_back(v);
      }
    if (fits) {  // pass 2: the indices
      out.table.upload(table);
      if (table.size() <= 256) {
        out.vkind = 1;
        std::vector<uint8_t> idx(sv.size());
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
          uint64_t bits;
          std::memcpy(&bits, &sv[static_cast<size_t>(i)], sizeof bits);
          idx[static_cast<size_t>(i)] = static_cast<uint8_t>(ids.find(bits)->second);
        }
        out.vi8.upload(idx);
      } else {
        out.vkind = 2;
        std::vector<uint16_t> idx(sv.size());
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
          uint64_t bits;
          std::memcpy(&bits, &sv[static_cast<size_t>(i)], sizeof bits);
          idx[static_cast<size_t>(i)] = static_cast<uint16_t>(ids.find(bits)->second);
        }
        out.vi16.upload(idx);
      }
      return;
    }
  }
  out.vkind = 0;
  out.vals.upload(sv);
}

void check_level(const pf_hierarchy* h, int level) {
  if (!h) invalid("null hierarchy");
  if (!h->finalized) state("hierarchy not finalized");
  if (level < 0 || level >= h->n_levels) invalid("level " + std::to_string(level) + " out of range");
}

void check_vec(const pf_hierarchy* h, const pf_vector* v, int level, const char* what) {
  if (!v) invalid(std::string(what) + ": null vector");
  if (v->h != h) invalid(std::string(what) + ": vector belongs to another hierarchy");
  if (v->level != level)
    invalid(std::string("vector length does not match mapper dof count (") + what + ": level " +
            std::to_string(v->level) + " vs " + std::to_string(level) + ")");
}

// ------------------------------------------------------------------ upload --

// SELL-32 from rows already in device order (entry order inside a row is preserved).
void sell_from_rows(int32_t n, const std::vector<int64_t>& off, const std::vector<int32_t>& col,
                    const std::vector<double>& val, DevSell& out, const Options& o) {
  const int64_t n_slices = (n + kSlice - 1) / kSlice;
  std::vector<int64_t> sptr(static_cast<size_t>(n_slices) + 1, 0);
  std::vector<int32_t> rlen(static_cast<size_t>(std::max<int64_t>(n_slices, 1) * kSlice), 0);
  for (int32_t d = 0; d < n; ++d) rlen[d] = static_cast<int32_t>(off[d + 1] - off[d]);
  for (int64_t s = 0; s < n_slices; ++s) {
    int32_t w = 0;
    for (int l = 0; l < kSlice; ++l) w = std::max(w, rlen[s * kSlice + l]);
    w = (w + kGroup - 1) / kGroup * kGroup;  // SELL-32x4: whole groups of 4
    sptr[s + 1] = sptr[s] + static_cast<int64_t>(w) * kSlice;
  }
  std::vector<double> sv(static_cast<size_t>(sptr[n_slices]), 0.0);
  std::vector<int32_t> sc(static_cast<size_t>(sptr[n_slices]), 0);
#pragma omp parallel for schedule(static)
  for (int64_t s = 0; s < n_slices; ++s) {
    const int64_t w = (sptr[s + 1] - sptr[s]) / kSlice;
    for (int l = 0; l < kSlice; ++l) {
      const int64_t d = s * kSlice + l;
      const int32_t len = d < n ? rlen[d] : 0;
      for (int64_t j = 0; j < w; ++j) {
        const int64_t e = sell_entry(sptr[s] + static_cast<int64_t>(l) * kGroup, static_cast<int>(j));
        if (j < len) {
          sc[e] = col[off[d] + j];
          sv[e] = val[off[d] + j];
        } else {  // padding, never read (row_len bounds every loop)
          sc[e] = 0;
          sv[e] = 0.0;
        }
      }
    }
  }
  out.slice_ptr.upload(sptr);
  out.row_len.upload(rlen);
  out.max_len = rlen.empty() ? 0 : *std::max_element(rlen.begin(), rlen.end());
  encode_values(sv, out.vals, o);
  out.smem_table = o.vtab_smem != 0;
  out.cols.upload(sc);
  out.nnz = n > 0 ? off[n] : 0;
  out.stored = sptr[n_slices];
}

// SELL-32x4 of a host CSR whose device row d is host row inv[d] and whose columns map
// through perm; entry order inside a row preserved.
void sell_from_csr(int32_t n, const std::vector<int32_t>& inv, const std::vector<int32_t>& perm,
                   const std::vector<int64_t>& rowptr, const std::vector<int32_t>& cols,
                   const std::vector<double>& vals, DevSell& out,
                   const Options& o, std::vector<int32_t>* keep_cols = nullptr) {
  const int64_t n_slices = (n + kSlice - 1) / kSlice;
  std::vector<int64_t> sptr(static_cast<size_t>(n_slices) + 1, 0);
  std::vector<int32_t> rlen(static_cast<size_t>(std::max<int64_t>(n_slices, 1) * kSlice), 0);
#pragma omp parallel for schedule(static)
  for (int32_t d = 0; d < n; ++d) rlen[d] = static_cast<int32_t>(rowptr[inv[d] + 1] - rowptr[inv[d]]);
  for (int64_t s = 0; s < n_slices; ++s) {
    int32_t w = 0;
    for (int l = 0; l < kSlice; ++l) w = std::max(w, rlen[s * kSlice + l]);
    w = (w + kGroup - 1) / kGroup * kGroup;
    sptr[s + 1] = sptr[s] + static_cast<int64_t>(w) * kSlice;
  }
  // columns, then values, one host array at a time (peak host memory on large grids)
  {
    std::vector<int32_t> sc(static_cast<size_t>(sptr[n_slices]), 0);
#pragma omp parallel for schedule(static)
    for (int32_t d = 0; d < n; ++d) {
      const int64_t base = sell_row_base(sptr.data(), d), k0 = rowptr[inv[d]];
      for (int j = 0; j < rlen[d]; ++j) sc[static_cast<size_t>(sell_entry(base, j))] = perm[cols[static_cast<size_t>(k0 + j)]];
    }
    out.cols.upload(sc);
    if (keep_cols) keep_cols->swap(sc);
  }
  {
    std::vector<double> sv(static_cast<size_t>(sptr[n_slices]), 0.0);
#pragma omp parallel for schedule(static)
    for (int32_t d = 0; d < n; ++d) {
      const int64_t base = sell_row_base(sptr.data(), d), k0 = rowptr[inv[d]];
      for (int j = 0; j < rlen[d]; ++j) sv[static_cast<size_t>(sell_entry(base, j))] = vals[static_cast<size_t>(k0 + j)];
    }
    encode_values(sv, out.vals, o);
    out.smem_table = o.vtab_smem != 0;
  }
  out.slice_ptr.upload(sptr);
  out.row_len.upload(rlen);
  out.max_len = rlen.empty() ? 0 : *std::max_element(rlen.begin(), rlen.end());
  out.nnz = n > 0 ? rowptr[n] : 0;
  out.stored = sptr[n_slices];
}

// Block windows of the own rows (WinView, pf_types.hpp; kernels in pf_window.cuh).  For
// every block of kBlock device rows the off-diagonal columns its own rows read, ascending,
// are covered greedily by chunks of 16 doubles starting at a multiple of 4 (a 32-byte
// sector); the diagonal and padding entries of a row point at the row's private slot.  A
// block whose cover exceeds Options::win_max_chunks (at most kWinChunksCap: the launches'
// shared memory), or with a row holding several diagonal entries, keeps an empty cover and
// its rows take the plain path inside the window kernels; a level keeps its windows when
// at least 90 % of its blocks have one — the structured levels do (colour-major placement:
// a block's neighbours are a few lattice lines of each other colour); an operator without
// that locality keeps the plain kernels.
void build_window(DevLevel& D, const std::vector<int32_t>& sc, const std::vector<int64_t>& sptr, int level,
                  const Options& o) {
  D.W = DevWin{};
  const int32_t n = D.n, n_own = D.n_own;
  if (!o.win || n_own < o.win_min_rows || D.rmap.n_col != 0 || D.A.max_len > 255) return;
  const int64_t blocks = grid_for(n), own_blocks = grid_for(n_own);
  std::vector<int32_t> rlen(static_cast<size_t>(n_own));
  PF_CUDA(cudaMemcpy(rlen.data(), D.A.row_len.p, sizeof(int32_t) * rlen.size(), cudaMemcpyDeviceToHost));
  std::vector<std::vector<int32_t>> cover(static_cast<size_t>(own_blocks));
  std::vector<uint16_t> c16(sc.size(), 0);
  std::vector<uint8_t> dpos(static_cast<size_t>(n_own), 0);
  const int64_t cap = std::min<int64_t>(o.win_max_chunks, kWinChunksCap);
  int64_t plain = 0;
#pragma omp parallel
  {
    std::vector<int32_t> cs, slot;
#pragma omp for schedule(dynamic, 16) reduction(+ : plain)
    for (int64_t bk = 0; bk < own_blocks; ++bk) {
      const int32_t r0 = static_cast<int32_t>(bk * kBlock), r1 = std::min<int64_t>(n_own, r0 + kBlock);
      cs.clear();
      bool ok = true;
      for (int32_t r = r0; r < r1; ++r) {
        const int64_t base = sell_row_base(sptr.data(), r);
        int diags = 0;
        for (int j = 0; j < rlen[r]; ++j) {
          const int32_t c = sc[static_cast<size_t>(sell_entry(base, j))];
          if (c == r) {
            dpos[r] = static_cast<uint8_t>(j);
            ++diags;
          } else {
            cs.push_back(c);
          }
        }
        ok = ok && diags == 1;
      }
      std::sort(cs.begin(), cs.end());
      cs.erase(std::unique(cs.begin(), cs.end()), cs.end());
      std::vector<int32_t>& ch = cover[static_cast<size_t>(bk)];
      slot.resize(cs.size());
      int32_t start = -kWinChunk;
      for (size_t i = 0; i < cs.size(); ++i) {
        if (cs[i] >= start + kWinChunk) {
          start = cs[i] & ~3;
          ch.push_back(start);
        }
        slot[i] = kBlock + static_cast<int32_t>(ch.size() - 1) * kWinChunk + (cs[i] - start);
      }
      if (!ok || ch.empty() || static_cast<int64_t>(ch.size()) > cap) {  // this block takes the plain row path
        ch.clear();
        ++plain;
        continue;
      }
      for (int32_t r = r0; r < r1; ++r) {
        const int64_t base = sell_row_base(sptr.data(), r);
        const int padded = (rlen[r] + kGroup - 1) / kGroup * kGroup;
        for (int j = 0; j < padded; ++j) {
          const size_t e = static_cast<size_t>(sell_entry(base, j));
          const int32_t c = j < rlen[r] ? sc[e] : r;
          const int32_t sl = c == r ? r - r0 : slot[std::lower_bound(cs.begin(), cs.end(), c) - cs.begin()];
          c16[e] = static_cast<uint16_t>(sl * 8);
        }
      }
    }
  }
  int64_t total = 0;
  size_t most = 0;
  for (const auto& ch : cover) {
    total += static_cast<int64_t>(ch.size());
    most = std::max(most, ch.size());
  }
  // windows pay when nearly every block has one
  const bool keep = 10 * plain <= own_blocks && total <= INT32_MAX;
  if (std::getenv("PF_TIMING"))
    std::fprintf(stderr, "[pf_window] level %d: %lld row blocks, %lld without a window, chunks per block mean %.1f max %zu%s\n",
                 level, static_cast<long long>(own_blocks), static_cast<long long>(plain),
                 own_blocks > plain ? double(total) / (own_blocks - plain) : 0.0, most, keep ? "" : " (plain kernels)");
  if (!keep) return;
  std::vector<int32_t> ptr(static_cast<size_t>(blocks) + 1, 0), flat;
  flat.reserve(static_cast<size_t>(total));
  for (int64_t bk = 0; bk < blocks; ++bk) {
    if (bk < own_blocks) flat.insert(flat.end(), cover[bk].begin(), cover[bk].end());
    ptr[static_cast<size_t>(bk) + 1] = static_cast<int32_t>(flat.size());
  }
  D.W.cols16.upload(c16);
  D.W.chunk_ptr.upload(ptr);
  D.W.chunks.upload(flat);
  D.W.dpos.upload(dpos);
  D.W.max_chunks = static_cast<int32_t>(most);
  D.W.on = true;
}

// Device layout of one subdomain level: own rows colour-major (stable in host order),
// then every other row in host order; SELL-32x4 operator; P (rows of this level).
void build_dev_level(const HostLevel& H, DevLevel& D, int level, const Options& o) {
  PhaseTimer tm;
  const int32_t n = H.n, n_own = H.n_own;
  D.n = n;
  D.n_own = n_own;
  // --- diagonal check (check_diagonal, solvers.cpp:10-15) and column sanity
  for (int32_t r = 0; r < n; ++r) {
    if (H.rowptr[r + 1] < H.rowptr[r]) invalid("row offsets must be non-decreasing");
  }
  {
    const int64_t nnz = H.rowptr[n];
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t k = 0; k < nnz; ++k) bad |= (H.cols[k] < 0 || H.cols[k] >= n) ? 1 : 0;
    if (bad) invalid("column index out of range");
    int32_t first_zero = INT32_MAX;
#pragma omp parallel for schedule(static) reduction(min : first_zero)
    for (int32_t r = 0; r < n_own; ++r) {
      double diag = 0.0;
      for (int64_t k = H.rowptr[r]; k < H.rowptr[r + 1]; ++k)
        if (H.cols[k] == r) diag = H.vals[k];
      if (diag == 0.0) first_zero = std::min(first_zero, r);
    }
    if (first_zero != INT32_MAX)
      throw Error(PF_ERR_SINGULAR_DIAGONAL, "zero diagonal at own dof " + std::to_string(first_zero) +
                                                " (level " + std::to_string(level) + ")");
  }
  tm("checks", level);
  // --- colours of own rows
  std::vector<int32_t> color(static_cast<size_t>(n_own), 0);
  if (!H.color.empty()) {
    for (int32_t i = 0; i < n_own; ++i) {
      if (H.color[i] < 0) invalid("negative colour");
      color[i] = H.color[i];
    }
    // a colour class must be an independent set of the own-row graph
    int64_t first_bad = INT64_MAX;
#pragma omp parallel for schedule(static) reduction(min : first_bad)
    for (int32_t i = 0; i < n_own; ++i)
      for (int64_t k = H.rowptr[i]; k < H.rowptr[i + 1]; ++k) {
        const int32_t c = H.cols[k];
        if (c != i && c < n_own && color[c] == color[i] && H.vals[k] != 0.0) first_bad = std::min(first_bad, k);
      }
    if (first_bad != INT64_MAX) {
      const int32_t i = static_cast<int32_t>(std::upper_bound(H.rowptr.begin(), H.rowptr.end(), first_bad) - H.rowptr.begin() - 1);
      invalid("colouring couples rows " + std::to_string(i) + " and " + std::to_string(H.cols[first_bad]));
    }
  } else {
    std::vector<int32_t> seen;
    for (int32_t i = 0; i < n_own; ++i) {
      seen.clear();
      for (int64_t k = H.rowptr[i]; k < H.rowptr[i + 1]; ++k) {
        const int32_t c = H.cols[k];
        if (c < i) seen.push_back(color[c]);
      }
      std::sort(seen.begin(), seen.end());
      int32_t pick = 0;
      for (int32_t s : seen) {
        if (s == pick) ++pick;
        else if (s > pick) break;
      }
      color[i] = pick;
    }
  }
  int32_t n_colors = 0;
  for (int32_t c : color) n_colors = std::max(n_colors, c + 1);
  D.n_colors = n_colors;
  D.color_start.assign(static_cast<size_t>(n_colors) + 1, 0);
  for (int32_t c : color) ++D.color_start[c + 1];
  for (int32_t c = 0; c < n_colors; ++c) D.color_start[c + 1] += D.color_start[c];
  // --- permutation host -> device
  D.perm.assign(static_cast<size_t>(n), 0);
  std::vector<int32_t> inv(static_cast<size_t>(n), 0);
  {
    std::vector<int32_t> next(D.color_start.begin(), D.color_start.end() - 1);
    if (H.order.empty()) {
      for (int32_t i = 0; i < n_own; ++i) D.perm[i] = next[color[i]]++;
    } else {  // placement hint: inside a colour, ascending (order, host index)
      std::vector<int32_t> own(static_cast<size_t>(n_own));
      std::iota(own.begin(), own.end(), 0);
      // (colour, order, index) is a strict total order, so any sort gives the stable result
      __gnu_parallel::sort(own.begin(), own.end(), [&](int32_t a, int32_t b) {
        if (color[a] != color[b]) return color[a] < color[b];
        if (H.order[a] != H.order[b]) return H.order[a] < H.order[b];
        return a < b;
      });
      for (int32_t i : own) D.perm[i] = next[color[i]]++;
    }
    for (int32_t i = n_own; i < n; ++i) D.perm[i] = i;
#pragma omp parallel for schedule(static)
    for (int32_t i = 0; i < n; ++i) inv[D.perm[i]] = i;
  }
  D.d_perm.upload(D.perm);
  // colour-interleaved block schedule when x outgrows L2 (RowMap, pf_types.hpp)
  D.rmap = RowMap{};
  D.rmap_grid = grid_for(n);
  if (n_colors >= 2 && n_colors <= 8 && 8 * static_cast<int64_t>(n) >= o.interleave_min_bytes) {
    int32_t chunks = 0;
    for (int c = 0; c < n_colors; ++c)
      chunks = std::max<int32_t>(chunks, static_cast<int32_t>(grid_for(D.color_start[c + 1] - D.color_start[c])));
    D.rmap.n_col = n_colors;
    D.rmap.chunks = chunks;
    for (int c = 0; c <= n_colors; ++c) D.rmap.start[c] = D.color_start[c];
    D.rmap_grid = static_cast<unsigned>(chunks) * n_colors + grid_for(n - n_own);
  }
  tm("colours + perm", level);
  // --- SELL-32x4 operator: rows in device order, columns mapped, entries in CSR order,
  // written straight from the host CSR (no intermediate re-layout: at 512^3 the finest
  // level alone is 44 GB of host CSR)
  const bool want_win = o.win && n_own >= o.win_min_rows && D.rmap.n_col == 0;
  std::vector<int32_t> dev_cols;
  sell_from_csr(n, inv, D.perm, H.rowptr, H.cols, H.vals, D.A, o, want_win ? &dev_cols : nullptr);
  D.A.own_nnz = H.rowptr[n_own];
  tm("sell", level);
  D.csr_rowptr = H.rowptr;
  D.sell_ptr.resize(static_cast<size_t>(D.A.slice_ptr.n));
  if (D.A.slice_ptr.n > 0)
    PF_CUDA(cudaMemcpy(D.sell_ptr.data(), D.A.slice_ptr.p, sizeof(int64_t) * D.sell_ptr.size(),
                       cudaMemcpyDeviceToHost));
  if (want_win) {
    build_window(D, dev_cols, D.sell_ptr, level, o);
    std::vector<int32_t>().swap(dev_cols);
    tm("windows", level);
  }
  {
    std::vector<uint8_t> touched(static_cast<size_t>(n), 0);
    const int64_t z = H.rowptr[n_own];
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < z; ++k) __atomic_store_n(&touched[static_cast<size_t>(H.cols[k])], 1, __ATOMIC_RELAXED);
    D.own_cols_touched = std::count(touched.begin(), touched.end(), 1);
  }
  // --- Dirichlet mask in device order
  std::vector<uint8_t> isdir(static_cast<size_t>(n), 0);
  for (int32_t i = 0; i < n; ++i) isdir[D.perm[i]] = H.is_dir.empty() ? 0 : H.is_dir[i];
  D.d_is_dir.upload(isdir);
  // --- residual-norm scratch
  D.resnorm_blocks = std::max<int>(1, static_cast<int>(grid_for(n_own)));
  // partials serve k_resnorm (grid over own rows) and k_jacobi_norm (grid over all rows)
  D.partials.alloc(std::max<int64_t>(D.resnorm_blocks, grid_for(n)));
  D.ticket.alloc(1);
  PF_CUDA(cudaMemset(D.ticket.p, 0, sizeof(unsigned int)));
  tm("touched + masks", level);
}

// P rows of the fine level in device order; R = P^T over owns_row fine rows as a
// parent-row gather with entries in ascending fine host index.
void build_transfer(const HostLevel& F, DevLevel& DF, const HostLevel& Cc, const DevLevel& DC, const Options& o) {
  const int32_t nf = F.n, nc = Cc.n;
  if (F.p_off.size() != static_cast<size_t>(nf) + 1) invalid("prolongation needs n_dofs + 1 offsets");
  for (int64_t e = 0; e < F.p_off[nf]; ++e)
    if (F.p_col[e] < 0 || F.p_col[e] >= nc) invalid("prolongation column out of the parent level");
  std::vector<int32_t> inv_f(static_cast<size_t>(nf));
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < nf; ++i) inv_f[DF.perm[i]] = i;
  std::vector<int64_t> poff(static_cast<size_t>(nf) + 1, 0);
  for (int32_t d = 0; d < nf; ++d) poff[d + 1] = poff[d] + (F.p_off[inv_f[d] + 1] - F.p_off[inv_f[d]]);
  std::vector<int32_t> pcol(static_cast<size_t>(poff[nf]));
  std::vector<double> pw(static_cast<size_t>(poff[nf]));
#pragma omp parallel for schedule(static)
  for (int32_t d = 0; d < nf; ++d) {
    const int32_t hr = inv_f[d];
    int64_t q = poff[d];
    for (int64_t e = F.p_off[hr]; e < F.p_off[hr + 1]; ++e, ++q) {
      pcol[static_cast<size_t>(q)] = DC.perm[F.p_col[e]];
      pw[static_cast<size_t>(q)] = F.p_w[e];
    }
  }
  sell_from_rows(nf, poff, pcol, pw, DF.P, o);
  // R rows: each parent row's contributions in ascending fine host index (the reference's
  // scatter-add order).  The owned P entries in fine host order, sorted by (parent device
  // row, position) — a strict order, so the parallel sort reproduces the counting sort.
  std::vector<int64_t> src;      // positions e of owned entries, ascending (= fine host order)
  std::vector<int32_t> fine_of;  // their fine host rows
  {
    std::vector<int64_t> cnt(static_cast<size_t>(nf) + 1, 0);
#pragma omp parallel for schedule(static)
    for (int32_t f = 0; f < nf; ++f) cnt[f + 1] = F.owns_row[f] ? F.p_off[f + 1] - F.p_off[f] : 0;
    for (int32_t f = 0; f < nf; ++f) cnt[f + 1] += cnt[f];
    src.resize(static_cast<size_t>(cnt[nf]));
    fine_of.resize(static_cast<size_t>(cnt[nf]));
#pragma omp parallel for schedule(static)
    for (int32_t f = 0; f < nf; ++f)
      if (F.owns_row[f])
        for (int64_t e = F.p_off[f], q = cnt[f]; e < F.p_off[f + 1]; ++e, ++q) {
          src[static_cast<size_t>(q)] = e;
          fine_of[static_cast<size_t>(q)] = f;
        }
  }
  // keys (parent device row << 35 | position): distinct, so sorting them is the stable sort
  std::vector<uint64_t> key(src.size());
  if (static_cast<int64_t>(src.size()) >= (int64_t(1) << 35)) invalid("prolongation too large");
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < static_cast<int64_t>(src.size()); ++q)
    key[static_cast<size_t>(q)] = static_cast<uint64_t>(DC.perm[F.p_col[src[static_cast<size_t>(q)]]]) << 35 |
                                  static_cast<uint64_t>(q);
  __gnu_parallel::sort(key.begin(), key.end());
  std::vector<int64_t> ord(src.size());
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < static_cast<int64_t>(key.size()); ++i)
    ord[static_cast<size_t>(i)] = static_cast<int64_t>(key[static_cast<size_t>(i)] & ((uint64_t(1) << 35) - 1));
  std::vector<uint64_t>().swap(key);
  std::vector<int64_t> roff(static_cast<size_t>(nc) + 1, 0);
  std::vector<int32_t> rcol(ord.size());
  std::vector<double> rwt(ord.size());
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < static_cast<int64_t>(ord.size()); ++i) {
    const int64_t q = ord[static_cast<size_t>(i)], e = src[static_cast<size_t>(q)];
    rcol[static_cast<size_t>(i)] = DF.perm[fine_of[static_cast<size_t>(q)]];
    rwt[static_cast<size_t>(i)] = F.p_w[e];
  }
  for (int64_t i = 0; i < static_cast<int64_t>(ord.size()); ++i)
    ++roff[static_cast<size_t>(DC.perm[F.p_col[src[static_cast<size_t>(ord[static_cast<size_t>(i)])]]]) + 1];
  for (int32_t c = 0; c < nc; ++c) roff[c + 1] += roff[c];
  sell_from_rows(nc, roff, rcol, rwt, DF.R, o);
}

const HostChannel* find_channel(const HostLevel& H, int kind, int peer) {
  for (const HostChannel& c : H.channels)
    if (c.kind == kind && c.peer == peer) return &c;
  return nullptr;
}

// Exchange plans of one level from the per-subdomain channel lists.  local: every peer
// is one of the subdomains in H (ranks rank_base + s); else one subdomain whose peers
// live in other processes (NCCL segments).
// One scatter plan over a set of channel kinds (several kinds: one message group; their
// send and receive sets must be independent — see build_fused_plans).
void build_scatter_plan(const std::vector<HostLevel>& H, const std::vector<DevLevel>& D, int rank_base, bool local,
                        const std::vector<int>& kinds, ExchangePlan& P) {
  const int n_sub = static_cast<int>(H.size());
  {
    auto in = [&](int k) { return std::find(kinds.begin(), kinds.end(), k) != kinds.end(); };
    if (local) {
      std::vector<int32_t> dst, src;
      for (int s = 0; s < n_sub; ++s) {
        const int R = rank_base + s;
        for (const HostChannel& c : H[s].channels) {
          if (!in(c.kind) || c.recv.empty()) continue;
          const int kind = c.kind;
          const int p = c.peer - rank_base;
          if (p < 0 || p >= n_sub || p == s) invalid("channel peer " + std::to_string(c.peer) + " out of range");
          const HostChannel* pc = find_channel(H[p], kind, R);
          if (!pc || pc->send.size() != c.recv.size())
            throw Error(PF_ERR_TRANSPORT, "channel lists of kind " + std::to_string(kind) +
                                              " between ranks " + std::to_string(c.peer) + " and " +
                                              std::to_string(R) + " do not pair up");
          for (size_t i = 0; i < c.recv.size(); ++i) {
            dst.push_back(static_cast<int32_t>(D[s].offset + D[s].perm[c.recv[i]]));
            src.push_back(static_cast<int32_t>(D[p].offset + D[p].perm[pc->send[i]]));
          }
        }
      }
      P.n = static_cast<int64_t>(dst.size());
      P.dst.upload(dst);
      P.src.upload(src);
    } else {
      const DevLevel& D0 = D[0];
      std::vector<int32_t> pk, up;
      for (const HostChannel& c : H[0].channels) {
        if (!in(c.kind)) continue;
        if (!c.send.empty()) {
          P.send_segs.push_back({c.peer, static_cast<int64_t>(pk.size()), static_cast<int64_t>(c.send.size())});
          for (int32_t d : c.send) pk.push_back(D0.perm[d]);
        }
        if (!c.recv.empty()) {
          P.recv_segs.push_back({c.peer, static_cast<int64_t>(up.size()), static_cast<int64_t>(c.recv.size())});
          for (int32_t d : c.recv) up.push_back(D0.perm[d]);
        }
      }
      P.n = static_cast<int64_t>(up.size());
      P.pack_idx.upload(pk);
      P.unpack_idx.upload(up);
      P.sendbuf.alloc(static_cast<int64_t>(pk.size()));
      P.recvbuf.alloc(static_cast<int64_t>(up.size()));
    }
  }
}

void build_exchange(const std::vector<HostLevel>& H, const std::vector<DevLevel>& D, int rank_base,
                    bool local, std::array<ExchangePlan, PF_NUM_CHANNEL_KINDS>& scatter, ExchangePlan& A) {
  const int n_sub = static_cast<int>(H.size());
  for (int kind = 0; kind < PF_NUM_CHANNEL_KINDS; ++kind) build_scatter_plan(H, D, rank_base, local, {kind}, scatter[kind]);
  // master/slave accumulate: slaves push v[recv_dofs], masters add in ascending peer order
  std::map<int32_t, std::vector<int32_t>> contrib;  // master dst -> sources, peer-ascending
  if (local) {
    for (int s = 0; s < n_sub; ++s) {
      const int R = rank_base + s;
      std::vector<const HostChannel*> ms;
      for (const HostChannel& c : H[s].channels)
        if (c.kind == PF_CH_MASTER_SLAVE && !c.send.empty()) ms.push_back(&c);
      std::sort(ms.begin(), ms.end(), [](const HostChannel* a, const HostChannel* b) { return a->peer < b->peer; });
      for (const HostChannel* c : ms) {
        const int p = c->peer - rank_base;
        const HostChannel* pc = find_channel(H[p], PF_CH_MASTER_SLAVE, R);
        if (!pc || pc->recv.size() != c->send.size())
          throw Error(PF_ERR_TRANSPORT, "master/slave lists do not pair up");
        for (size_t i = 0; i < c->send.size(); ++i)
          contrib[static_cast<int32_t>(D[s].offset + D[s].perm[c->send[i]])].push_back(
              static_cast<int32_t>(D[p].offset + D[p].perm[pc->recv[i]]));
      }
    }
  } else {
    const DevLevel& D0 = D[0];
    std::vector<const HostChannel*> ms;
    for (const HostChannel& c : H[0].channels)
      if (c.kind == PF_CH_MASTER_SLAVE) ms.push_back(&c);
    std::sort(ms.begin(), ms.end(), [](const HostChannel* a, const HostChannel* b) { return a->peer < b->peer; });
    std::vector<int32_t> pk;
    int64_t rpos = 0;
    for (const HostChannel* c : ms) {
      if (!c->recv.empty()) {  // slave side: push partial sums to the master
        A.send_segs.push_back({c->peer, static_cast<int64_t>(pk.size()), static_cast<int64_t>(c->recv.size())});
        for (int32_t d : c->recv) pk.push_back(D0.perm[d]);
      }
      if (!c->send.empty()) {  // master side
        A.recv_segs.push_back({c->peer, rpos, static_cast<int64_t>(c->send.size())});
        for (size_t i = 0; i < c->send.size(); ++i)
          contrib[D0.perm[c->send[i]]].push_back(static_cast<int32_t>(rpos + static_cast<int64_t>(i)));
        rpos += static_cast<int64_t>(c->send.size());
      }
    }
    A.pack_idx.upload(pk);
    A.sendbuf.alloc(static_cast<int64_t>(pk.size()));
    A.recvbuf.alloc(rpos);
  }
  std::vector<int32_t> off{0}, srcs, dsts;
  for (const auto& [d, list] : contrib) {
    dsts.push_back(d);
    srcs.insert(srcs.end(), list.begin(), list.end());
    off.push_back(static_cast<int32_t>(srcs.size()));
  }
  A.n_masters = static_cast<int32_t>(dsts.size());
  A.n = static_cast<int64_t>(srcs.size());
  A.acc_off.upload(off);
  A.acc_src.upload(srcs);
  A.acc_dst.upload(dsts);
}

// Fused exchanges (pf_hierarchy_set_fused_exchanges): master/slave + halo1 as one message
// group per sweep, + halo2 after a smoothing phase.  Valid when no halo send entry is a
// master/slave receive entry of the same subdomain (the halo value would otherwise be the
// one the master/slave scatter is still delivering) — pf_setup's direct_halos lists.
void build_fused_plans(pf_hierarchy* h, int l) {
  Level& L = h->levels[l];
  for (const HostLevel& H : L.host) {
    std::vector<uint8_t> slave(static_cast<size_t>(H.n), 0);
    for (const HostChannel& c : H.channels)
      if (c.kind == PF_CH_MASTER_SLAVE)
        for (int32_t d : c.recv) slave[static_cast<size_t>(d)] = 1;
    for (const HostChannel& c : H.channels)
      if (c.kind != PF_CH_MASTER_SLAVE)
        for (int32_t d : c.send)
          if (slave[static_cast<size_t>(d)])
            invalid("fused exchanges need halo lists that never forward a Slave-held value "
                    "(level " + std::to_string(l) + "): build them with direct_halos");
  }
  const bool local = h->world == h->n_sub;
  if (!local) {
    // multi-process: the own rows whose values leave this rank (master/slave and halo
    // sends) form the boundary set; a Jacobi sweep computes them first, starts the
    // exchange on the side stream, and sweeps the interior rows meanwhile
    const HostLevel& H = L.host[0];
    DevLevel& D = L.sub[0];
    std::vector<uint8_t> isb(static_cast<size_t>(D.n), 0);
    for (const HostChannel& c : H.channels)
      for (int32_t d : c.send)
        if (d < H.n_own) isb[static_cast<size_t>(D.perm[d])] = 1;
    std::vector<int32_t> list;
    for (int32_t r = 0; r < D.n_own; ++r)
      if (isb[static_cast<size_t>(r)]) list.push_back(r);
    D.n_brows = static_cast<int32_t>(list.size());
    D.brows.upload(list);
    D.is_brow.upload(isb);
    // coloured smoothers: the last colour's rows that send or read a non-own copy
    if (D.n_colors >= 1) {
      const int32_t c0 = D.color_start[D.n_colors - 1], c1 = D.color_start[D.n_colors];
      std::vector<uint8_t> pre(static_cast<size_t>(D.n), 0);
      for (int32_t r = c0; r < c1; ++r)
        pre[static_cast<size_t>(r)] = isb[static_cast<size_t>(r)] || D.reads_nonown[static_cast<size_t>(r)];
      std::vector<int32_t> pl;
      for (int32_t r = c0; r < c1; ++r)
        if (pre[static_cast<size_t>(r)]) pl.push_back(r);
      D.n_cpre = static_cast<int32_t>(pl.size());
      D.cpre.upload(pl);
      D.is_cpre.upload(pre);
    }
    std::vector<uint8_t>().swap(D.reads_nonown);
  }
  build_scatter_plan(L.host, L.sub, h->rank_base, local, {PF_CH_MASTER_SLAVE, PF_CH_HALO1}, L.fused_ms_h1);
  build_scatter_plan(L.host, L.sub, h->rank_base, local, {PF_CH_MASTER_SLAVE, PF_CH_HALO1, PF_CH_HALO2},
                     L.fused_all);
}

void build_plans(pf_hierarchy* h, int l) {
  Level& L = h->levels[l];
  build_exchange(L.host, L.sub, h->rank_base, h->world == h->n_sub, L.scatter, L.accumulate);
  if (h->fused) build_fused_plans(h, l);
}

// Pack a coarse level (all subdomains of H/D, level-global indices) for the shared-memory
// coarse solve: own rows per subdomain in host order, entries in stored order.
CoarsePack make_coarse_pack(const std::vector<HostLevel>& H, const std::vector<DevLevel>& D,
                            const std::array<ExchangePlan, PF_NUM_CHANNEL_KINDS>& plans,
                            DevBuf<int32_t>& sub_rows, DevBuf<int32_t>& rowptr, DevBuf<int32_t>& rowdev,
                            DevBuf<int32_t>& cols, DevBuf<double>& vals) {
  std::vector<int32_t> sr{0}, rp{0}, rd, cc;
  std::vector<double> vv;
  int64_t total = 0;
  for (size_t s = 0; s < H.size(); ++s) {
    const HostLevel& h = H[s];
    const DevLevel& d = D[s];
    for (int32_t i = 0; i < h.n_own; ++i) {
      rd.push_back(static_cast<int32_t>(d.offset + d.perm[i]));
      for (int64_t k = h.rowptr[i]; k < h.rowptr[i + 1]; ++k) {
        cc.push_back(static_cast<int32_t>(d.offset + d.perm[h.cols[k]]));
        vv.push_back(h.vals[k]);
      }
      rp.push_back(static_cast<int32_t>(cc.size()));
    }
    sr.push_back(static_cast<int32_t>(rd.size()));
    total = std::max<int64_t>(total, d.offset + d.n);
  }
  sub_rows.upload(sr);
  rowptr.upload(rp);
  rowdev.upload(rd);
  cols.upload(cc);
  vals.upload(vv);
  CoarsePack P{};
  P.n_total = static_cast<int32_t>(total);
  P.n_rows = static_cast<int32_t>(rd.size());
  P.nnz = static_cast<int32_t>(cc.size());
  P.n_sub = static_cast<int32_t>(H.size());
  P.sub_rows = sub_rows.p;
  P.rowptr = rowptr.p;
  P.rowdev = rowdev.p;
  P.cols = cols.p;
  P.vals = vals.p;
  P.ms_dst = plans[PF_CH_MASTER_SLAVE].dst.p;
  P.ms_src = plans[PF_CH_MASTER_SLAVE].src.p;
  P.ms_n = static_cast<int32_t>(plans[PF_CH_MASTER_SLAVE].n);
  P.h1_dst = plans[PF_CH_HALO1].dst.p;
  P.h1_src = plans[PF_CH_HALO1].src.p;
  P.h1_n = static_cast<int32_t>(plans[PF_CH_HALO1].n);
  P.max_row = 0;
  for (size_t i = 0; i + 1 < rp.size(); ++i) P.max_row = std::max(P.max_row, rp[i + 1] - rp[i]);
  return P;
}


HostLevel parse_desc(const pf_level_desc& dd, int me, int world, bool need_p) {
  const pf_level_desc* d = &dd;
  if (d->n_dofs < 0 || d->n_own_dofs < 0 || d->n_own_dofs > d->n_dofs) invalid("bad dof counts");
  if (!d->row_offsets || (d->n_dofs > 0 && (!d->owns_row))) invalid("missing level arrays");
  HostLevel H;
  H.set = true;
  H.n = d->n_dofs;
  H.n_own = d->n_own_dofs;
  const int64_t nnz = d->row_offsets[d->n_dofs];
  if (d->row_offsets[0] != 0 || nnz < 0) invalid("row offsets must start at 0");
  if (nnz > 0 && (!d->col_indices || !d->values)) invalid("missing matrix arrays");
  H.rowptr.assign(d->row_offsets, d->row_offsets + d->n_dofs + 1);
  H.cols.assign(d->col_indices, d->col_indices + nnz);
  H.vals.assign(d->values, d->values + nnz);
  H.owns_row.assign(d->owns_row, d->owns_row + d->n_dofs);
  if (d->is_dirichlet) H.is_dir.assign(d->is_dirichlet, d->is_dirichlet + d->n_dofs);
  else H.is_dir.assign(static_cast<size_t>(d->n_dofs), 0);
  if (d->color) H.color.assign(d->color, d->color + d->n_own_dofs);
  if (d->row_order) H.order.assign(d->row_order, d->row_order + d->n_dofs);
  for (int i = 0; i < d->n_channels; ++i) {
    const pf_channel_desc& c = d->channels[i];
    if (c.kind < 0 || c.kind >= PF_NUM_CHANNEL_KINDS) invalid("bad channel kind");
    if (c.peer < 0 || c.peer >= world || c.peer == me) invalid("bad channel peer");
    HostChannel hc;
    hc.kind = c.kind;
    hc.peer = c.peer;
    hc.send.assign(c.send_dofs, c.send_dofs + c.n_send);
    hc.recv.assign(c.recv_dofs, c.recv_dofs + c.n_recv);
    for (int32_t v : hc.send)
      if (v < 0 || v >= d->n_dofs) invalid("channel send dof out of range");
    for (int32_t v : hc.recv)
      if (v < 0 || v >= d->n_dofs) invalid("channel recv dof out of range");
    H.channels.push_back(std::move(hc));
  }
  std::sort(H.channels.begin(), H.channels.end(), [](const HostChannel& a, const HostChannel& b) {
    return a.kind != b.kind ? a.kind < b.kind : a.peer < b.peer;
  });
  if (need_p) {
    if (!d->p_offsets) invalid("level > 0 needs a prolongation map");
    H.p_off.assign(d->p_offsets, d->p_offsets + d->n_dofs + 1);
    const int64_t pn = H.p_off.back();
    H.p_col.assign(d->p_cols, d->p_cols + pn);
    H.p_w.assign(d->p_weights, d->p_weights + pn);
  }
  return H;
}

void build_replica(pf_hierarchy* h) {
  auto& R = h->rep;
  if (R.lv.empty() || R.lv[0].host.size() != static_cast<size_t>(h->world))
    state("multi-process hierarchy needs pf_hierarchy_set_coarse_replica for every rank");
  const int top = static_cast<int>(R.lv.size()) - 1;
  if (top >= h->n_levels) invalid("more replicated levels than the hierarchy has");
  int64_t max_stride = 1;
  for (int l = 0; l <= top; ++l) {
    auto& RL = R.lv[static_cast<size_t>(l)];
    if (RL.host.size() != static_cast<size_t>(h->world)) state("replica level " + std::to_string(l) + " incomplete");
    RL.sub.resize(static_cast<size_t>(h->world));
    int64_t stride = 1;
    for (int r = 0; r < h->world; ++r) {
      if (!RL.host[r].set)
        state("replica of rank " + std::to_string(r) + " level " + std::to_string(l) + " not set");
      build_dev_level(RL.host[r], RL.sub[r], l, h->opt);
      stride = std::max<int64_t>(stride, RL.sub[r].n);
    }
    RL.stride = stride;
    max_stride = std::max(max_stride, stride);
    for (int r = 0; r < h->world; ++r) RL.sub[r].offset = r * stride;
    const DevLevel& mine = h->levels[l].sub[0];
    if (RL.sub[h->rank_base].n != mine.n || RL.sub[h->rank_base].perm != mine.perm)
      invalid("replica of this rank differs from its own level " + std::to_string(l));
    if (l > 0)
      for (int r = 0; r < h->world; ++r)
        build_transfer(RL.host[r], RL.sub[r], R.lv[static_cast<size_t>(l - 1)].host[r],
                       R.lv[static_cast<size_t>(l - 1)].sub[r], h->opt);
    build_exchange(RL.host, RL.sub, 0, true, RL.scatter, RL.acc);
    RL.x.alloc(2 * stride * h->world);
    RL.b.alloc(stride * h->world);
    RL.r.alloc(stride * h->world);
    PF_CUDA(cudaMemset(RL.x.p, 0, sizeof(double) * 2 * stride * h->world));
    PF_CUDA(cudaMemset(RL.b.p, 0, sizeof(double) * stride * h->world));
  }
  auto& R0 = R.lv[0];
  std::vector<CoarseSub> cs;
  for (DevLevel& D : R0.sub) cs.push_back(CoarseSub{view(D.A), D.d_perm.p, D.n_own, D.offset});
  R.subs.upload(cs);
  R.cpack = make_coarse_pack(R0.host, R0.sub, R0.scatter, R.cp_sub_rows, R.cp_rowptr, R.cp_rowdev, R.cp_cols,
                             R.cp_vals);
  R.send.alloc(max_stride);
  PF_CUDA(cudaMemset(R.send.p, 0, sizeof(double) * max_stride));
  R.coarse_stats.alloc(4);
  PF_CUDA(cudaMemset(R.coarse_stats.p, 0, 4 * sizeof(double)));
  R.active = true;
}

// One level as the bottom kernel sees it.
struct BotSrc {
  const std::vector<DevLevel>* sub;
  int64_t total;
  const std::array<ExchangePlan, PF_NUM_CHANNEL_KINDS>* scatter;
  const ExchangePlan* acc;
  double *x, *xa, *b, *r;
};

// The bottom kernel reads fp64 values (its latency-bound rows have one dependent load
// fewer): an index-encoded operator of a bottom level gets a decoded fp64 copy (a few KB
// to a few MB: the bottom levels are tiny), the same doubles the table holds.
SellView fp64_view(pf_hierarchy::Bottom& bot, const DevSell& S) {
  SellView v = view(S);
  if (S.vals.vkind == 0) return v;
  std::vector<double> table(static_cast<size_t>(S.vals.table.n));
  PF_CUDA(cudaMemcpy(table.data(), S.vals.table.p, sizeof(double) * table.size(), cudaMemcpyDeviceToHost));
  std::vector<double> vals(static_cast<size_t>(S.stored));
  if (S.vals.vkind == 1) {
    std::vector<uint8_t> ix(vals.size());
    PF_CUDA(cudaMemcpy(ix.data(), S.vals.vi8.p, ix.size(), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < vals.size(); ++i) vals[i] = table[ix[i]];
  } else {
    std::vector<uint16_t> ix(vals.size());
    PF_CUDA(cudaMemcpy(ix.data(), S.vals.vi16.p, sizeof(uint16_t) * ix.size(), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < vals.size(); ++i) vals[i] = table[ix[i]];
  }
  bot.val_bufs.emplace_back();
  bot.val_bufs.back().upload(vals);
  v.vals = bot.val_bufs.back().p;
  v.vidx = nullptr;
  v.table = nullptr;
  v.vkind = 0;
  v.table_n = 0;
  return v;
}

// Plan and build the shared-memory staging of the block levels (BotStage, pf_bottom.cuh):
// levels 0, 1, ... up to block_top are staged while they fit the opt-in shared memory next
// to the descriptor and the coarse pack — each with its vectors, operator, restriction,
// colour ranges, Dirichlet flags and plans; then the prolongations, lowest level first,
// as far as they still fit (C2: levels 0-2 and every P but level 2's, ~200 KB).
void stage_block_levels(pf_hierarchy* h, pf_hierarchy::Bottom& bot, BotDesc& d, const std::vector<BotSrc>& src) {
  d.stage = BotStage{};
  d.stage.hs = -1;
  if (!h->opt.bottom_stage || d.block_top < 0) return;
  int optin = 0;
  PF_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
  auto r16 = [](int64_t b) { return (b + 15) / 16 * 16; };
  const int64_t smem_off = r16(sizeof(BotDesc)) + r16(static_cast<int64_t>(coarse_pack_smem(d.coarse)));
  const int64_t budget = static_cast<int64_t>(optin) - static_cast<int64_t>(bottom_kernel_static_smem()) - smem_off - 1024;
  struct Piece {
    const void* src;
    int64_t bytes, off;
  };
  std::vector<Piece> pieces;
  std::vector<std::pair<void**, int64_t>> fix;  // field of t -> blob offset
  int64_t used = 0, vec_bytes = 0;
  BotDesc t = d;
  auto add = [&](auto* field, const void* p, int64_t bytes) {  // field: a pointer member of t
    if (!p || bytes <= 0) return;
    pieces.push_back(Piece{p, bytes, used});
    fix.push_back({(void**)field, used});  // C cast: the members are __restrict__-qualified
    used += r16(bytes);
  };
  auto add_view = [&](SellView& v, const DevSell& S) {
    const int64_t n_slices = static_cast<int64_t>(S.slice_ptr.n);
    add(&v.cols, v.cols, S.stored * 4);
    add(&v.slice_ptr, v.slice_ptr, n_slices * 8);
    add(&v.row_len, v.row_len, S.row_len.bytes());
    if (S.vals.vkind == 1) {  // the 8-bit value index and its table
      v.vals = nullptr;
      v.vkind = 1;
      v.vidx = S.vals.vi8.p;
      v.table = S.vals.table.p;
      v.table_n = static_cast<int32_t>(S.vals.table.n);
      add(&v.vidx, v.vidx, S.stored);
      add(&v.table, v.table, S.vals.table.bytes());
    } else {  // the decoded fp64 copy the descriptor already holds
      add(&v.vals, v.vals, S.stored * 8);
    }
  };
  auto plan = [&](BotPlan& P) {
    add(&P.dst, P.dst, static_cast<int64_t>(P.n) * 4);
    add(&P.src, P.src, static_cast<int64_t>(P.n) * 4);
  };
  int hs = -1;
  for (int l = 0; l <= d.block_top; ++l) {
    const size_t p0 = pieces.size();
    const int64_t u0 = used;
    bool ok = true;
    const BotSrc& L = src[static_cast<size_t>(l)];
    BotLevel& B = t.lev[l];
    plan(B.ms);
    plan(B.h1);
    plan(B.h2);
    if (B.acc_n > 0) {
      add(&B.acc_off, B.acc_off, (static_cast<int64_t>(B.acc_n) + 1) * 4);
      add(&B.acc_src, B.acc_src, L.acc->acc_src.bytes());
      add(&B.acc_dst, B.acc_dst, static_cast<int64_t>(B.acc_n) * 4);
    }
    for (int s = 0; s < t.n_sub; ++s) {
      const DevLevel& D = (*L.sub)[static_cast<size_t>(s)];
      BotSub& S = t.sub[l][s];
      if (D.A.max_len > kBotChunk) ok = false;
      add_view(S.A, D.A);
      if (l > 0) add_view(S.R, D.R);
      add(&S.color_start, S.color_start, (static_cast<int64_t>(S.n_colors) + 1) * 4);
      add(&S.is_dir, S.is_dir, D.d_is_dir.bytes());
    }
    const int64_t vb = 4 * r16(L.total * 8);
    if (!ok || used + vec_bytes + vb > budget) {  // roll back level l and stop
      pieces.resize(p0);
      fix.resize(p0);
      used = u0;
      t.lev[l] = d.lev[l];
      for (int s = 0; s < t.n_sub; ++s) t.sub[l][s] = d.sub[l][s];
      break;
    }
    vec_bytes += vb;
    hs = l;
  }
  if (hs < 0) return;
  for (int l = 1; l <= hs; ++l)  // prolongations, as far as they fit
    for (int s = 0; s < t.n_sub; ++s) {
      const DevLevel& D = (*src[static_cast<size_t>(l)].sub)[static_cast<size_t>(s)];
      const size_t p0 = pieces.size();
      const int64_t u0 = used;
      const BotSub keep = t.sub[l][s];
      add_view(t.sub[l][s].P, D.P);
      if (used + vec_bytes > budget) {
        pieces.resize(p0);
        fix.resize(p0);
        used = u0;
        t.sub[l][s] = keep;
      }
    }
  bot.stage_blob.alloc(used);
  for (const Piece& q : pieces)
    PF_CUDA(cudaMemcpy(bot.stage_blob.p + q.off, q.src, static_cast<size_t>(q.bytes), cudaMemcpyDeviceToDevice));
  for (auto& f : fix) *f.first = bot.stage_blob.p + f.second;
  t.stage.blob = bot.stage_blob.p;
  t.stage.blob_bytes = used;
  t.stage.hs = hs;
  t.stage.smem_off = smem_off;
  int64_t off = used;
  for (int l = 0; l <= hs; ++l)
    for (int k = 0; k < 4; ++k) {
      t.stage.vec_off[l][k] = off;
      off += r16(src[static_cast<size_t>(l)].total * 8);
    }
  t.stage.arena_bytes = off;
  d = t;
}

// Fill and upload a BotDesc for levels 0..top = src.size()-1; false if unsupported.
bool fill_bottom(pf_hierarchy* h, pf_hierarchy::Bottom& bot, const std::vector<BotSrc>& src,
                 const CoarsePack& pack, double* coarse_stats) {
  const int top = static_cast<int>(src.size()) - 1;
  const int n_sub = static_cast<int>(src[0].sub->size());
  if (top < 1 || top >= kBotMaxLevels || n_sub > kBotMaxSubs) return false;
  if (coarse_pack_smem(pack) > kCoarseSmemMax) return false;
  BotDesc d;
  std::memset(&d, 0, sizeof d);
  d.n_sub = n_sub;
  d.n_levels = top + 1;
  const int64_t block_rows = h->opt.bottom_block_rows;
  d.block_top = -1;
  for (int l = 0; l <= top; ++l)
    if (src[l].total <= block_rows) d.block_top = l;
  d.coarse = pack;
  d.coarse_stats = coarse_stats;
  auto plan = [](const ExchangePlan& P) { return BotPlan{P.dst.p, P.src.p, static_cast<int32_t>(P.n)}; };
  int64_t max_total = 0;
  for (int l = 0; l <= top; ++l) {
    const BotSrc& L = src[l];
    BotLevel& B = d.lev[l];
    B.x = L.x;
    B.xa = L.xa;
    B.b = L.b;
    B.r = L.r;
    B.total = static_cast<int32_t>(L.total);
    max_total = std::max(max_total, L.total);
    B.ms = plan((*L.scatter)[PF_CH_MASTER_SLAVE]);
    B.h1 = plan((*L.scatter)[PF_CH_HALO1]);
    B.h2 = plan((*L.scatter)[PF_CH_HALO2]);
    B.acc_off = L.acc->acc_off.p;
    B.acc_src = L.acc->acc_src.p;
    B.acc_dst = L.acc->acc_dst.p;
    B.acc_n = L.acc->n_masters;
    for (int s = 0; s < n_sub; ++s) {
      const DevLevel& D = (*L.sub)[s];
      BotSub& S = d.sub[l][s];
      B.max_colors = std::max(B.max_colors, D.n_colors);
      bot.color_bufs.emplace_back();
      bot.color_bufs.back().upload(D.color_start);
      S.A = fp64_view(bot, D.A);
      S.host_of_own = D.d_perm.p;
      S.color_start = bot.color_bufs.back().p;
      S.P = fp64_view(bot, D.P);
      S.R = fp64_view(bot, D.R);
      S.is_dir = D.d_is_dir.p;
      S.n = D.n;
      S.n_own = D.n_own;
      S.n_colors = D.n_colors;
      S.off = static_cast<int32_t>(D.offset);
    }
  }
  stage_block_levels(h, bot, d, src);
  if (std::getenv("PF_BOTTOM_PROFILE")) {
    PF_CUDA(cudaMalloc(&bot.stamps, 256 * sizeof(unsigned long long)));
    PF_CUDA(cudaMemset(bot.stamps, 0, 256 * sizeof(unsigned long long)));
    d.stamps = static_cast<unsigned long long*>(bot.stamps);
  }
  PF_CUDA(cudaMalloc(&bot.desc, sizeof(BotDesc)));
  PF_CUDA(cudaMemcpy(bot.desc, &d, sizeof d, cudaMemcpyHostToDevice));
  int sms = 0, occ = 0;
  PF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
  bot.smem = d.stage.hs >= 0 ? static_cast<size_t>(d.stage.smem_off + d.stage.arena_bytes)
                            : ((sizeof(BotDesc) + 15) / 16) * 16 + coarse_pack_smem(d.coarse);
  if (bot.smem > 48 * 1024) bottom_kernel_caps(h->device);  // the cap, not the size
  occ = bottom_kernel_occupancy(bot.smem);
  if (occ < 1) return false;
  int64_t want = std::max<int64_t>(sms, (max_total + kBlock - 1) / kBlock);
  if (h->opt.bottom_grid > 0) want = h->opt.bottom_grid;
  bot.grid = static_cast<int>(std::min<int64_t>(want, static_cast<int64_t>(occ) * sms));
  // every bottom level staged for block 0: the other blocks would only wait at barriers
  bot.staged_all = d.stage.hs == top && d.block_top == top;
  if (bot.staged_all && h->opt.bottom_grid <= 0) bot.grid = 1;
  bot.top = top;
  bot.active = true;
  return true;
}

// Single-device bottom kernel: levels up to Options::bottom_rows rows (default 1024: at C2
// the coloured smoothers' V-cycle is 1.443 ms with no bottom kernel, 1.383 with levels <=
// 64k rows, 1.356 with levels <= 1k rows).  Damped Jacobi does not use it unless
// Options::bottom_jacobi: with programmatic dependent launch in the graph, separate
// per-level kernels are faster for it (0.715 vs 0.744 ms).  Multi-process runs replicate
// levels up to Options::rep_bottom_rows rows in total (one allgather per cycle).
bool bottom_for(const pf_hierarchy* h, const pf_multigrid_config& cfg) {
  return cfg.smoother.kind != PF_SMOOTHER_JACOBI || h->opt.bottom_jacobi != 0;
}
// Levels whose total row count stays below the limit run as one cooperative kernel when
// every rank of the level lives on this device.
void build_bottom(pf_hierarchy* h) {
  const int64_t limit = h->opt.bottom_rows;
  if (h->world != h->n_sub || limit <= 0) return;
  int top = -1;
  for (int l = 0; l < h->n_levels - 1 && l < kBotMaxLevels; ++l)
    if (h->levels[l].total <= limit) top = l;
  if (top < 1) return;
  std::vector<BotSrc> src;
  for (int l = 0; l <= top; ++l) {
    Level& L = h->levels[l];
    src.push_back(BotSrc{&L.sub, L.total, &L.scatter, &L.accumulate, L.x->cur(), L.x->alt(), L.b->cur(), L.r.p});
  }
  fill_bottom(h, h->bot, src, h->levels[0].cpack, h->levels[0].coarse_stats.p);
}

// Multi-process: the bottom kernel over the replicated levels (all ranks on every GPU),
// if they are all small enough; otherwise only the coarse replica is used.
void build_rep_bottom(pf_hierarchy* h) {
  auto& R = h->rep;
  const int top = static_cast<int>(R.lv.size()) - 1;
  const int64_t limit = h->opt.rep_bottom_rows;
  if (top < 1 || top >= h->n_levels - 1 || limit <= 0) return;
  std::vector<BotSrc> src;
  for (int l = 0; l <= top; ++l) {
    auto& RL = R.lv[static_cast<size_t>(l)];
    const int64_t total = RL.stride * h->world;
    if (total > limit) return;
    src.push_back(BotSrc{&RL.sub, total, &RL.scatter, &RL.acc, RL.x.p, RL.x.p + total, RL.b.p, RL.r.p});
  }
  fill_bottom(h, R.bot, src, R.cpack, h->levels[0].coarse_stats.p);
}

}  // namespace rt
}  // namespace pf
