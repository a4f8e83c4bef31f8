// pf_assembly.cuh — device assembly of the finest-level Q1 stiffness system (SURVEY.md §8f
// rank 2; assemble_system / apply_dirichlet_rows, assembly.cpp:103-142, :162-170).
#pragma once

#include "pf_heat.cuh"
#include "pf_kernels.cuh"

namespace pf {

struct AsmView {
  const int32_t* lattice;    // [3 n], device order
  const uint8_t* cell_mask;  // [n], device order
  const uint8_t* is_dir;     // [n], device order
  const double* kappa;       // [N^d] or null
  const double* elem;        // [classes][64]
  const int32_t* cls;        // [3][N]
  int32_t N, nh, n_coarse, level;
};

// global cell number (mesh.cpp:93-100, :170-176): coarse cells lexicographic, children
// nc * parent + child index, child offset (c/4, c/2 % 2, c % 2)
template <int kDim>
__device__ __forceinline__ int64_t cell_gcn(const AsmView& V, int32_t x, int32_t y, int32_t z) {
  const int64_t n = V.n_coarse;
  const int L = V.level;
  int64_t g = kDim == 3 ? ((static_cast<int64_t>(x >> L) * n) + (y >> L)) * n + (z >> L)
                        : static_cast<int64_t>(x >> L) * n + (y >> L);
  for (int b = L - 1; b >= 0; --b) {
    const int64_t ci = kDim == 3 ? (((x >> b) & 1) << 2) | (((y >> b) & 1) << 1) | ((z >> b) & 1)
                                 : (((x >> b) & 1) << 1) | ((y >> b) & 1);
    g = g * (1 << kDim) + ci;
  }
  return g;
}

// One thread per row: every stored entry (p, q) of the row is the sum, over the local cells
// containing both vertices in ascending gcn, of kappa_c * K_e(c)[slot p][slot q]
// (assembly.cpp:114-131, gcn-ordered cell loop); Dirichlet rows -> identity (:162-170).
template <int kDim>
__global__ void __launch_bounds__(kBlock) k_assemble(AsmView V, SellView P, double* __restrict__ out, int32_t n) {
  PF_PDL_ENTRY();
  const int32_t row = blockIdx.x * kBlock + threadIdx.x;
  if (row >= n) return;
  const int64_t base = sell_row_base(P.slice_ptr, row);
  const int len = P.row_len[row];
  const int32_t px = V.lattice[3 * row], py = V.lattice[3 * row + 1], pz = V.lattice[3 * row + 2];
  const uint32_t mask = V.cell_mask[row];
  const bool dir = V.is_dir[row] != 0;
  const int64_t N = V.N;
  for (int j = 0; j < len; ++j) {
    const int64_t e = sell_entry(base, j);
    const int32_t c = P.cols[e];
    if (dir) {
      out[e] = c == row ? 1.0 : 0.0;
      continue;
    }
    const int32_t qx = V.lattice[3 * c], qy = V.lattice[3 * c + 1], qz = V.lattice[3 * c + 2];
    int64_t key[8];
    int kk[8];
    int nc = 0;
    for (int k = 0; k < (1 << kDim); ++k) {
      if (!((mask >> k) & 1u)) continue;
      const int32_t cx = px - 1 + (k & 1), cy = py - 1 + ((k >> 1) & 1), cz = kDim == 3 ? pz - 1 + ((k >> 2) & 1) : 0;
      if (qx < cx || qx > cx + 1 || qy < cy || qy > cy + 1 || (kDim == 3 && (qz < cz || qz > cz + 1))) continue;
      key[nc] = cell_gcn<kDim>(V, cx, cy, cz);
      kk[nc] = k;
      ++nc;
    }
    for (int a = 1; a < nc; ++a)  // ascending gcn
      for (int b = a; b > 0 && key[b - 1] > key[b]; --b) {
        const int64_t tk = key[b - 1];
        key[b - 1] = key[b];
        key[b] = tk;
        const int t = kk[b - 1];
        kk[b - 1] = kk[b];
        kk[b] = t;
      }
    double v = 0.0;
    for (int a = 0; a < nc; ++a) {
      const int k = kk[a];
      const int32_t cx = px - 1 + (k & 1), cy = py - 1 + ((k >> 1) & 1), cz = kDim == 3 ? pz - 1 + ((k >> 2) & 1) : 0;
      const int si = c_ring_slot[(~k) & ((1 << kDim) - 1)];
      const int oq = (qx - cx) | ((qy - cy) << 1) | (kDim == 3 ? (qz - cz) << 2 : 0);
      const int sj = c_ring_slot[oq];
      const int cl = kDim == 3 ? (V.cls[cx] * V.nh + V.cls[N + cy]) * V.nh + V.cls[2 * N + cz]
                               : V.cls[cx] * V.nh + V.cls[N + cy];
      const double ke = V.elem[cl * 64 + si * 8 + sj];
      const double val = V.kappa ? __dmul_rn(V.kappa[(static_cast<int64_t>(cx) * N + cy) * (kDim == 3 ? N : 1) + cz], ke)
                                 : ke;
      v = __dadd_rn(v, val);
    }
    out[e] = v;
  }
}

}  // namespace pf
