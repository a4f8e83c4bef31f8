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

// ------------------------------------------------------- Q2 and rotated Q1 (pf_fe.h) --

struct FeAsmView {
  const int32_t* lattice;  // [3 n] entity coordinates, device order
  const uint8_t* orient;   // [n] face orientation (rotated Q1), device order
  const uint8_t* is_dir;   // [n], device order
  const double* elem;      // 27 x 27 (Q2) or 6 x 6 (rotated Q1), h included
  const double* kappa;     // [N^3] (rotated Q1) or null
  int32_t N;
};

// Q2: cells along one axis containing node i, ascending (at most 2)
__device__ __forceinline__ int fe_q2_cells(int32_t i, int32_t N, int32_t* out) {
  if (i & 1) {
    out[0] = (i - 1) >> 1;
    return 1;
  }
  int n = 0;
  if ((i >> 1) - 1 >= 0) out[n++] = (i >> 1) - 1;
  if ((i >> 1) < N) out[n++] = i >> 1;
  return n;
}

// One thread per row; every stored entry is the sum over the cells containing both
// entities in ascending cell order of [kappa_c *] K_e[slot row][slot col], exactly as
// pf_fe_setup.cpp's q2_level / rt_level form it; Dirichlet rows -> identity.
template <int kFamily>
__global__ void __launch_bounds__(kBlock) k_fe_assemble(FeAsmView V, SellView P, double* __restrict__ out,
                                                        int32_t n) {
  PF_PDL_ENTRY();
  const int32_t row = blockIdx.x * kBlock + threadIdx.x;
  if (row >= n) return;
  const int64_t base = sell_row_base(P.slice_ptr, row);
  const int len = P.row_len[row];
  const int32_t a[3] = {V.lattice[3 * row], V.lattice[3 * row + 1], V.lattice[3 * row + 2]};
  const bool dir = V.is_dir[row] != 0;
  const int32_t N = V.N;
  if (kFamily == 2) {  // Q2
    int32_t ac[3][2];
    int na[3];
    for (int t = 0; t < 3; ++t) na[t] = fe_q2_cells(a[t], N, ac[t]);
    for (int j = 0; j < len; ++j) {
      const int64_t e = sell_entry(base, j);
      const int32_t c = P.cols[e];
      if (dir) {
        out[e] = c == row ? 1.0 : 0.0;
        continue;
      }
      const int32_t b[3] = {V.lattice[3 * c], V.lattice[3 * c + 1], V.lattice[3 * c + 2]};
      int32_t sc[3][2];
      int ns[3];
      for (int t = 0; t < 3; ++t) {
        int32_t bc[2];
        const int nb = fe_q2_cells(b[t], N, bc);
        ns[t] = 0;
        for (int u = 0; u < na[t]; ++u)
          for (int w = 0; w < nb; ++w)
            if (ac[t][u] == bc[w]) sc[t][ns[t]++] = ac[t][u];
      }
      double v = 0.0;
      for (int u = 0; u < ns[0]; ++u)
        for (int w = 0; w < ns[1]; ++w)
          for (int q = 0; q < ns[2]; ++q) {
            const int32_t cx = sc[0][u], cy = sc[1][w], cz = sc[2][q];
            const int la = ((a[0] - 2 * cx) * 3 + (a[1] - 2 * cy)) * 3 + (a[2] - 2 * cz);
            const int lb = ((b[0] - 2 * cx) * 3 + (b[1] - 2 * cy)) * 3 + (b[2] - 2 * cz);
            v = __dadd_rn(v, V.elem[la * 27 + lb]);
          }
      out[e] = v;
    }
  } else {  // rotated Q1: faces (o, a); the cells of a face differ along o only
    const int o = V.orient[row];
    for (int j = 0; j < len; ++j) {
      const int64_t e = sell_entry(base, j);
      const int32_t c = P.cols[e];
      if (dir) {
        out[e] = c == row ? 1.0 : 0.0;
        continue;
      }
      const int o2 = V.orient[c];
      const int32_t b[3] = {V.lattice[3 * c], V.lattice[3 * c + 1], V.lattice[3 * c + 2]};
      double v = 0.0;
      for (int side = 0; side < 2; ++side) {  // the row face's cells, ascending
        int32_t cc[3] = {a[0], a[1], a[2]};
        cc[o] = a[o] - 1 + side;
        if (cc[o] < 0 || cc[o] >= N) continue;
        // is the column face a face of this cell?
        bool in = true;
        for (int t = 0; t < 3; ++t)
          if (t != o2 && b[t] != cc[t]) in = false;
        if (!in || (b[o2] != cc[o2] && b[o2] != cc[o2] + 1)) continue;
        const int sa = 2 * o + (side == 0 ? 1 : 0);
        const int sb = 2 * o2 + (b[o2] == cc[o2] + 1 ? 1 : 0);
        const double k = V.kappa[(static_cast<int64_t>(cc[0]) * N + cc[1]) * N + cc[2]];
        v = __dadd_rn(v, __dmul_rn(k, V.elem[sa * 6 + sb]));
      }
      out[e] = v;
    }
  }
}

}  // namespace pf
