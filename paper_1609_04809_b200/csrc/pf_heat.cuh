// pf_heat.cuh — device kernels of the Crank-Nicolson heat loop (app.cpp:146-230).
//
// Every kernel reproduces the reference's floating-point expression tree with
// round-to-nearest intrinsics (no contraction), so the loop's iterates equal the
// reference's bit for bit.
#pragma once

#include "pf_kernels.cuh"

namespace pf {

// The finest-level load description on the device (pf_load_desc), per-row arrays in
// device order.
struct LoadView {
  const int32_t* lattice;  // [3 * n]
  const uint32_t* cells;   // [n] count | 3-bit cell codes in gcn order
  const double* factor;    // [3][N][2]
  const double* extent;    // [3][N]
  const double* phi;       // [8][8]
  double qweight;
  int32_t n_cells;
  int32_t dim;
};

// ring slot (mesh.cpp:16-21) of the vertex at offset (ox, oy, oz) in {0,1}^3 of a cell,
// indexed by ox | oy << 1 | oz << 2
__constant__ int8_t c_ring_slot[8] = {0, 1, 3, 2, 4, 5, 7, 6};

// assemble_load (assembly.cpp:144-160) gathered per dof: for each own cell around the
// dof in ascending gcn order, the element load of the dof's slot,
//   sum_q (w * f(t, x_q)) * phi_q(slot),  w = qweight * volume,  f = s * profile(x_q),
// (element_matrices, assembly.cpp:60-88), added into the dof's sum in cell order.
template <int kDim>
__global__ void __launch_bounds__(kBlock) k_load(LoadView L, double s, double* __restrict__ out, int32_t n) {
  PF_PDL_ENTRY();
  const int32_t row = blockIdx.x * kBlock + threadIdx.x;
  if (row >= n) return;
  const uint32_t w = L.cells[row];
  const int cnt = static_cast<int>(w & 15u);
  double acc = 0.0;
  if (cnt > 0) {
    const int32_t x = L.lattice[3 * row], y = L.lattice[3 * row + 1], z = L.lattice[3 * row + 2];
    const int64_t N = L.n_cells;
    for (int k = 0; k < cnt; ++k) {
      const uint32_t bits = (w >> (4 + 3 * k)) & 7u;
      const int32_t cx = x - 1 + static_cast<int32_t>(bits & 1u);
      const int32_t cy = y - 1 + static_cast<int32_t>((bits >> 1) & 1u);
      const int32_t cz = kDim == 3 ? z - 1 + static_cast<int32_t>((bits >> 2) & 1u) : 0;
      // the dof's offset inside the cell is 1 - bit per axis
      const int slot = c_ring_slot[(~bits) & (kDim == 3 ? 7u : 3u)];
      const double hx = __ldg(L.extent + cx), hy = __ldg(L.extent + N + cy);
      const double vol = kDim == 3 ? __dmul_rn(__dmul_rn(hx, hy), __ldg(L.extent + 2 * N + cz))
                                   : __dmul_rn(hx, hy);
      const double wq = __dmul_rn(L.qweight, vol);
      const double* fx = L.factor + 2 * cx;
      const double* fy = L.factor + 2 * (N + cy);
      const double* fz = L.factor + 2 * (2 * N + cz);
      double el = 0.0;
#pragma unroll
      for (int q = 0; q < (1 << kDim); ++q) {
        const int ix = kDim == 3 ? q >> 2 : q >> 1;
        const int iy = kDim == 3 ? (q >> 1) & 1 : q & 1;
        double prof = __dmul_rn(__ldg(fx + ix), __ldg(fy + iy));
        if (kDim == 3) prof = __dmul_rn(prof, __ldg(fz + (q & 1)));
        const double fq = __dmul_rn(s, prof);
        el = __dadd_rn(el, __dmul_rn(__dmul_rn(wq, fq), __ldg(L.phi + q * 8 + slot)));
      }
      acc = __dadd_rn(acc, el);
    }
  }
  out[row] = acc;
}

// b = Op u + half_dt (load_now + load_next) on every non-Dirichlet row (app.cpp:191-194:
// spmv, then b_i += 0.5 dt (ln_i + lnx_i)); Dirichlet rows are written by k_dirichlet.
template <int kVK>
__global__ void __launch_bounds__(kBlock, minb_for<kVK>(PF_ROW_MINB)) k_cn_rhs(SellView Op, const double* __restrict__ u,
                                                   const double* __restrict__ ln,
                                                   const double* __restrict__ lnx, double half_dt,
                                                   const uint8_t* __restrict__ is_dir,
                                                   double* __restrict__ b, int32_t n) {
  PF_PDL_ENTRY();
  const int32_t row = blockIdx.x * kBlock + threadIdx.x;
  if (row >= n || is_dir[row]) return;
  const double y = row_dot<false, true, kVK>(Op, row, u, 0.0);
  b[row] = __dadd_rn(y, __dmul_rn(half_dt, __dadd_rn(ln[row], lnx[row])));
}

// apply_dirichlet_rhs (assembly.cpp:172-179) with g = scale * profile, and u_D = b_D
// (app.cpp:196-200) when u is given.
static __global__ void __launch_bounds__(kBlock) k_dirichlet(const int32_t* __restrict__ idx,
                                                      const double* __restrict__ prof, int32_t n_dir,
                                                      int has, double scale, double* __restrict__ b,
                                                      double* __restrict__ u) {
  PF_PDL_ENTRY();
  const int32_t i = blockIdx.x * kBlock + threadIdx.x;
  if (i >= n_dir) return;
  const double v = has ? __dmul_rn(scale, prof[i]) : 0.0;
  const int32_t r = idx[i];
  b[r] = v;
  if (u) u[r] = v;
}

}  // namespace pf
