// pf_ops.cu — the C ABI around the V-cycle for the time-dependent model problem and the
// device assembly: a second value set on a level's pattern (the CN rhs operator M - dt/2 K,
// app.cpp:185-191), the load assembly (assembly.cpp:144-160) and Dirichlet rows
// (assembly.cpp:172-179), the CN right-hand side, the heat time loop of heat_rank_body
// (app.cpp:180-213), and the device assembly of level operators (assembly.cpp:103-170;
// Q2 / rotated Q1: pf_fe.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "pf_assembly.cuh"
#include "pf_heat.cuh"
#include "pf_internal.hpp"
#include "pf_kernels.cuh"

using namespace pf;
using namespace pf::rt;

// A second value set on a level's operator pattern (pf_operator_create).
struct pf_operator {
  pf_hierarchy* h = nullptr;
  int level = 0;
  std::vector<pf::DevVals> vals;  // per subdomain, SELL layout of DevLevel::A
  std::vector<bool> set;
};

// Device assembly description per subdomain (pf_assembly_create / pf_assembly_set).
struct pf_assembly {
  pf_hierarchy* h = nullptr;
  int level = 0;
  struct Sub {
    bool set = false;
    int dim = 3;
    int32_t N = 0, nh = 0, n_coarse = 0, grid_level = 0;
    pf::DevBuf<int32_t> lattice, cls;
    pf::DevBuf<uint8_t> cell_mask;
    pf::DevBuf<double> kappa, elem;
    int family = 0;  // 0: Q1 (pf_assembly_desc); PF_FE_Q2 / PF_FE_ROTATED_Q1 (pf_fe_assembly_desc)
    pf::DevBuf<uint8_t> orient;
  };
  std::vector<Sub> sub;
};

// The finest-level load description on the device (pf_load_create / pf_load_set).
struct pf_load {
  pf_hierarchy* h = nullptr;
  int level = 0;
  struct Sub {
    bool set = false;
    int dim = 3;
    int32_t n_cells = 0;
    double qweight = 0.0;
    pf::DevBuf<int32_t> lattice;
    pf::DevBuf<uint32_t> cells;
    pf::DevBuf<double> factor, extent, phi;
    pf::DevBuf<int32_t> dir_idx;   // Dirichlet rows, level-global device index
    pf::DevBuf<double> dir_prof;   // profile at those rows
  };
  std::vector<Sub> sub;
  std::unique_ptr<pf_vector> next;  // pf_heat_run's next-load scratch (kept across calls)
};

// ------------------------------------------------------------ heat (Crank-Nicolson) --

namespace pf {
namespace {

SellView op_view(const pf_operator* op, int s) {
  return view_of(op->vals[s], op->h->levels[op->level].sub[s].A);
}

void check_op(const pf_operator* op) {
  if (!op) invalid("null operator");
  for (size_t s = 0; s < op->set.size(); ++s)
    if (!op->set[s]) state("operator values of subdomain " + std::to_string(s) + " not set");
}

void check_load(const pf_load* ld) {
  if (!ld) invalid("null load");
  for (size_t s = 0; s < ld->sub.size(); ++s)
    if (!ld->sub[s].set) state("load description of subdomain " + std::to_string(s) + " not set");
}

void enq_load(pf_load* ld, double scale, double* out) {
  pf_hierarchy* h = ld->h;
  Level& L = h->levels[ld->level];
  auto launch = launcher(h);
  for (int s = 0; s < h->n_sub; ++s) {
    const pf_load::Sub& S = ld->sub[s];
    const DevLevel& D = L.sub[s];
    const LoadView v{S.lattice.p, S.cells.p, S.factor.p, S.extent.p, S.phi.p, S.qweight, S.n_cells, S.dim};
    if (S.dim == 3)
      launch(grid_for(D.n), kBlock, k_load<3>, v, scale, out + D.offset, D.n);
    else
      launch(grid_for(D.n), kBlock, k_load<2>, v, scale, out + D.offset, D.n);
  }
  enq_update_ms(h, ld->level, out, PF_UPDATE_ACCUMULATE_THEN_SCATTER);
}

void enq_dirichlet(pf_load* ld, int has, double scale, double* b, double* u) {
  pf_hierarchy* h = ld->h;
  auto launch = launcher(h);
  for (int s = 0; s < h->n_sub; ++s) {
    const pf_load::Sub& S = ld->sub[s];
    launch(grid_for(S.dir_idx.n), kBlock, k_dirichlet, static_cast<const int32_t*>(S.dir_idx.p),
           static_cast<const double*>(S.dir_prof.p), static_cast<int32_t>(S.dir_idx.n), has, scale, b, u);
  }
}

void enq_cn_rhs(pf_operator* op, pf_load* ld, const double* u, const double* ln, const double* lnx,
                double half_dt, int has, double gscale, double* b, double* u_out) {
  pf_hierarchy* h = op->h;
  Level& L = h->levels[op->level];
  auto launch = launcher(h);
  for (int s = 0; s < h->n_sub; ++s) {
    const DevLevel& D = L.sub[s];
    vk_dispatch(op->vals[s].vkind, [&](auto V) {
      launch(grid_for(D.n), kBlock, k_cn_rhs<decltype(V)::value>, op_view(op, s), u + D.offset, ln + D.offset,
             lnx + D.offset, half_dt, static_cast<const uint8_t*>(D.d_is_dir.p), b + D.offset, D.n);
    });
  }
  enq_dirichlet(ld, has, gscale, b, u_out);
}

}  // namespace
}  // namespace pf

extern "C" {

pf_status pf_operator_create(pf_hierarchy* h, int level, pf_operator** out) {
  PF_API_BEGIN
  check_level(h, level);
  if (!out) invalid("null output");
  auto op = std::make_unique<pf_operator>();
  op->h = h;
  op->level = level;
  op->vals.resize(static_cast<size_t>(h->n_sub));
  op->set.assign(static_cast<size_t>(h->n_sub), false);
  *out = op.release();
  PF_API_END
}

pf_status pf_operator_set_values(pf_operator* op, int sub, const double* values, int64_t nnz) {
  PF_API_BEGIN
  if (!op || !values) invalid("null argument");
  pf_hierarchy* h = op->h;
  if (sub < 0 || sub >= h->n_sub) invalid("subdomain out of range");
  const DevLevel& D = h->levels[op->level].sub[sub];
  if (nnz != D.A.nnz)
    invalid("operator nnz " + std::to_string(nnz) + " does not match the level's " + std::to_string(D.A.nnz));
  PF_CUDA(cudaSetDevice(h->device));
  std::vector<double> sv(static_cast<size_t>(D.A.stored), 0.0);
  for (int32_t hr = 0; hr < D.n; ++hr) {
    const int32_t d = D.perm[hr];
    const int64_t base = sell_row_base(D.sell_ptr.data(), d);
    for (int64_t k = D.csr_rowptr[hr]; k < D.csr_rowptr[hr + 1]; ++k)
      sv[static_cast<size_t>(sell_entry(base, static_cast<int>(k - D.csr_rowptr[hr])))] = values[k];
  }
  encode_values(sv, op->vals[sub], op->h->opt);
  op->set[sub] = true;
  PF_API_END
}

pf_status pf_operator_apply(pf_operator* op, const pf_vector* x, pf_vector* y) {
  PF_API_BEGIN
  check_op(op);
  pf_hierarchy* h = op->h;
  check_vec(h, x, op->level, "x");
  check_vec(h, y, op->level, "y");
  PF_CUDA(cudaSetDevice(h->device));
  Level& L = h->levels[op->level];
  auto launch = launcher(h);
  for (int s = 0; s < h->n_sub; ++s) {
    const DevLevel& D = L.sub[s];
    vk_dispatch(op->vals[s].vkind, [&](auto V) {
      launch(grid_for(D.n), kBlock, k_spmv<decltype(V)::value>, op_view(op, s), x->cur() + D.offset, y->cur() + D.offset, D.n);
    });
  }
  sync(h);
  PF_API_END
}

pf_status pf_operator_get_values(const pf_operator* op, int sub, double* values, int64_t nnz) {
  PF_API_BEGIN
  if (!op || !values) invalid("null argument");
  pf_hierarchy* h = op->h;
  if (sub < 0 || sub >= h->n_sub) invalid("subdomain out of range");
  if (!op->set[static_cast<size_t>(sub)]) state("operator values not set");
  const DevLevel& D = h->levels[op->level].sub[sub];
  if (nnz != D.A.nnz) invalid("nnz does not match the level");
  PF_CUDA(cudaSetDevice(h->device));
  const DevVals& V = op->vals[static_cast<size_t>(sub)];
  std::vector<double> sv(static_cast<size_t>(D.A.stored));
  if (V.vkind == 0) {
    PF_CUDA(cudaMemcpy(sv.data(), V.vals.p, sizeof(double) * sv.size(), cudaMemcpyDeviceToHost));
  } else {
    std::vector<double> table(static_cast<size_t>(V.table.n));
    PF_CUDA(cudaMemcpy(table.data(), V.table.p, sizeof(double) * table.size(), cudaMemcpyDeviceToHost));
    if (V.vkind == 1) {
      std::vector<uint8_t> ix(sv.size());
      PF_CUDA(cudaMemcpy(ix.data(), V.vi8.p, ix.size(), cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < sv.size(); ++i) sv[i] = table[ix[i]];
    } else {
      std::vector<uint16_t> ix(sv.size());
      PF_CUDA(cudaMemcpy(ix.data(), V.vi16.p, 2 * ix.size(), cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < sv.size(); ++i) sv[i] = table[ix[i]];
    }
  }
  for (int32_t hr = 0; hr < D.n; ++hr) {
    const int64_t base = sell_row_base(D.sell_ptr.data(), D.perm[hr]);
    for (int64_t k = D.csr_rowptr[hr]; k < D.csr_rowptr[hr + 1]; ++k)
      values[k] = sv[static_cast<size_t>(sell_entry(base, static_cast<int>(k - D.csr_rowptr[hr])))];
  }
  PF_API_END
}

pf_status pf_assembly_create(pf_hierarchy* h, int level, pf_assembly** out) {
  PF_API_BEGIN
  check_level(h, level);
  if (!out) invalid("null output");
  auto a = std::make_unique<pf_assembly>();
  a->h = h;
  a->level = level;
  a->sub.resize(static_cast<size_t>(h->n_sub));
  *out = a.release();
  PF_API_END
}

pf_status pf_assembly_set(pf_assembly* a, int sub, const pf_assembly_desc* d) {
  PF_API_BEGIN
  if (!a || !d) invalid("null argument");
  pf_hierarchy* h = a->h;
  if (sub < 0 || sub >= h->n_sub) invalid("subdomain out of range");
  const DevLevel& D = h->levels[a->level].sub[sub];
  if (d->n_dofs != D.n) invalid("assembly description does not match the level's dof count");
  if (d->dim != 2 && d->dim != 3) invalid("dimension must be 2 or 3");
  if (!d->lattice || !d->cell_mask || !d->elem || !d->elem_class || d->n_classes < 1 || d->n_cells < 1)
    invalid("null assembly array");
  if (d->n_coarse < 1 || d->level < 0 || (static_cast<int64_t>(d->n_coarse) << d->level) != d->n_cells)
    invalid("n_cells must be n_coarse * 2^level");
  PF_CUDA(cudaSetDevice(h->device));
  const int32_t n = D.n;
  std::vector<int32_t> lat(static_cast<size_t>(3 * n));
  std::vector<uint8_t> mask(static_cast<size_t>(n));
  for (int32_t i = 0; i < n; ++i) {
    const int32_t r = D.perm[i];
    for (int k = 0; k < 3; ++k) lat[3 * static_cast<size_t>(r) + k] = d->lattice[3 * static_cast<int64_t>(i) + k];
    mask[static_cast<size_t>(r)] = d->cell_mask[i];
  }
  const int64_t N = d->n_cells, ncells = d->dim == 3 ? N * N * N : N * N;
  const int64_t nel = d->dim == 3 ? int64_t(d->n_classes) * d->n_classes * d->n_classes
                                  : int64_t(d->n_classes) * d->n_classes;
  pf_assembly::Sub& S = a->sub[static_cast<size_t>(sub)];
  S.family = 0;
  S.dim = d->dim;
  S.N = d->n_cells;
  S.nh = d->n_classes;
  S.n_coarse = d->n_coarse;
  S.grid_level = d->level;
  S.lattice.upload(lat);
  S.cell_mask.upload(mask);
  S.cls.upload(std::vector<int32_t>(d->elem_class, d->elem_class + 3 * N));
  S.elem.upload(std::vector<double>(d->elem, d->elem + 64 * nel));
  if (d->kappa) S.kappa.upload(std::vector<double>(d->kappa, d->kappa + ncells));
  else S.kappa.reset();
  S.set = true;
  PF_API_END
}

pf_status pf_fe_assembly_set(pf_assembly* a, int sub, const pf_fe_assembly_desc* d) {
  PF_API_BEGIN
  if (!a || !d) invalid("null argument");
  pf_hierarchy* h = a->h;
  if (sub < 0 || sub >= h->n_sub) invalid("subdomain out of range");
  const DevLevel& D = h->levels[a->level].sub[sub];
  if (d->n_dofs != D.n) invalid("assembly description does not match the level's dof count");
  if (d->family != PF_FE_Q2 && d->family != PF_FE_ROTATED_Q1) invalid("unknown element family");
  if (!d->keys4 || !d->elem || d->n_cells < 1 || (d->family == PF_FE_ROTATED_Q1 && !d->kappa))
    invalid("null assembly array");
  PF_CUDA(cudaSetDevice(h->device));
  const int32_t n = D.n;
  std::vector<int32_t> lat(static_cast<size_t>(3 * n));
  std::vector<uint8_t> ori(static_cast<size_t>(n));
  for (int32_t i = 0; i < n; ++i) {
    const int32_t r = D.perm[i];
    for (int k = 0; k < 3; ++k) lat[3 * static_cast<size_t>(r) + k] = static_cast<int32_t>(d->keys4[4 * static_cast<int64_t>(i) + 1 + k]);
    ori[static_cast<size_t>(r)] = static_cast<uint8_t>(d->keys4[4 * static_cast<int64_t>(i)]);
  }
  const int64_t N = d->n_cells;
  pf_assembly::Sub& S = a->sub[static_cast<size_t>(sub)];
  S.family = d->family;
  S.dim = 3;
  S.N = d->n_cells;
  S.lattice.upload(lat);
  S.orient.upload(ori);
  S.elem.upload(std::vector<double>(d->elem, d->elem + (d->family == PF_FE_Q2 ? 27 * 27 : 36)));
  if (d->kappa) S.kappa.upload(std::vector<double>(d->kappa, d->kappa + N * N * N));
  else S.kappa.reset();
  S.set = true;
  PF_API_END
}

pf_status pf_assemble_operator(pf_assembly* a, pf_operator* op) {
  PF_API_BEGIN
  if (!a || !op) invalid("null argument");
  pf_hierarchy* h = a->h;
  if (op->h != h || op->level != a->level) invalid("operator of another level");
  for (const auto& S : a->sub)
    if (!S.set) state("assembly description not set for every subdomain");
  PF_CUDA(cudaSetDevice(h->device));
  auto launch = launcher(h);
  for (int s = 0; s < h->n_sub; ++s) {
    const DevLevel& D = h->levels[a->level].sub[s];
    const pf_assembly::Sub& S = a->sub[static_cast<size_t>(s)];
    DevVals& out = op->vals[static_cast<size_t>(s)];
    if (out.vkind != 0 || out.vals.n != D.A.stored) {  // fp64 values, allocated once
      out = DevVals{};
      out.vkind = 0;
      out.vals.alloc(D.A.stored);
      PF_CUDA(cudaMemsetAsync(out.vals.p, 0, sizeof(double) * static_cast<size_t>(D.A.stored), h->stream));
    }
    if (S.family != 0) {
      const FeAsmView fv{S.lattice.p, S.orient.p, D.d_is_dir.p, S.elem.p, S.kappa.p, S.N};
      if (S.family == PF_FE_Q2)
        launch(grid_for(D.n), kBlock, k_fe_assemble<PF_FE_Q2>, fv, view(D.A), out.vals.p, D.n);
      else
        launch(grid_for(D.n), kBlock, k_fe_assemble<PF_FE_ROTATED_Q1>, fv, view(D.A), out.vals.p, D.n);
      op->set[static_cast<size_t>(s)] = true;
      continue;
    }
    const AsmView v{S.lattice.p, S.cell_mask.p, D.d_is_dir.p, S.kappa.p, S.elem.p, S.cls.p, S.N, S.nh, S.n_coarse,
                    S.grid_level};
    if (S.dim == 3)
      launch(grid_for(D.n), kBlock, k_assemble<3>, v, view(D.A), out.vals.p, D.n);
    else
      launch(grid_for(D.n), kBlock, k_assemble<2>, v, view(D.A), out.vals.p, D.n);
    op->set[static_cast<size_t>(s)] = true;
  }
  sync(h);
  PF_API_END
}

pf_status pf_assembly_destroy(pf_assembly* a) {
  PF_API_BEGIN
  if (a) cudaSetDevice(a->h->device);
  delete a;
  PF_API_END
}

pf_status pf_operator_destroy(pf_operator* op) {
  PF_API_BEGIN
  if (op) cudaSetDevice(op->h->device);
  delete op;
  PF_API_END
}

pf_status pf_load_create(pf_hierarchy* h, int level, pf_load** out) {
  PF_API_BEGIN
  check_level(h, level);
  if (!out) invalid("null output");
  auto ld = std::make_unique<pf_load>();
  ld->h = h;
  ld->level = level;
  ld->sub.resize(static_cast<size_t>(h->n_sub));
  *out = ld.release();
  PF_API_END
}

pf_status pf_load_set(pf_load* ld, int sub, const pf_load_desc* d) {
  PF_API_BEGIN
  if (!ld || !d) invalid("null argument");
  pf_hierarchy* h = ld->h;
  if (sub < 0 || sub >= h->n_sub) invalid("subdomain out of range");
  const DevLevel& D = h->levels[ld->level].sub[sub];
  if (d->n_dofs != D.n) invalid("load description has " + std::to_string(d->n_dofs) + " dofs, level has " + std::to_string(D.n));
  if (d->dim != 2 && d->dim != 3) invalid("dimension must be 2 or 3");
  if (d->n_cells < 1) invalid("n_cells must be >= 1");
  if (!d->lattice || !d->cells || !d->factor || !d->extent || !d->phi || !d->boundary || !d->is_dirichlet)
    invalid("null load array");
  PF_CUDA(cudaSetDevice(h->device));
  const int32_t n = D.n;
  std::vector<int32_t> lat(static_cast<size_t>(3 * n));
  std::vector<uint32_t> cells(static_cast<size_t>(n));
  std::vector<int32_t> didx;
  std::vector<double> dprof;
  const int64_t N = d->n_cells;
  for (int32_t i = 0; i < n; ++i) {
    const int32_t r = D.perm[i];
    const uint32_t w = d->cells[i];
    const int cnt = static_cast<int>(w & 15u);
    if (cnt > (1 << d->dim)) invalid("load cell count out of range at dof " + std::to_string(i));
    for (int a = 0; a < 3; ++a) {
      const int32_t c = d->lattice[3 * static_cast<int64_t>(i) + a];
      if (cnt > 0 && (a < d->dim) && (c < 0 || c > N)) invalid("lattice coordinate out of range");
      lat[3 * static_cast<size_t>(r) + a] = c;
    }
    cells[static_cast<size_t>(r)] = w;
    if (d->is_dirichlet[i]) {
      didx.push_back(static_cast<int32_t>(D.offset) + r);
      dprof.push_back(d->boundary[i]);
    }
  }
  pf_load::Sub& S = ld->sub[static_cast<size_t>(sub)];
  S.dim = d->dim;
  S.n_cells = d->n_cells;
  S.qweight = d->qweight;
  S.lattice.upload(lat);
  S.cells.upload(cells);
  S.factor.upload(std::vector<double>(d->factor, d->factor + 3 * N * 2));
  S.extent.upload(std::vector<double>(d->extent, d->extent + 3 * N));
  S.phi.upload(std::vector<double>(d->phi, d->phi + 64));
  S.dir_idx.upload(didx);
  S.dir_prof.upload(dprof);
  S.set = true;
  PF_API_END
}

pf_status pf_load_assemble(pf_load* ld, double source_scale, pf_vector* out) {
  PF_API_BEGIN
  check_load(ld);
  pf_hierarchy* h = ld->h;
  check_vec(h, out, ld->level, "out");
  PF_CUDA(cudaSetDevice(h->device));
  enq_load(ld, source_scale, out->cur());
  sync(h);
  PF_API_END
}

pf_status pf_load_apply_dirichlet(pf_load* ld, int has_dirichlet, double scale, pf_vector* b, pf_vector* u) {
  PF_API_BEGIN
  check_load(ld);
  pf_hierarchy* h = ld->h;
  check_vec(h, b, ld->level, "b");
  if (u) check_vec(h, u, ld->level, "u");
  PF_CUDA(cudaSetDevice(h->device));
  enq_dirichlet(ld, has_dirichlet, scale, b->cur(), u ? u->cur() : nullptr);
  sync(h);
  PF_API_END
}

pf_status pf_load_destroy(pf_load* ld) {
  PF_API_BEGIN
  if (ld) cudaSetDevice(ld->h->device);
  delete ld;
  PF_API_END
}

pf_status pf_cn_rhs(pf_operator* op, pf_load* ld, const pf_vector* u_in, const pf_vector* load_now,
                    const pf_vector* load_next, double half_dt, int has_dirichlet, double dirichlet_scale,
                    pf_vector* b, pf_vector* u) {
  PF_API_BEGIN
  check_op(op);
  check_load(ld);
  pf_hierarchy* h = op->h;
  if (ld->h != h || ld->level != op->level) invalid("operator and load belong to different levels");
  check_vec(h, u_in, op->level, "u_in");
  check_vec(h, load_now, op->level, "load_now");
  check_vec(h, load_next, op->level, "load_next");
  check_vec(h, b, op->level, "b");
  if (u) check_vec(h, u, op->level, "u");
  if (b == u_in || b == load_now || b == load_next) invalid("b must not alias an input");
  PF_CUDA(cudaSetDevice(h->device));
  enq_cn_rhs(op, ld, u_in->cur(), load_now->cur(), load_next->cur(), half_dt, has_dirichlet, dirichlet_scale,
             b->cur(), u ? u->cur() : nullptr);
  sync(h);
  PF_API_END
}

pf_status pf_heat_run(pf_hierarchy* h, pf_operator* op, pf_load* ld, pf_vector* u, pf_vector* load_now,
                      int first_step, int steps, double half_dt, const double* source_scale, int has_dirichlet,
                      const double* dirichlet_scale, const pf_multigrid_config* cfg, pf_solve_stats* stats,
                      double* residuals, int max_residuals, int* failed_step) {
  PF_API_BEGIN
  if (failed_step) *failed_step = 0;
  check_level(h, h ? h->n_levels - 1 : 0);
  check_op(op);
  check_load(ld);
  const int top = h->n_levels - 1;
  if (op->h != h || ld->h != h || op->level != top || ld->level != top)
    invalid("operator and load must live on the hierarchy's finest level");
  check_vec(h, u, top, "u");
  check_vec(h, load_now, top, "load_now");
  if (!cfg || !source_scale || (has_dirichlet && !dirichlet_scale)) invalid("null argument");
  if (steps < 0 || first_step < 0) invalid("steps must be >= 0");
  PF_CUDA(cudaSetDevice(h->device));
  Level& T = h->levels[top];
  // the finest level's b scratch carries the step's rhs; one extra vector for the next load,
  // allocated once per load object (a step-by-step caller must not pay a cudaMalloc/Free,
  // which synchronises the device, every step)
  if (!ld->next) ld->next.reset(new_vector(h, top));
  pf_vector* lnx = ld->next.get();
  pf_vector* b = T.b;
  if (b == u || b == load_now) invalid("u / load_now alias the hierarchy's scratch");
  for (int k = 0; k < steps; ++k) {
    enq_load(ld, source_scale[k], lnx->cur());
    enq_cn_rhs(op, ld, u->cur(), load_now->cur(), lnx->cur(), half_dt, has_dirichlet,
               has_dirichlet ? dirichlet_scale[k] : 0.0, b->cur(), u->cur());
    try {
      solve_outer_dev(h, u, b, *cfg, stats, residuals, max_residuals);
    } catch (const pf::Error& e) {
      if (e.code == PF_ERR_NO_CONVERGENCE) {
        const int step = first_step + k + 1;
        if (failed_step) *failed_step = step;
        throw pf::Error(e.code, "time step " + std::to_string(step) + ": " + e.what());  // app.cpp:205-207
      }
      throw;
    }
    std::swap(load_now->data, lnx->data);  // load_now = std::move(load_next) (app.cpp:212)
  }
  sync(h);
  PF_API_END
}

}  // extern "C"
