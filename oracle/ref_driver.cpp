// ORACLE / TEST INFRASTRUCTURE — not part of the product.
//
// C driver over the *unmodified* reference library (/root/reference/proj,
// compiled from its own sources by oracle/Makefile into oracle/_ref/).  Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg load it, and only as the checker or the timed CPU baseline.
//
// It drives the reference exactly the way its own tests and app do:
//   generate_unit_mesh -> partition_cells(CoordinateBisection) ->
//   build_hierarchy(PoissonStiffness) -> load + apply_dirichlet_rhs ->
//   solve_outer / smooth / v_cycle          (app.cpp:241-263,
//                                            test_multigrid.cpp:16-40)
// with the BASELINE right-hand side f = d*pi^2 * prod sin(pi x_a), g = 0
// (SURVEY.md §8d), plus the reference's own PoissonProblem and f = 1.
// Level data (CSR, classes, keys, channels, prolongation) is copied out of
// the rank threads in the reference's host order so the Python side can feed
// the same bytes to the restated oracle and to the GPU library.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "parfem/app.hpp"
#include "parfem/multigrid.hpp"
#ifdef PF_BRIDGE
// the reference-side binding of the GPU hot path (integration/parfem_gpu_bridge.hpp)
#include "parfem_gpu_bridge.hpp"
#endif

using namespace parfem;

namespace {

thread_local std::string g_err;
int g_use_gpu = 0;  // PF_BRIDGE builds: solve_outer goes through parfem::gpu::solve_outer

SolveStats outer(MultigridHierarchy& h, DistributedVector& x, const DistributedVector& b,
                 const MultigridConfig& cfg) {
#ifdef PF_BRIDGE
  if (g_use_gpu) return parfem::gpu::solve_outer(h, x, b, cfg);
#endif
  return solve_outer(h, x, b, cfg);
}

void done_with(MultigridHierarchy& h) {
#ifdef PF_BRIDGE
  if (g_use_gpu) parfem::gpu::release(h);
#endif
  (void)h;
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

const double kPi = std::acos(-1.0);

// problem 3 = HeatProblem (model.cpp:19-31) with the CN system M + dt/2 K; dt and the
// number of extra load times (t_k = k dt, k = 1..n) come from ref_set_heat.
double g_heat_dt = 0.01;
int g_heat_loads = 2;

ScalarField problem_source(int problem, int dim) {
  if (problem == 3) return HeatProblem{dim}.source();
  if (problem == 0)
    return [dim](double, const std::array<double, 3>& x) {
      double u = std::sin(kPi * x[0]) * std::sin(kPi * x[1]);
      if (dim == 3) u *= std::sin(kPi * x[2]);
      return dim * kPi * kPi * u;
    };
  if (problem == 1) return PoissonProblem{dim}.source();
  return [](double, const std::array<double, 3>&) { return 1.0; };
}

ScalarField problem_dirichlet(int problem, int dim) {
  if (problem == 1) return PoissonProblem{dim}.dirichlet();
  if (problem == 3) return HeatProblem{dim}.dirichlet();
  return [](double, const std::array<double, 3>&) { return 0.0; };
}

struct ChannelData {
  int kind, peer;
  std::vector<int> send, recv;
};

struct LevelData {
  int n_dofs = 0, n_own = 0;
  std::int64_t n_global = 0;
  std::vector<std::int64_t> row_offsets;
  std::vector<int> cols;
  std::vector<double> vals;
  std::vector<std::uint8_t> owns_row, class_of;
  std::vector<std::int64_t> keys;  // 4 per dof: kind, key[0..2]
  std::vector<std::int64_t> global_of;
  std::vector<ChannelData> channels;
  std::vector<std::int64_t> p_offsets;
  std::vector<int> p_cols;
  std::vector<double> p_w;
};

struct RankData {
  std::vector<LevelData> levels;
  std::vector<double> b, x0;  // finest
  // heat: M - dt/2 K (app.cpp:185-189) and assemble_load at t_k = k dt, k = 1..n
  std::vector<double> rhs_op;
  std::vector<std::vector<double>> loads;
};

struct Built {
  int dim, n_coarse, n_levels, K, problem;
  std::vector<RankData> ranks;
};

MultigridHierarchy build(int dim, int n_coarse, int levels, int problem, Transport& tp) {
  const MeshLevel coarse = generate_unit_mesh(dim, n_coarse);
  const PartitionMap pmap =
      partition_cells(coarse, tp.size(), PartitionStrategy::CoordinateBisection);
  HierarchyOptions opt;
  opt.n_levels = levels;
  opt.kind = problem == 3 ? SystemKind::HeatCrankNicolson : SystemKind::PoissonStiffness;
  opt.dt = g_heat_dt;
  opt.source = problem_source(problem, dim);
  opt.dirichlet = problem_dirichlet(problem, dim);
  return build_hierarchy(coarse, pmap, opt, tp);
}

// b = load with Dirichlet rhs applied; x0 = 0 except Dirichlet entries (app.cpp:253-260).
void start_vectors(const MultigridHierarchy& h, DistributedVector& x, DistributedVector& b) {
  const MultigridLevel& top = h.finest();
  b = top.load;
  apply_dirichlet_rhs(b, h.options.dirichlet, h.options.time0, *top.mapper);
  x = DistributedVector(static_cast<std::size_t>(top.mapper->n_dofs), 0.0);
  for (int i = 0; i < top.mapper->n_dofs; ++i)
    if (top.mapper->class_of[static_cast<std::size_t>(i)] == DofClass::Dirichlet)
      x[static_cast<std::size_t>(i)] = b[static_cast<std::size_t>(i)];
}

LevelData extract(const MultigridLevel& L) {
  const ParFEMapper& m = *L.mapper;
  LevelData d;
  d.n_dofs = m.n_dofs;
  d.n_own = m.n_own_dofs;
  d.n_global = m.n_global;
  d.row_offsets.assign(L.system.row_offsets.begin(), L.system.row_offsets.end());
  d.cols = L.system.col_indices;
  d.vals = L.system.values;
  d.owns_row.assign(m.owns_row.begin(), m.owns_row.end());
  for (DofClass c : m.class_of) d.class_of.push_back(static_cast<std::uint8_t>(c));
  for (const DofInfo& info : m.dofs) {
    d.keys.push_back(static_cast<std::int64_t>(info.kind));
    for (int a = 0; a < 3; ++a) d.keys.push_back(info.key[static_cast<std::size_t>(a)]);
  }
  d.global_of = m.global_of;
  for (int k = 0; k < kNumChannelKinds; ++k)
    for (const auto& [peer, ch] : m.channels[static_cast<std::size_t>(k)])
      d.channels.push_back({k, peer, ch.send_dofs, ch.recv_dofs});
  if (!L.prolong_map.empty()) {
    d.p_offsets.push_back(0);
    for (const auto& row : L.prolong_map) {
      for (const auto& [cd, w] : row) {
        d.p_cols.push_back(cd);
        d.p_w.push_back(w);
      }
      d.p_offsets.push_back(static_cast<std::int64_t>(d.p_cols.size()));
    }
  }
  return d;
}

// Deterministic value in [-1, 1) keyed by (kind, key) — the reference test
// fixture key_noise (tests/support.cpp:17-25), restated.
double key_noise(const std::int64_t* k4, std::uint64_t salt) {
  std::uint64_t h = salt * 0x9e3779b97f4a7c15ULL;
  for (int i = 0; i < 4; ++i) {
    h ^= static_cast<std::uint64_t>(k4[i]) + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
    h *= 0xbf58476d1ce4e5b9ULL;
    h ^= h >> 31;
  }
  return static_cast<double>(h >> 11) / static_cast<double>(1ULL << 52) - 1.0;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const SingularDiagonalError& e) {
    g_err = e.what();
    return 2;
  } catch (const NoConvergenceError& e) {
    g_err = e.what();
    return 3;
  } catch (const TransportError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 6;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// 1: solve_outer calls go through the GPU bridge (only in libparfem_bridge.so).
int ref_set_gpu(int on) {
#ifdef PF_BRIDGE
  g_use_gpu = on;
  return 0;
#else
  return on ? 1 : 0;
#endif
}

double ref_key_noise(const std::int64_t* k4, std::uint64_t salt) { return key_noise(k4, salt); }

// Build the reference hierarchy on K logical ranks and keep a plain copy of every
// rank's level data.  Returns NULL on failure (see ref_last_error).
void* ref_build(int dim, int n_coarse, int levels, int K, int problem) {
  Built* out = nullptr;
  const int rc = guarded([&] {
    auto b = std::make_unique<Built>();
    b->dim = dim;
    b->n_coarse = n_coarse;
    b->n_levels = levels;
    b->K = K;
    b->problem = problem;
    b->ranks = run_on_ranks_collect<RankData>(K, [&](Transport& tp) {
      MultigridHierarchy h = build(dim, n_coarse, levels, problem, tp);
      RankData rd;
      for (const MultigridLevel& L : h.levels) rd.levels.push_back(extract(L));
      if (problem == 3) {
        // heat_rank_body's start (app.cpp:173-185): rhs operator, u(0) everywhere, load(0)
        const MultigridLevel& top = h.finest();
        const ParFEMapper& m = *top.mapper;
        rd.rhs_op.resize(top.stiffness.values.size());
        for (std::size_t i = 0; i < rd.rhs_op.size(); ++i)
          rd.rhs_op[i] = top.mass.values[i] - 0.5 * g_heat_dt * top.stiffness.values[i];
        const ScalarField uex = HeatProblem{dim}.exact();
        rd.x0.resize(static_cast<std::size_t>(m.n_dofs));
        for (int i = 0; i < m.n_dofs; ++i) rd.x0[static_cast<std::size_t>(i)] = uex(0.0, m.dofs[static_cast<std::size_t>(i)].coords);
        rd.b = top.load.values;
        for (int k = 1; k <= g_heat_loads; ++k)
          rd.loads.push_back(assemble_load(m, *top.comm, h.options.source, k * g_heat_dt).values);
        return rd;
      }
      DistributedVector x, bb;
      start_vectors(h, x, bb);
      rd.b = bb.values;
      rd.x0 = x.values;
      return rd;
    });
    out = b.release();
  });
  return rc == 0 ? out : nullptr;
}

void ref_free(void* h) { delete static_cast<Built*>(h); }

// sizes: [n_dofs, n_own, nnz, p_nnz, n_channels, n_global, channel_entries]
int ref_level_sizes(void* hv, int rank, int level, std::int64_t* out) {
  const Built* h = static_cast<const Built*>(hv);
  const LevelData& d = h->ranks.at(static_cast<std::size_t>(rank)).levels.at(static_cast<std::size_t>(level));
  out[0] = d.n_dofs;
  out[1] = d.n_own;
  out[2] = static_cast<std::int64_t>(d.cols.size());
  out[3] = static_cast<std::int64_t>(d.p_cols.size());
  out[4] = static_cast<std::int64_t>(d.channels.size());
  out[5] = d.n_global;
  std::int64_t e = 0;
  for (const ChannelData& c : d.channels) e += static_cast<std::int64_t>(c.send.size() + c.recv.size());
  out[6] = e;
  return 0;
}

int ref_level_copy(void* hv, int rank, int level, std::int64_t* row_offsets, int* cols,
                   double* vals, std::uint8_t* owns_row, std::uint8_t* class_of,
                   std::int64_t* keys4, std::int64_t* global_of, std::int64_t* p_offsets,
                   int* p_cols, double* p_w) {
  const Built* h = static_cast<const Built*>(hv);
  const LevelData& d = h->ranks.at(static_cast<std::size_t>(rank)).levels.at(static_cast<std::size_t>(level));
  std::copy(d.row_offsets.begin(), d.row_offsets.end(), row_offsets);
  std::copy(d.cols.begin(), d.cols.end(), cols);
  std::copy(d.vals.begin(), d.vals.end(), vals);
  std::copy(d.owns_row.begin(), d.owns_row.end(), owns_row);
  std::copy(d.class_of.begin(), d.class_of.end(), class_of);
  std::copy(d.keys.begin(), d.keys.end(), keys4);
  std::copy(d.global_of.begin(), d.global_of.end(), global_of);
  if (p_offsets && !d.p_offsets.empty()) {
    std::copy(d.p_offsets.begin(), d.p_offsets.end(), p_offsets);
    std::copy(d.p_cols.begin(), d.p_cols.end(), p_cols);
    std::copy(d.p_w.begin(), d.p_w.end(), p_w);
  }
  return 0;
}

// Channel table: meta[4*i..] = (kind, peer, n_send, n_recv); entries = send then recv
// lists concatenated in table order.
int ref_level_channels(void* hv, int rank, int level, int* meta, int* entries) {
  const Built* h = static_cast<const Built*>(hv);
  const LevelData& d = h->ranks.at(static_cast<std::size_t>(rank)).levels.at(static_cast<std::size_t>(level));
  std::size_t e = 0;
  for (std::size_t i = 0; i < d.channels.size(); ++i) {
    const ChannelData& c = d.channels[i];
    meta[4 * i + 0] = c.kind;
    meta[4 * i + 1] = c.peer;
    meta[4 * i + 2] = static_cast<int>(c.send.size());
    meta[4 * i + 3] = static_cast<int>(c.recv.size());
    for (int v : c.send) entries[e++] = v;
    for (int v : c.recv) entries[e++] = v;
  }
  return 0;
}

void ref_set_heat(double dt, int n_loads) {
  g_heat_dt = dt;
  g_heat_loads = n_loads;
}

// heat builds: rhs operator (nnz of the finest level) and the loads, n_loads x n_dofs
int ref_heat_data(void* hv, int rank, double* rhs_op, double* loads) {
  const Built* h = static_cast<const Built*>(hv);
  const RankData& rd = h->ranks.at(static_cast<std::size_t>(rank));
  if (rd.rhs_op.empty()) {
    g_err = "not a heat build";
    return 1;
  }
  std::copy(rd.rhs_op.begin(), rd.rhs_op.end(), rhs_op);
  std::size_t at = 0;
  for (const auto& l : rd.loads) {
    std::copy(l.begin(), l.end(), loads + at);
    at += l.size();
  }
  return 0;
}

int ref_rhs(void* hv, int rank, double* b, double* x0) {
  const Built* h = static_cast<const Built*>(hv);
  const RankData& rd = h->ranks.at(static_cast<std::size_t>(rank));
  std::copy(rd.b.begin(), rd.b.end(), b);
  std::copy(rd.x0.begin(), rd.x0.end(), x0);
  return 0;
}

// Run the reference hot path on K logical ranks.
//  op 0: solve_outer from x_in (or x0)                  -> residuals, stats
//  op 1: n_ops x smooth(finest, sweeps=1)               -> x
//  op 2: n_ops x v_cycle                                -> x
//  op 3: residual_norm(finest) at x_in                  -> stats[0]
//  op 4: spmv + r = b - A x on the finest level          -> x_out holds r
// x_in / x_out: arrays of K host-order pointers (x_in may be NULL); smoother_kind
// 0 = Jacobi, 1 = Gauss-Seidel.  stats = [iterations, r0, final, solve_s(max over
// ranks), setup_s(max), converged, comm_s(max)].
int ref_run(int dim, int n_coarse, int levels, int K, int problem, int op, int n_ops,
            int smoother_kind, double damping, int pre, int post, double outer_tol,
            int max_cycles, double* const* x_in, double* const* x_out, double* residuals,
            int max_res, int* n_res, double* stats) {
  std::mutex mu;
  double solve_s = 0, setup_s = 0, comm_s = 0;
  std::vector<double> res;
  SolveStats st0;
  return guarded([&] {
    run_on_ranks(K, [&](Transport& tp) {
      const double t0 = now_s();
      MultigridHierarchy h = build(dim, n_coarse, levels, problem, tp);
      const double t1 = now_s();
      DistributedVector x, b;
      start_vectors(h, x, b);
      const std::size_t r = static_cast<std::size_t>(tp.rank());
      if (x_in && x_in[r]) std::copy(x_in[r], x_in[r] + x.size(), x.values.begin());
      MultigridConfig cfg;
      cfg.smoother.kind = smoother_kind == 0 ? SmootherKind::Jacobi : SmootherKind::GaussSeidel;
      cfg.smoother.damping = damping;
      cfg.pre_smooth = pre;
      cfg.post_smooth = post;
      cfg.outer_tol = outer_tol;
      cfg.outer_max_cycles = max_cycles;
      MultigridLevel& top = h.finest();
      SolveStats st;
      double t2 = now_s(), t3 = t2;
      const double c0 = tp.comm_seconds();
      if (op == 0) {
        barrier(tp);
        t2 = now_s();
        st = outer(h, x, b, cfg);
        t3 = now_s();
      } else if (op == 1) {
        SmootherConfig sc = cfg.smoother;
        sc.sweeps = 1;
        t2 = now_s();
        for (int i = 0; i < n_ops; ++i) smooth(top.system, x, b, sc, *top.mapper, *top.comm);
        t3 = now_s();
      } else if (op == 2) {
        t2 = now_s();
        for (int i = 0; i < n_ops; ++i) st = v_cycle(h, x, b, cfg);
        t3 = now_s();
      } else if (op == 3) {
        st.initial_residual = residual_norm(top.system, x, b, *top.mapper, tp);
      } else if (op == 4) {
        std::vector<double> y(x.size(), 0.0);
        spmv(top.system, x.values, y);
        for (std::size_t i = 0; i < y.size(); ++i) x.values[i] = b.values[i] - y[i];
      }
      const double cs = tp.comm_seconds() - c0;
      done_with(h);
      if (x_out && x_out[r]) std::copy(x.values.begin(), x.values.end(), x_out[r]);
      std::lock_guard<std::mutex> lock(mu);
      solve_s = std::max(solve_s, t3 - t2);
      setup_s = std::max(setup_s, t1 - t0);
      comm_s = std::max(comm_s, cs);
      if (r == 0) {
        st0 = st;
        res = st.residuals;
      }
    });
    int n = 0;
    for (double v : res)
      if (n < max_res) residuals[n++] = v;
    if (n_res) *n_res = n;
    stats[0] = st0.iterations;
    stats[1] = st0.initial_residual;
    stats[2] = st0.final_residual;
    stats[3] = solve_s;
    stats[4] = setup_s;
    stats[5] = st0.converged ? 1 : 0;
    stats[6] = comm_s;
  });
}

// CPU baseline: build once, then `warmup + steps` solve_outer calls from x0, each
// bracketed by a barrier; step_seconds[i] = max over ranks of step i's solve time.
int ref_bench(int dim, int n_coarse, int levels, int K, int problem, int smoother_kind,
              double damping, int pre, int post, double outer_tol, int warmup, int steps,
              double* step_seconds, double* setup_seconds, std::int64_t* n_global,
              int* iterations) {
  std::mutex mu;
  std::vector<double> per(static_cast<std::size_t>(steps), 0.0);
  double setup = 0;
  std::int64_t ng = 0;
  int its = 0;
  const int rc = guarded([&] {
    run_on_ranks(K, [&](Transport& tp) {
      const double t0 = now_s();
      MultigridHierarchy h = build(dim, n_coarse, levels, problem, tp);
      const double t1 = now_s();
      MultigridConfig cfg;
      cfg.smoother.kind = smoother_kind == 0 ? SmootherKind::Jacobi : SmootherKind::GaussSeidel;
      cfg.smoother.damping = damping;
      cfg.pre_smooth = pre;
      cfg.post_smooth = post;
      cfg.outer_tol = outer_tol;
      std::vector<double> mine(static_cast<std::size_t>(steps), 0.0);
      int it = 0;
      for (int s = 0; s < warmup + steps; ++s) {
        DistributedVector x, b;
        start_vectors(h, x, b);
        barrier(tp);
        const double a = now_s();
        const SolveStats st = outer(h, x, b, cfg);
        const double e = now_s();
        it = st.iterations;
        if (s >= warmup) mine[static_cast<std::size_t>(s - warmup)] = e - a;
      }
      done_with(h);
      std::lock_guard<std::mutex> lock(mu);
      for (int s = 0; s < steps; ++s)
        per[static_cast<std::size_t>(s)] = std::max(per[static_cast<std::size_t>(s)], mine[static_cast<std::size_t>(s)]);
      setup = std::max(setup, t1 - t0);
      ng = h.finest().mapper->n_global;
      its = it;
    });
  });
  if (rc == 0) {
    std::copy(per.begin(), per.end(), step_seconds);
    *setup_seconds = setup;
    *n_global = ng;
    *iterations = its;
  }
  return rc;
}

// Time per Crank-Nicolson step of heat_rank_body's loop (app.cpp:180-213: assemble_load,
// spmv with M - dt/2 K, Dirichlet rows, solve_outer), max over K rank threads, driven
// through the reference's own public functions; setup (build_hierarchy) excluded.
int ref_heat_bench(int dim, int n_coarse, int levels, int K, double dt, int smoother_kind, double damping,
                   int pre, int post, double outer_tol, int warmup, int steps, double* step_seconds,
                   double* setup_seconds, std::int64_t* n_global, int* iterations) {
  std::mutex mu;
  std::vector<double> per(static_cast<std::size_t>(steps), 0.0);
  double setup = 0;
  std::int64_t ng = 0;
  int its = 0;
  g_heat_dt = dt;
  const int rc = guarded([&] {
    run_on_ranks(K, [&](Transport& tp) {
      const double t0 = now_s();
      MultigridHierarchy h = build(dim, n_coarse, levels, 3, tp);
      const double t1 = now_s();
      MultigridLevel& top = h.finest();
      const ParFEMapper& mapper = *top.mapper;
      const ScalarField f = HeatProblem{dim}.source();
      const ScalarField g = HeatProblem{dim}.dirichlet();
      CsrSparseMatrix rhs_op = top.stiffness;
      for (std::size_t i = 0; i < rhs_op.values.size(); ++i)
        rhs_op.values[i] = top.mass.values[i] - 0.5 * dt * top.stiffness.values[i];
      MultigridConfig cfg;
      cfg.smoother.kind = smoother_kind == 0 ? SmootherKind::Jacobi : SmootherKind::GaussSeidel;
      cfg.smoother.damping = damping;
      cfg.pre_smooth = pre;
      cfg.post_smooth = post;
      cfg.outer_tol = outer_tol;
      const ScalarField uex = HeatProblem{dim}.exact();
      DistributedVector u(static_cast<std::size_t>(mapper.n_dofs), 0.0);
      for (int i = 0; i < mapper.n_dofs; ++i) u[static_cast<std::size_t>(i)] = uex(0.0, mapper.dofs[static_cast<std::size_t>(i)].coords);
      DistributedVector load_now = top.load;
      DistributedVector b(static_cast<std::size_t>(mapper.n_dofs), 0.0);
      std::vector<double> mine(static_cast<std::size_t>(steps), 0.0);
      int it = 0;
      for (int step = 0; step < warmup + steps; ++step) {
        const double t_next = static_cast<double>(step + 1) * dt;
        barrier(tp);
        const double a = now_s();
        DistributedVector load_next = assemble_load(mapper, *top.comm, f, t_next);
        spmv(rhs_op, u.values, b.values);
        for (std::size_t i = 0; i < b.values.size(); ++i) b[i] += 0.5 * dt * (load_now[i] + load_next[i]);
        apply_dirichlet_rhs(b, g, t_next, mapper);
        for (int i = 0; i < mapper.n_dofs; ++i)
          if (mapper.class_of[static_cast<std::size_t>(i)] == DofClass::Dirichlet)
            u[static_cast<std::size_t>(i)] = b[static_cast<std::size_t>(i)];
        const SolveStats st = outer(h, u, b, cfg);
        load_now = std::move(load_next);
        const double e = now_s();
        it = st.iterations;
        if (step >= warmup) mine[static_cast<std::size_t>(step - warmup)] = e - a;
      }
      done_with(h);
      std::lock_guard<std::mutex> lock(mu);
      for (int k = 0; k < steps; ++k)
        per[static_cast<std::size_t>(k)] = std::max(per[static_cast<std::size_t>(k)], mine[static_cast<std::size_t>(k)]);
      setup = std::max(setup, t1 - t0);
      ng = mapper.n_global;
      its = it;
    });
  });
  if (rc == 0) {
    std::copy(per.begin(), per.end(), step_seconds);
    *setup_seconds = setup;
    *n_global = ng;
    *iterations = its;
  }
  return rc;
}

// The reference's own MatrixMarket export (export_system, app.cpp:379-396): <prefix>.mtx and
// <prefix>_rhs.mtx of its PoissonProblem on K rank threads.
int ref_export(int dim, int n_coarse, int levels, int K, const char* prefix) {
  return guarded([&] {
    AppConfig cfg;
    cfg.dimension = dim;
    cfg.n_coarse = n_coarse;
    cfg.ranks = K;
    cfg.levels = levels;
    export_system(cfg, prefix);
  });
}

// The reference's own Crank-Nicolson heat run (run_heat, app.cpp:146-230,
// :299-305), unmodified: returns a handle to its SolveReport (NULL on failure).
void* ref_heat(int dim, int n_coarse, int levels, int K, double dt, double end_time, int smoother_kind,
               double damping, int pre, int post, double outer_tol) {
  SolveReport* out = nullptr;
  const int rc = guarded([&] {
    AppConfig cfg;
    cfg.dimension = dim;
    cfg.n_coarse = n_coarse;
    cfg.ranks = K;
    cfg.levels = levels;
    cfg.pre_smooth = pre;
    cfg.post_smooth = post;
    cfg.dt = dt;
    cfg.end_time = end_time;
    cfg.outer_tol = outer_tol;
    cfg.smoother = smoother_kind == 0 ? "jacobi" : "gauss_seidel";
    cfg.damping = damping;
    out = new SolveReport(run_heat(cfg));
  });
  return rc == 0 ? out : nullptr;
}

// entries of solution_by_key, residual count, errors, phases {init, assembling, solving,
// communication, total}
int ref_heat_info(void* hv, std::int64_t* n_entries, int* n_res, double* l2, double* linf, double* phases) {
  const SolveReport& r = *static_cast<SolveReport*>(hv);
  *n_entries = static_cast<std::int64_t>(r.solution_by_key.size());
  *n_res = static_cast<int>(r.cycle_residuals.size());
  *l2 = r.l2_error;
  *linf = r.linf_error;
  const PhaseTimes& p = r.metrics.phases;
  const double ph[5] = {p.initialization, p.assembling, p.solving, p.communication, p.total};
  std::copy(ph, ph + 5, phases);
  return 0;
}

int ref_heat_copy(void* hv, std::int64_t* keys, double* values, double* residuals) {
  const SolveReport& r = *static_cast<SolveReport*>(hv);
  std::size_t i = 0;
  for (const auto& [k, v] : r.solution_by_key) {
    for (int a = 0; a < 4; ++a) keys[4 * i + static_cast<std::size_t>(a)] = k[static_cast<std::size_t>(a)];
    values[i++] = v;
  }
  std::copy(r.cycle_residuals.begin(), r.cycle_residuals.end(), residuals);
  return 0;
}

void ref_heat_free(void* hv) { delete static_cast<SolveReport*>(hv); }

}  // extern "C"
