// parfem_b200.hpp — header-only C++ shim over the C ABI (pf_gpu.h, pf_setup.h).
//
// Mirrors the reference's multigrid / linear-algebra / communicator API
// (/root/reference/proj/include/parfem/{multigrid,solvers,linalg,fecomm}.hpp): same names,
// same argument meaning, and the reference's exception types re-thrown from pf_status
// codes (errors.hpp:9-42).  Device data lives in Hierarchy / DeviceVector; host vectors
// cross in the reference's host order.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "pf_gpu.h"
#include "pf_setup.h"

namespace parfem_b200 {

struct Error : std::runtime_error {
  explicit Error(const std::string& w) : std::runtime_error(w) {}
};
struct TransportError : Error {
  using Error::Error;
};
struct SingularDiagonalError : Error {
  using Error::Error;
};
struct NoConvergenceError : Error {
  using Error::Error;
};

inline void check(pf_status s) {
  if (s == PF_OK) return;
  const std::string m = pf_last_error();
  switch (s) {
    case PF_ERR_INVALID_ARGUMENT: throw std::invalid_argument(m);
    case PF_ERR_SINGULAR_DIAGONAL: throw SingularDiagonalError(m);
    case PF_ERR_NO_CONVERGENCE: throw NoConvergenceError(m);
    case PF_ERR_TRANSPORT: throw TransportError(m);
    default: throw Error(m);
  }
}

enum class SmootherKind { Jacobi = PF_SMOOTHER_JACOBI, GaussSeidel = PF_SMOOTHER_GAUSS_SEIDEL,
                          MulticolorSor = PF_SMOOTHER_MULTICOLOR_SOR };
enum class UpdateMode { Scatter = PF_UPDATE_SCATTER, AccumulateThenScatter = PF_UPDATE_ACCUMULATE_THEN_SCATTER };

// solvers.hpp:9-14
struct SmootherConfig {
  SmootherKind kind = SmootherKind::GaussSeidel;
  int sweeps = 3;
  int local_sweeps = 1;
  double damping = 0.8;
  pf_smoother_config c() const { return {static_cast<int32_t>(kind), sweeps, local_sweeps, damping}; }
};

// multigrid.hpp:53-62
struct MultigridConfig {
  int cycles = 1;
  SmootherConfig smoother;
  int pre_smooth = 3;
  int post_smooth = 3;
  double coarse_tol = 1e-12;
  int coarse_max_iter = 20000;
  double outer_tol = 1e-9;
  int outer_max_cycles = 100;
  pf_multigrid_config c() const {
    return {cycles, smoother.c(), pre_smooth, post_smooth, coarse_tol, coarse_max_iter, outer_tol,
            outer_max_cycles};
  }
};

// linalg.hpp:37-45
struct SolveStats {
  int iterations = 0;
  double initial_residual = 0;
  double final_residual = 0;
  bool converged = true;
  std::vector<double> residuals;
  double solve_seconds = 0;
  double comm_seconds = 0;
};

class Hierarchy;

// DistributedVector (fecomm.hpp:16-26) on the device.
class DeviceVector {
 public:
  DeviceVector(Hierarchy& h, int level);
  DeviceVector(const DeviceVector&) = delete;
  DeviceVector& operator=(const DeviceVector&) = delete;
  ~DeviceVector() { pf_vector_destroy(v_); }
  void upload(const std::vector<double>& host, int subdomain = 0) {
    check(pf_vector_upload(v_, subdomain, host.data(), static_cast<int64_t>(host.size())));
  }
  void download(std::vector<double>& host, int subdomain = 0) const {
    check(pf_vector_download(v_, subdomain, host.data(), static_cast<int64_t>(host.size())));
  }
  pf_vector* raw() const { return v_; }
  int level() const { return level_; }

 private:
  pf_vector* v_ = nullptr;
  int level_ = 0;
};

// MultigridHierarchy (multigrid.hpp:43-51) on the device.
class Hierarchy {
 public:
  Hierarchy(int device, int n_levels, int n_subdomains = 1, int rank_base = 0, int world_size = 1) {
    check(pf_hierarchy_create(device, n_levels, n_subdomains, rank_base, world_size, &h_));
    n_levels_ = n_levels;
  }
  Hierarchy(const Hierarchy&) = delete;
  Hierarchy& operator=(const Hierarchy&) = delete;
  ~Hierarchy() { pf_hierarchy_destroy(h_); }
  void set_level(int level, int subdomain, const pf_level_desc& d) {
    check(pf_hierarchy_set_level(h_, level, subdomain, &d));
  }
  void set_coarse_replica(int rank, const pf_level_desc& d) {
    check(pf_hierarchy_set_coarse_replica(h_, rank, &d));
  }
  void finalize() { check(pf_hierarchy_finalize(h_)); }
  void init_nccl(const void* unique_id, int nbytes) { check(pf_hierarchy_init_nccl(h_, unique_id, nbytes)); }
  void init_loopback(void* hub) { check(pf_hierarchy_init_loopback(h_, hub)); }
  int finest() const { return n_levels_ - 1; }
  pf_hierarchy* raw() const { return h_; }

 private:
  pf_hierarchy* h_ = nullptr;
  int n_levels_ = 0;
};

inline DeviceVector::DeviceVector(Hierarchy& h, int level) : level_(level) {
  check(pf_vector_create(h.raw(), level, &v_));
}

// linalg.cpp:45-74
inline void spmv(Hierarchy& h, int level, const DeviceVector& x, DeviceVector& y) {
  check(pf_spmv(h.raw(), level, x.raw(), y.raw()));
}
inline double residual_norm(Hierarchy& h, int level, const DeviceVector& x, const DeviceVector& b) {
  double out = 0;
  check(pf_residual_norm(h.raw(), level, x.raw(), b.raw(), &out));
  return out;
}
// solvers.cpp:56-92
inline void smooth(Hierarchy& h, int level, DeviceVector& x, const DeviceVector& b, const SmootherConfig& cfg) {
  const pf_smoother_config c = cfg.c();
  check(pf_smooth(h.raw(), level, x.raw(), b.raw(), &c));
}
inline SolveStats coarse_solve(Hierarchy& h, int level, DeviceVector& x, const DeviceVector& b, double tol,
                               int max_iter) {
  pf_solve_stats s{};
  check(pf_coarse_solve(h.raw(), level, x.raw(), b.raw(), tol, max_iter, &s));
  return SolveStats{s.iterations, s.initial_residual, s.final_residual, s.converged != 0, {}, s.solve_seconds,
                    s.comm_seconds};
}
// multigrid.cpp:121-146
inline void prolongate(Hierarchy& h, int fine, const DeviceVector& coarse, DeviceVector& out) {
  check(pf_prolongate(h.raw(), fine, coarse.raw(), out.raw()));
}
inline void restrict_residual(Hierarchy& h, int fine, const DeviceVector& r, DeviceVector& rc) {
  check(pf_restrict_residual(h.raw(), fine, r.raw(), rc.raw()));
}
// fecomm.cpp:41-72
inline void update_master_slave(Hierarchy& h, int level, DeviceVector& v, UpdateMode mode) {
  check(pf_update_master_slave(h.raw(), level, v.raw(), static_cast<int>(mode)));
}
inline void update_halo1(Hierarchy& h, int level, DeviceVector& v) { check(pf_update_halo1(h.raw(), level, v.raw())); }
inline void update_halo2(Hierarchy& h, int level, DeviceVector& v) { check(pf_update_halo2(h.raw(), level, v.raw())); }
// multigrid.cpp:194-246
inline SolveStats v_cycle(Hierarchy& h, DeviceVector& x, const DeviceVector& b, const MultigridConfig& cfg) {
  const pf_multigrid_config c = cfg.c();
  pf_solve_stats s{};
  check(pf_v_cycle(h.raw(), x.raw(), b.raw(), &c, &s));
  return SolveStats{s.iterations, s.initial_residual, s.final_residual, s.converged != 0, {}, s.solve_seconds,
                    s.comm_seconds};
}
inline SolveStats solve_outer(Hierarchy& h, DeviceVector& x, const DeviceVector& b, const MultigridConfig& cfg) {
  const pf_multigrid_config c = cfg.c();
  pf_solve_stats s{};
  std::vector<double> res(static_cast<size_t>(cfg.outer_max_cycles > 0 ? cfg.outer_max_cycles : 1));
  const pf_status st = pf_solve_outer(h.raw(), x.raw(), b.raw(), &c, &s, res.data(), static_cast<int>(res.size()));
  if (std::getenv("PF_BRIDGE_TRACE")) std::fprintf(stderr, "[shim] pf_solve_outer -> %d, %d iterations\n", static_cast<int>(st), s.iterations);
  SolveStats out{s.iterations, s.initial_residual, s.final_residual, s.converged != 0,
                 std::vector<double>(res.begin(), res.begin() + s.iterations), s.solve_seconds, s.comm_seconds};
  check(st);
  return out;
}

}  // namespace parfem_b200
