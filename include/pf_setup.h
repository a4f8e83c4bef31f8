/*
 * pf_setup.h — structured, communication-free setup of the GMG hierarchy data that the
 * hot path consumes ("scalable setup").
 *
 * For the unit square/cube Q1 Poisson problem on n_coarse^d cells refined n_levels-1
 * times and partitioned by coordinate bisection of the coarse cells (the reference's
 * only data-parallel decomposition, partition.cpp:35-142, ownership inherited by
 * children, partition.cpp:255-265), it computes for one rank and every level exactly
 * what the reference's setup pipeline computes with std::map and a cross-rank
 * handshake:
 *   - the subdomain (own cells + one-layer halo closure)     partition.cpp:156-365
 *   - dof classes Master/Independent/Dependent1/Dependent2/Slave/Halo1/Halo2/Dirichlet,
 *     including the greedy master balance in key order     femapper.cpp:66-165
 *   - the MasterSlave / Halo1 / Halo2 channels in key order  femapper.cpp:222-351
 *   - the Q1 stiffness with Dirichlet rows set to identity   assembly.cpp:48-170
 *   - the load vector (own cells + accumulate) and rhs       assembly.cpp:144-160
 *   - the multilinear prolongation map                       multigrid.cpp:35-72
 * but from closed-form lattice rules, so each rank builds its own data (and its
 * neighbours' requests) without talking to anyone, in O(local dofs).
 *
 * The local numbering is the product's own: own dofs first in lexicographic lattice
 * order, then Slave, Halo1, Halo2, Dirichlet (each lexicographic) — the reference's
 * class-sorted layout (femapper.hpp:16-25) with a different order inside each class.
 * Own rows carry the lattice-parity colour (2^d colours) used by the coloured smoothers.
 * Results are compared with the reference per carrier key (Key4, tests/support.hpp:18-21).
 */
#ifndef PF_SETUP_H
#define PF_SETUP_H

#include "pf_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pf_setup pf_setup;

/* Problems: 0 = BASELINE (f = d pi^2 prod_a sin(pi x_a), g = 0);
 *           1 = the reference's PoissonProblem (model.cpp:33-43: sin(pi x) cos(pi y)
 *               [cos(pi z)], Dirichlet data from the exact solution);
 *           2 = f = 1, g = 0. */
/*           3 = the reference's HeatProblem (model.cpp:19-31): u = exp(-t/10) sin(pi x)
 *               cos(pi y) [cos(pi z)], f = (d pi^2 - 1/10) u; every level's system is the
 *               Crank-Nicolson matrix M + dt/2 K (multigrid.cpp:18-28). */
/*           4 = BASELINE's rhs with a piecewise-constant lognormal(0, 1) coefficient per finest
 *               cell (BASELINE configs 3-4): kappa_c = exp(z_c), z_c from a
 *               counter-based generator keyed by (seed, finest gcn); coarse element matrices
 *               are the Galerkin products of their children's.  Not in the reference. */
enum { PF_PROBLEM_BASELINE = 0, PF_PROBLEM_REFERENCE_POISSON = 1, PF_PROBLEM_UNIT_SOURCE = 2,
       PF_PROBLEM_HEAT = 3, PF_PROBLEM_LOGNORMAL = 4 };

pf_status pf_setup_create(int dim, int n_coarse, int n_levels, int n_ranks, int rank, int problem,
                          pf_setup** out);
/* All options at once.  direct_halos = 1: a Halo1/Halo2 request for a carrier that its
 * owner holds as Slave goes to the carrier's Master instead (which holds the same value
 * after the master/slave scatter), so the halo exchanges no longer depend on the
 * master/slave one; with pf_hierarchy_set_fused_exchanges() a smoothing sweep then needs
 * one message group instead of two (results unchanged bit for bit).  The channel lists
 * then differ from the reference's (which routes through the Slave). */
typedef struct {
  int32_t dim, n_coarse, n_levels, n_ranks, rank, problem;
  double dt;               /* PF_PROBLEM_HEAT */
  uint64_t seed;           /* PF_PROBLEM_LOGNORMAL */
  int32_t direct_halos;
} pf_setup_options;
pf_status pf_setup_create_opts(const pf_setup_options* opts, pf_setup** out);
/* The lognormal-coefficient problem with its seed. */
pf_status pf_setup_create_lognormal(int dim, int n_coarse, int n_levels, int n_ranks, int rank, uint64_t seed,
                                    pf_setup** out);
/* kappa of every finest cell, lexicographic (x * N + y) * Nz + z. */
pf_status pf_setup_kappa(const pf_setup* s, const double** kappa, int64_t* n);
/* Same, with the time step of the heat problem (AppConfig::dt, config.hpp:22). */
pf_status pf_setup_create_heat(int dim, int n_coarse, int n_levels, int n_ranks, int rank, double dt,
                               pf_setup** out);
pf_status pf_setup_destroy(pf_setup* s);

/* Level data in the layout pf_hierarchy_set_level takes; pointers stay valid until
 * pf_setup_destroy. level 0 = coarsest. */
pf_status pf_setup_level(const pf_setup* s, int level, pf_level_desc* out);
/* Per-dof carrier key (entity kind 0 = vertex, lattice x, y, z), 4 int64 per dof, and
 * DofClass value (femapper.hpp:16-25) per dof. */
pf_status pf_setup_level_keys(const pf_setup* s, int level, const int64_t** keys4,
                              const uint8_t** class_of);
/* Finest-level right-hand side (load with Dirichlet rhs applied) and start vector
 * (zero except Dirichlet entries = boundary data), app.cpp:253-260. */
pf_status pf_setup_rhs(const pf_setup* s, const double** b, const double** x0, int64_t* n);
/* Global dof count of the finest level ((N+1)^d) and this rank's local counts. */
pf_status pf_setup_counts(const pf_setup* s, int level, int64_t* n_global, int64_t* n_dofs,
                          int64_t* n_own, int64_t* nnz);
/* Heat: the finest-level right-hand-side operator M - dt/2 K (app.cpp:185-189), raw rows,
 * in the CSR entry order of pf_setup_level(finest). */
pf_status pf_setup_rhs_operator(const pf_setup* s, const double** values, int64_t* nnz);
/* Finest-level load at time t (assemble_load, assembly.cpp:144-160, after the master /
 * slave accumulate), host order; Dirichlet rows 0.  n must equal the finest n_dofs. */
pf_status pf_setup_load_at(const pf_setup* s, double t, double* out, int64_t n);
/* The device description of the same load (pf_load_set).  Pointers stay valid until
 * pf_setup_destroy. */
pf_status pf_setup_load_desc(const pf_setup* s, pf_load_desc* out);
/* The device assembly description of the finest level (pf_assembly_set). */
pf_status pf_setup_assembly_desc(pf_setup* s, pf_assembly_desc* out);
/* f(t) = source_scale * profile, g(t) = dirichlet_scale * profile (or 0 when
 * !has_dirichlet), evaluated with this library's libm exactly as model.cpp does. */
pf_status pf_setup_scales(const pf_setup* s, double t, double* source_scale, int32_t* has_dirichlet,
                          double* dirichlet_scale);
/* MatrixMarket export of the finest level (export_system, app.cpp:379-396, through
 * export_matrixmarket, matrix_market.cpp:47-112): setups[r] = rank r of one n_ranks
 * decomposition, all in this process.  Global numbering as assign_global_numbers
 * (femapper.cpp:353-472): own dofs rank by rank, then each rank's owned Dirichlet dofs.
 * Writes the same bytes as the reference: "%lld %lld %.17g" coordinate entries of every
 * owned row, and the rhs b as an array.  (The reference exports its PoissonProblem:
 * build the setups with PF_PROBLEM_REFERENCE_POISSON for identical files.) */
pf_status pf_setup_export_matrixmarket(const pf_setup* const* setups, int n_ranks, const char* matrix_path,
                                       const char* rhs_path, int64_t* n_global, int64_t* nnz);
/* Hands level `level` of a setup to a hierarchy (instead of pf_setup_level +
 * pf_hierarchy_set_level) by moving its arrays: no second host copy of the matrices, which
 * is what makes a 512^3 grid fit in host memory.  The setup's level descriptions are
 * unavailable afterwards (its rhs, keys and device descriptions stay). */
pf_status pf_hierarchy_set_level_from_setup(pf_hierarchy* h, int level, int subdomain, pf_setup* s);
/* Frees every level's matrices (CSR, prolongation, rhs operator) once a hierarchy holds
 * its own copy (after pf_hierarchy_set_level of every level): large grids keep only one
 * host copy alive.  pf_setup_level fails afterwards; rhs, keys and descriptions stay. */
pf_status pf_setup_release_matrices(pf_setup* s);
/* Seconds spent in pf_setup_create. */
pf_status pf_setup_seconds(const pf_setup* s, double* out);

#ifdef __cplusplus
}
#endif

#endif /* PF_SETUP_H */
