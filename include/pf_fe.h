/*
 * pf_fe.h — hierarchies of the two element families BASELINE.json names beside Q1
 * (configs[2] and configs[3]), for one subdomain on the unit cube.
 * They feed the same V-cycle (pf_gpu.h) through the same pf_level_desc.
 *
 *   PF_FE_Q2         conforming tensor-product Q2 (27-node hexahedra, nodal dofs on the
 *                    lattice of half-cells); stiffness by 3-point Gauss; prolongation by
 *                    Q2 interpolation (1D weights 1 | 3/8, 3/4, -1/8).
 *   PF_FE_ROTATED_Q1 nonconforming rotated Q1 of Rannacher and Turek, face-mean-value
 *                    dofs, span{1, x, y, z, x^2-y^2, y^2-z^2} per cell; stiffness by
 *                    2-point Gauss (exact); a piecewise-constant coefficient per cell,
 *                    coarse coefficients the mean of the children's; prolongation = face
 *                    means of the coarse function, averaged over the two sides of a coarse
 *                    face (weights 1, 1/2, +-1/4, +-1/8), none onto Dirichlet faces.
 *
 * The reference has neither family (its assembly is Q1 only, assembly.cpp:48-142); both
 * follow its algorithmic pattern — element matrices by tensor Gauss quadrature summed in
 * ascending cell order, Dirichlet rows kept with identity values (assembly.cpp:162-170),
 * the prolongation as per-fine-dof (coarse dof, weight) lists (multigrid.cpp:35-72) —
 * and are pinned to the numpy restatement oracle/fe_restated.py (tests/test_fe_setup.py).
 *
 * Numbering (host order): own (interior) dofs first, lexicographic; then the Dirichlet
 * dofs, lexicographic.  Q2 lattice (i, j, k) in [0, 2N]^3; rotated-Q1 faces (o, a0, a1,
 * a2) with a_o in [0, N] and the two tangential indices in [0, N).  Cells are numbered
 * lexicographically, (cx * N + cy) * N + cz; the lognormal coefficient of finest cell c is
 * the counter-based exp(N(0,1)) of pf_setup.h keyed by (seed, c).
 * Colours of own rows: Q2 27 (per axis: i = 0 mod 4, i = 2 mod 4, i odd — a cell's 27
 * nodes are a clique, so 27 is the minimum); rotated Q1 6 (orientation x parity of the
 * normal index).
 */
#ifndef PF_FE_H
#define PF_FE_H

#include "pf_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { PF_FE_Q2 = 2, PF_FE_ROTATED_Q1 = 3 };
enum { PF_COEF_CONSTANT = 0, PF_COEF_LOGNORMAL = 1 };

typedef struct pf_fe_setup pf_fe_setup;

const char* pf_fe_last_error(void);

/* 3D, n_coarse^3 cells refined n_levels - 1 times, rhs f = 3 pi^2 sin(pi x) sin(pi y)
 * sin(pi z), g = 0, x0 = 0.  Q2 takes PF_COEF_CONSTANT only. */
pf_status pf_fe_setup_create(int family, int n_coarse, int n_levels, int coefficient, uint64_t seed,
                             pf_fe_setup** out);
/* One rank of a box partition: the coarse cells split by coordinate bisection (as
 * pf_setup.h), each rank's subdomain its own cells plus one cell layer.  Own entities are
 * those whose lowest-ranked owning cell is this rank's; every other local non-Dirichlet
 * entity is a Slave of its owner on the master/slave channel (no halo channels: the
 * scatter after each sweep refreshes every copy, and AccumulateThenScatter gathers the
 * restricted partial sums of every copy).  n_ranks = 1 is pf_fe_setup_create. */
pf_status pf_fe_setup_create_part(int family, int n_coarse, int n_levels, int coefficient, uint64_t seed,
                                  int n_ranks, int rank, pf_fe_setup** out);
pf_status pf_fe_setup_destroy(pf_fe_setup* s);
/* Level data (level 0 = coarsest); pointers valid until pf_fe_setup_destroy. */
pf_status pf_fe_setup_level(const pf_fe_setup* s, int level, pf_level_desc* out);
pf_status pf_fe_setup_level_keys(const pf_fe_setup* s, int level, const int64_t** keys4,
                                 const uint8_t** class_of);
/* Finest rhs, start vector and the dof values of the constant-coefficient exact solution
 * u = sin(pi x) sin(pi y) sin(pi z) (nodal values for Q2, face means for rotated Q1). */
pf_status pf_fe_setup_rhs(const pf_fe_setup* s, const double** b, const double** x0, const double** exact,
                          int64_t* n);
/* The coefficient of every finest cell (lexicographic; all 1 for PF_COEF_CONSTANT). */
pf_status pf_fe_setup_kappa(const pf_fe_setup* s, const double** kappa, int64_t* n);
pf_status pf_fe_setup_seconds(const pf_fe_setup* s, double* out);

/* Device assembly of a level's system: what the device needs to
 * recompute every stored entry of the level from the entity lattice, the level's element
 * matrix and the cell coefficient.  Hand it to pf_fe_assembly_set (pf_gpu.h's pf_assembly,
 * created on the hierarchy holding this level), then pf_assemble_operator fills a
 * pf_operator with values equal to the setup's, bit for bit. */
typedef struct {
  int32_t family;              /* PF_FE_Q2 or PF_FE_ROTATED_Q1 */
  int32_t n_cells;             /* N: cells per axis */
  int32_t n_dofs;
  const int64_t* keys4;        /* [4 * n_dofs] host order: (0 | orientation, a0, a1, a2) */
  const uint8_t* is_dirichlet; /* [n_dofs] */
  const double* elem;          /* the level's element matrix, 27 x 27 or 6 x 6, row-major */
  const double* kappa;         /* [N^3] cell coefficient (rotated Q1), or NULL (Q2: 1) */
} pf_fe_assembly_desc;
pf_status pf_fe_setup_assembly_desc(const pf_fe_setup* s, int level, pf_fe_assembly_desc* out);
pf_status pf_fe_assembly_set(pf_assembly* a, int subdomain, const pf_fe_assembly_desc* desc);

#ifdef __cplusplus
}
#endif

#endif /* PF_FE_H */
