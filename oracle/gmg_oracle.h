/*
 * ORACLE / TEST INFRASTRUCTURE — CPU restatement of the reference hot path.
 *
 * gmg_oracle.c restates, in plain C on host arrays in the reference's host order,
 * the functions the GPU library replaces (each function cites the reference line it
 * follows).  It takes exactly the pf_level_desc data the GPU library takes, so tests
 * feed identical bytes to both.  It is pinned against the compiled reference
 * (oracle/_ref) and the golden vectors in tests/golden/, and only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * Smoother kinds: PF_SMOOTHER_JACOBI / _GAUSS_SEIDEL / _MULTICOLOR_SOR as in pf_gpu.h
 * (Gauss-Seidel and SOR in the explicit colour order), plus ORC_SMOOTHER_LEX_GS: the
 * reference's own in-place lexicographic Gauss-Seidel (solvers.cpp:21-34).
 */
#ifndef GMG_ORACLE_H
#define GMG_ORACLE_H

#include "pf_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_SMOOTHER_LEX_GS = 3 };

typedef struct orc_hier orc_hier;

const char* orc_last_error(void);
int orc_create(int n_levels, int n_sub, orc_hier** out);
int orc_set_level(orc_hier* h, int level, int sub, const pf_level_desc* d);
int orc_finalize(orc_hier* h);
int orc_set_coarse_direct(orc_hier* h, int on);
/* Colour-wise exchange of the coloured smoothers (pf_hierarchy_set_colorwise_exchange). */
int orc_set_colorwise(orc_hier* h, int on);
void orc_destroy(orc_hier* h);
int orc_n_dofs(const orc_hier* h, int level, int sub);

/* Vectors are arrays of n_sub host pointers (one per subdomain, host order). */
int orc_spmv(orc_hier* h, int level, double* const* x, double* const* y);
int orc_cycle_residual(orc_hier* h, int level, double* const* x, double* const* b, double* const* r);
int orc_residual_norm(orc_hier* h, int level, double* const* x, double* const* b, double* out);
int orc_smooth(orc_hier* h, int level, double* const* x, double* const* b, const pf_smoother_config* c);
int orc_coarse_solve(orc_hier* h, int level, double* const* x, double* const* b, double tol,
                     int max_iter, pf_solve_stats* st);
int orc_prolongate(orc_hier* h, int fine, double* const* xc, double* const* out);
int orc_restrict_residual(orc_hier* h, int fine, double* const* r, double* const* rc);
int orc_update_master_slave(orc_hier* h, int level, double* const* v, int mode);
int orc_update_halo(orc_hier* h, int level, int kind, double* const* v);
int orc_v_cycle(orc_hier* h, double* const* x, double* const* b, const pf_multigrid_config* c,
                pf_solve_stats* st);
int orc_solve_outer(orc_hier* h, double* const* x, double* const* b, const pf_multigrid_config* c,
                    pf_solve_stats* st, double* residuals, int max_residuals);

#ifdef __cplusplus
}
#endif

#endif
