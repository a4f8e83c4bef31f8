/*
 * pf_gpu.h — C-ABI of the B200 (sm_100a) geometric-multigrid V-cycle hot path.
 *
 * This is the drop-in boundary for the data-parallel hot path of the reference
 * `parfem` library (arXiv:1609.04809 restated as /root/reference/proj).  Every
 * entry point below replaces one reference C++ function, named in its comment
 * as `file:line` relative to /root/reference/proj.  The reference keeps its own
 * mesh / partition / ParFEMapper construction; it hands each MultigridLevel to
 * pf_hierarchy_set_level() once and then calls the pf_* operations instead of
 * the CPU loops.  The C++ shim that rethrows the reference's exception types is
 * include/parfem_b200.hpp; the reference-side binding is shown in
 * INTEGRATION.md and built in integration/parfem_gpu_bridge.cpp.
 *
 * Conventions
 *  - plain pointers and sizes only; no torch / CUDA types in signatures;
 *  - every function returns a pf_status; on failure pf_last_error() returns a
 *    thread-local message.  Status codes map 1:1 onto the reference's
 *    exception hierarchy (include/parfem/errors.hpp:9-42);
 *  - "host order" means the reference's rank-local consecutive dof numbering
 *    (class-sorted, own dofs [0, n_own_dofs) first — femapper.hpp:16-25).
 *    The device keeps its own permuted layout; vectors cross the boundary in
 *    host order through pf_vector_upload / pf_vector_download;
 *  - a hierarchy holds `n_subdomains` consecutive ranks [rank_base,
 *    rank_base + n_subdomains) of a `world_size`-rank decomposition.  With one
 *    process per GPU n_subdomains = 1; several subdomains on one device are the
 *    single-GPU stand-in for several ranks (exchanges become device copies);
 *  - all arithmetic is fp64 with the reference's per-row summation order and
 *    no fused multiply-add, so damped Jacobi reproduces the reference
 *    iterate for iterate.
 */
#ifndef PF_GPU_H
#define PF_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PF_OK = 0,
  PF_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument (linalg.cpp:46-48, fecomm.cpp:18-23) */
  PF_ERR_SINGULAR_DIAGONAL = 2, /* SingularDiagonalError (solvers.cpp:10-15)                */
  PF_ERR_NO_CONVERGENCE = 3,    /* NoConvergenceError (multigrid.cpp:241-244)              */
  PF_ERR_TRANSPORT = 4,         /* TransportError (transport.cpp:49-60)                    */
  PF_ERR_CUDA = 5,              /* Error: device / driver failure                          */
  PF_ERR_STATE = 6              /* Error: API used out of order                            */
} pf_status;

/* Thread-local message of the last failing call on this thread. */
const char* pf_last_error(void);
/* Library version string and build flags (arch, compiler). */
const char* pf_version(void);
/* Number of CUDA devices visible to this process. */
pf_status pf_device_count(int* out);
/* Host threads of the library's OpenMP work (the product setup, the device-layout build):
 * n > 0 threads, n <= 0 every processor; *out (optional) = the count now in effect.  One
 * process per GPU on a shared host divides the cores (launchers such as torchrun default
 * the OpenMP thread count to 1). */
pf_status pf_set_host_threads(int n, int* out);

/* ---------------------------------------------------------------- enums -- */

/* parfem::ChannelKind (femapper.hpp:27). */
enum { PF_CH_MASTER_SLAVE = 0, PF_CH_HALO1 = 1, PF_CH_HALO2 = 2, PF_NUM_CHANNEL_KINDS = 3 };

/* parfem::UpdateMode (fecomm.hpp:28). */
enum { PF_UPDATE_SCATTER = 0, PF_UPDATE_ACCUMULATE_THEN_SCATTER = 1 };

/* parfem::SmootherKind (solvers.hpp:7) plus the B200 multicolour SOR.
 * PF_SMOOTHER_GAUSS_SEIDEL on the device is multicolour Gauss-Seidel (omega = 1)
 * in the explicit colour order given at upload. */
enum { PF_SMOOTHER_JACOBI = 0, PF_SMOOTHER_GAUSS_SEIDEL = 1, PF_SMOOTHER_MULTICOLOR_SOR = 2 };

/* ---------------------------------------------------------------- types -- */

/* One peer of one ParFECommunicator channel (femapper.hpp:38-41): the i-th entry
 * of send_dofs here and of recv_dofs on `peer` name the same carrier. */
typedef struct {
  int32_t kind;  /* PF_CH_* */
  int32_t peer;  /* global rank, != own rank */
  int32_t n_send;
  int32_t n_recv;
  const int32_t* send_dofs; /* host order */
  const int32_t* recv_dofs; /* host order */
} pf_channel_desc;

/* One rank's view of one MultigridLevel (multigrid.hpp:15-31) in host order. */
typedef struct {
  int32_t n_dofs;     /* ParFEMapper::n_dofs */
  int32_t n_own_dofs; /* ParFEMapper::n_own_dofs: rows [0, n_own) are swept and normed */
  /* level operator `system` (Dirichlet rows applied), full local CSR, n_dofs rows,
   * columns sorted ascending per row (linalg.hpp:12-22) */
  const int64_t* row_offsets; /* n_dofs + 1 */
  const int32_t* col_indices;
  const double* values;
  const uint8_t* owns_row;     /* n_dofs, ParFEMapper::owns_row            */
  const uint8_t* is_dirichlet; /* n_dofs, class_of == DofClass::Dirichlet  */
  /* colour of each own row for the coloured smoothers, or NULL: greedy colouring
   * of the own-row graph in host order */
  const int32_t* color;
  int32_t n_channels;
  const pf_channel_desc* channels;
  /* MultigridLevel::prolong_map (multigrid.cpp:35-72) as CSR over the n_dofs fine
   * rows, entries in the reference's (coarse dof, weight) order; NULL on level 0 */
  const int64_t* p_offsets;
  const int32_t* p_cols;
  const double* p_weights;
  /* optional placement hint, n_dofs entries or NULL: inside each colour the device lays
   * own rows out in ascending row_order (ties: host order), e.g. a lexicographic lattice
   * index so that a warp's 32 rows are neighbours and their column gathers coalesce.
   * Placement never changes a result (rows of one colour are independent; every
   * order-dependent sum is fixed by the host order). */
  const int64_t* row_order;
} pf_level_desc;

/* parfem::SmootherConfig (solvers.hpp:9-14). `damping` is the Jacobi damping and
 * the SOR relaxation factor; ignored for Gauss-Seidel. */
typedef struct {
  int32_t kind;
  int32_t sweeps;
  int32_t local_sweeps;
  double damping;
} pf_smoother_config;

/* parfem::MultigridConfig (multigrid.hpp:53-62). */
typedef struct {
  int32_t cycles;
  pf_smoother_config smoother;
  int32_t pre_smooth;
  int32_t post_smooth;
  double coarse_tol;
  int32_t coarse_max_iter;
  double outer_tol;
  int32_t outer_max_cycles;
} pf_multigrid_config;

/* parfem::SolveStats (linalg.hpp:37-45) minus the residual vector, which the
 * solve functions write to a caller array. */
typedef struct {
  int32_t iterations;
  int32_t converged;
  double initial_residual;
  double final_residual;
  double solve_seconds;
  double comm_seconds;
} pf_solve_stats;

typedef struct pf_hierarchy pf_hierarchy;
typedef struct pf_vector pf_vector;

/* One rank's finest-level load f(t, x) = s(t) * profile(x), profile = F0(pi x) F1(pi y)
 * [F2(pi z)] multiplied left to right (model.cpp:11-31), as assemble_load evaluates it
 * over the rank's own cells (assembly.cpp:60-88, :144-160).  Host order; the per-axis
 * tables make every product the reference forms available bit for bit. */
typedef struct {
  int32_t dim;
  int32_t n_cells;          /* N: cells per axis (table length) */
  int32_t n_dofs;
  const int32_t* lattice;   /* [3 * n_dofs] vertex lattice coordinates x, y, z */
  /* [n_dofs] own cells around the vertex in ascending global cell number: bits 0-3 the
   * count, cell k in bits 4+3k .. 6+3k, bit a set = the cell's low corner along axis a is
   * the vertex itself (else vertex - 1).  Rows without own cells, and Dirichlet rows,
   * have count 0 (their load is never read: apply_dirichlet_rhs overwrites it). */
  const uint32_t* cells;
  const double* factor;     /* [3][N][2]: F_a(pi * (lo_a(c) + p_k * h_a(c))) */
  const double* extent;     /* [3][N]: h_a(c) = hi - lo (volume = (h0 h1) h2) */
  const double* phi;        /* [8][8]: value of ring vertex v at Gauss point q, phi[q * 8 + v] */
  double qweight;           /* Gauss weight product: 0.25 (2D) or 0.125 (3D) */
  const double* boundary;   /* [n_dofs]: profile at the dof coordinates (read on Dirichlet rows) */
  const uint8_t* is_dirichlet;  /* [n_dofs] */
} pf_load_desc;

/* Defaults of the reference structs. */
void pf_default_smoother_config(pf_smoother_config* out);
void pf_default_multigrid_config(pf_multigrid_config* out);

/* ------------------------------------------------------------ hierarchy -- */

/* Replaces the device side of build_hierarchy (multigrid.cpp:76-119). */
pf_status pf_hierarchy_create(int device, int n_levels, int n_subdomains, int rank_base,
                              int world_size, pf_hierarchy** out);
/* Copies one rank's level data; arrays may be freed after the call. */
pf_status pf_hierarchy_set_level(pf_hierarchy* h, int level, int subdomain,
                                 const pf_level_desc* desc);
/* Uploads all levels: device layout, colour permutation, R = P^T, exchange plans.
 * Raises PF_ERR_SINGULAR_DIAGONAL for a zero or missing own-row diagonal — the check
 * smooth() repeats on every call in the reference (solvers.cpp:10-15, :57). */
pf_status pf_hierarchy_finalize(pf_hierarchy* h);
/* Direct coarse solve (BASELINE configs[0] names a "coarse direct solve"): coarse_solve on
 * level 0 becomes x_own = inv(A_oo) (b_own - A_o,rest x_rest) — the inverse of the own-own
 * block formed once on the host by Gauss-Jordan elimination with partial pivoting
 * (restated in oracle/gmg_oracle.c) — instead of the reference's Gauss-Seidel iteration to
 * coarse_tol (solvers.cpp:70-92); stats report 1 iteration.  The V-cycle iterates then
 * differ from the reference's at the coarse-tolerance level.  One subdomain in one
 * process; call after pf_hierarchy_finalize (captured solve graphs are rebuilt). */
pf_status pf_hierarchy_set_coarse_direct(pf_hierarchy* h, int on);

/* Tuning options of one hierarchy (the measured-best defaults, overridden by the PF_*
 * environment variable of the same upper-case name when the hierarchy is created; the list
 * and their meaning: DESIGN.md section 6 "Knobs").  "build" options shape the device layout
 * and must be set before pf_hierarchy_finalize (PF_ERR_STATE after); "launch" options can be
 * changed at any time (cached graphs are dropped).  Unknown names: PF_ERR_INVALID_ARGUMENT.
 * Results never depend on them: every combination is bit-identical (tests/test_gpu_variants.py). */
pf_status pf_hierarchy_set_option(pf_hierarchy* h, const char* name, int64_t value);
pf_status pf_hierarchy_get_option(const pf_hierarchy* h, const char* name, int64_t* out);
/* Space-separated "name:build|launch" list of every option (needs no GPU). */
pf_status pf_option_names(char* buf, int64_t capacity);

/* Memory checking (tests): with PF_GUARD=1 in the environment every device buffer of the
 * library is followed by a 4 KB guard zone of 0xFF bytes (NaN / -1 for a kernel reading
 * past an array), verified when the buffer is freed.  The number of guard zones found
 * overwritten so far; and a self-test that plants one write past the end of a guarded
 * buffer on `device` (*detected = 1 when the check catches it). */
pf_status pf_debug_guard_failures(int64_t* out);
pf_status pf_debug_guard_selftest(int device, int* detected);
/* Multi-process: join the NCCL communicator of `world_size` ranks (one hierarchy per
 * process).  `unique_id` is the 128-byte ncclUniqueId from pf_nccl_unique_id() on
 * rank 0, broadcast by the caller. */
pf_status pf_nccl_unique_id(void* out, int nbytes);
/* Transport self-test on the current device: a one-rank NCCL communicator, a grouped
 * send/recv to itself and an allgather through the same wrapper the exchanges use; *ok = 1
 * when the payloads arrive intact.  (Proves the dlopen'd NCCL path on a one-GPU box.) */
pf_status pf_nccl_selftest(int device, int* ok);
pf_status pf_hierarchy_init_nccl(pf_hierarchy* h, const void* unique_id, int nbytes);
/* Multi-process: level 0 (coarsest) of every rank r in [0, world_size), set before
 * pf_hierarchy_finalize.  Each GPU replays the reference's communicating coarse
 * Gauss-Seidel of all ranks on this replica after one allgather of the coarse rhs,
 * instead of one allreduce and two halo exchanges per coarse iteration; the result is
 * the same bit for bit (same sequential order, same exchange order). */
pf_status pf_hierarchy_set_coarse_replica(pf_hierarchy* h, int rank, const pf_level_desc* desc);
/* Multi-process: level `level` of every rank (levels 0..top, all ranks each, set before
 * finalize; level 0 == pf_hierarchy_set_coarse_replica).  When every replicated level is
 * small, each GPU runs the whole bottom of the V-cycle (levels 0..top) for all ranks
 * after ONE allgather of the restricted residual, instead of the per-sweep halo
 * exchanges the reference performs on those latency-bound levels; bit-identical. */
pf_status pf_hierarchy_set_replica_level(pf_hierarchy* h, int level, int rank, const pf_level_desc* desc);
/* Before finalize: run each smoothing sweep's master/slave and halo1 scatters (and the
 * halo2 scatter that follows a smoothing phase) as ONE message group instead of two or
 * three dependent ones.  Needs halo channel lists that never forward a Slave-held value
 * (pf_setup_options.direct_halos; checked at finalize, PF_ERR_INVALID_ARGUMENT otherwise).
 * Must be set identically on every rank.  Results are unchanged bit for bit. */
pf_status pf_hierarchy_set_fused_exchanges(pf_hierarchy* h, int on);
/* Coloured smoothers (Gauss-Seidel / SOR) on several subdomains: run the master/slave and
 * halo1 scatters after EVERY colour instead of once per sweep (solvers.cpp:56-68), so a
 * K-subdomain coloured sweep relaxes like the single-domain coloured sweep for any K (the
 * processor-local sweep of the reference lags the copies by one sweep, which makes
 * over-relaxed SOR diverge on the rotated-Q1 lognormal operator at K = 8).  Off by
 * default (reference semantics).  Must be set identically on every rank; restated in
 * oracle/gmg_oracle.c (orc_set_colorwise). */
pf_status pf_hierarchy_set_colorwise_exchange(pf_hierarchy* h, int on);
pf_status pf_hierarchy_destroy(pf_hierarchy* h);

/* Single-GPU test bench of the multi-process path: `world_size` single-subdomain
 * hierarchies on one device, each driven by its own host thread, exchange through a
 * shared loopback hub (device copies ordered by CUDA events) instead of NCCL.  Every
 * pack / unpack / accumulate / allgather / replicated-coarse code path is the one NCCL
 * runs; only the transport differs.  A rank that never reaches an exchange raises
 * PF_ERR_TRANSPORT after the watchdog (transport.cpp:44-65 semantics). */
pf_status pf_loopback_create(int world_size, void** hub);
pf_status pf_loopback_destroy(void* hub);
pf_status pf_hierarchy_init_loopback(pf_hierarchy* h, void* hub);

/* Peer-memory transport (NVLink / NVSwitch P2P over CUDA IPC, several processes on one
 * GPU, or several hierarchies of one process): every exchange of the V-cycle — the
 * master/slave and halo scatters, the master accumulate, the allgathers of the norm and of
 * the replicated coarse levels — becomes ONE kernel that stores the values straight into
 * the receiving rank's memory and synchronises through per-pair sequence flags there
 * (replaces Transport send/recv, transport.cpp:92-104, under fecomm.cpp:25-62, and the
 * allgather of allreduce_sum, transport.cpp:139-165).  Capturable: solve_outer records the
 * exchanges into its CUDA graph.  Setup, collective over the ranks, after finalize:
 *   1. pf_hierarchy_peer_export(h, NULL, 0, &n) sizes this rank's blob (allocating the
 *      peer-visible arena); pf_hierarchy_peer_export(h, buf, n, &n) writes it;
 *   2. the caller allgathers the blobs (any host fabric), each padded to a common stride;
 *   3. pf_hierarchy_init_peer(h, blobs, stride) maps every peer's arena and activates.
 * Every rank must pass the same hierarchy shape (levels, fused exchanges, replicas).
 * Ranks that are hierarchies of ONE process share its device context: finish every
 * allocation and device-synchronising call on all of them (a host barrier) before the first
 * exchange, since an exchange kernel waiting for a peer is work such a call would wait for.
 * A wait that exceeds PF_WATCHDOG_S (default 120 s) raises PF_ERR_TRANSPORT at the next
 * synchronisation (the reference fabric's watchdog, transport.cpp:54-60). */
pf_status pf_hierarchy_peer_export(pf_hierarchy* h, void* blob, int64_t capacity, int64_t* size);
pf_status pf_hierarchy_init_peer(pf_hierarchy* h, const void* blobs, int64_t stride);
/* Detach the hierarchy's transport (NCCL, loopback or peer; captured graphs are dropped) so
 * another can be attached — e.g. NCCL when peer mapping fails on some rank.  Collective in
 * effect: every rank must switch together. */
pf_status pf_hierarchy_drop_transport(pf_hierarchy* h);
/* CUDA graphs the hierarchy has captured and cached (solve graphs, outer-cycle graphs). */
pf_status pf_hierarchy_graph_count(const pf_hierarchy* h, int64_t* out);

/* Device bytes held by the hierarchy (matrices, transfers, plans, scratch). */
pf_status pf_hierarchy_device_bytes(const pf_hierarchy* h, int64_t* out);

/* -------------------------------------------------------------- vectors -- */

/* DistributedVector (fecomm.hpp:16-26) on one level: one device array per subdomain. */
pf_status pf_vector_create(pf_hierarchy* h, int level, pf_vector** out);
pf_status pf_vector_destroy(pf_vector* v);
/* Host order in/out.  Pinned host memory (pf_host_alloc) makes these asynchronous-
 * fast; pageable memory works but is staged. */
pf_status pf_vector_upload(pf_vector* v, int subdomain, const double* host, int64_t n);
pf_status pf_vector_download(const pf_vector* v, int subdomain, double* host, int64_t n);
pf_status pf_vector_fill(pf_vector* v, double value);
/* dst = src (same level), on the device. */
pf_status pf_vector_copy(const pf_vector* src, pf_vector* dst);
pf_status pf_host_alloc(void** out, int64_t bytes);
pf_status pf_host_free(void* p);

/* ------------------------------------------------------------ operations -- */

/* spmv (linalg.cpp:45-57): y = A x on every local row. */
pf_status pf_spmv(pf_hierarchy* h, int level, const pf_vector* x, pf_vector* y);

/* residual_norm (linalg.cpp:59-74): sqrt of the ascending-rank sum of per-rank
 * sum_{r < n_own} (b_r - A_r x)^2. */
pf_status pf_residual_norm(pf_hierarchy* h, int level, const pf_vector* x, const pf_vector* b,
                           double* out);

/* smooth (solvers.cpp:56-68): `sweeps` x [local_sweeps x sweep on own rows, then
 * update_master_slave(Scatter) and update_halo1]. */
pf_status pf_smooth(pf_hierarchy* h, int level, pf_vector* x, const pf_vector* b,
                    const pf_smoother_config* cfg);

/* coarse_solve (solvers.cpp:70-92): Gauss-Seidel + residual_norm until
 * <= tol * r0 or max_iter; non-convergence is reported in stats, not raised. */
pf_status pf_coarse_solve(pf_hierarchy* h, int level, pf_vector* x, const pf_vector* b,
                          double tol, int max_iter, pf_solve_stats* stats);

/* prolongate (multigrid.cpp:121-129): out = P xc on every local fine dof. */
pf_status pf_prolongate(pf_hierarchy* h, int fine_level, const pf_vector* coarse, pf_vector* out);

/* restrict_residual (multigrid.cpp:131-146): rc = P^T r over owns_row fine rows,
 * then update_master_slave(AccumulateThenScatter) on the coarse level. */
pf_status pf_restrict_residual(pf_hierarchy* h, int fine_level, const pf_vector* r, pf_vector* rc);

/* ParFECommunicator (fecomm.cpp:41-72). */
pf_status pf_update_master_slave(pf_hierarchy* h, int level, pf_vector* v, int mode);
pf_status pf_update_halo1(pf_hierarchy* h, int level, pf_vector* v);
pf_status pf_update_halo2(pf_hierarchy* h, int level, pf_vector* v);

/* allreduce_sum(Transport&, double) (transport.cpp:139-165): one value per local
 * subdomain in, ascending-rank sum out (identical on every rank). */
pf_status pf_allreduce_sum(pf_hierarchy* h, const double* per_subdomain, double* out);

/* v_cycle (multigrid.cpp:194-208) on the finest level; stats = coarse-solve stats. */
pf_status pf_v_cycle(pf_hierarchy* h, pf_vector* x, const pf_vector* b,
                     const pf_multigrid_config* cfg, pf_solve_stats* stats);

/* solve_outer (multigrid.cpp:210-246).  residuals[i] = residual after outer cycle i+1
 * (at most max_residuals written).  Returns PF_ERR_NO_CONVERGENCE after
 * outer_max_cycles, with stats filled. */
pf_status pf_solve_outer(pf_hierarchy* h, pf_vector* x, const pf_vector* b,
                         const pf_multigrid_config* cfg, pf_solve_stats* stats,
                         double* residuals, int max_residuals);

/* End-to-end solve_outer from host memory: per local subdomain s, x_host[s] (in: start
 * vector, out: solution) and b_host[s], host order.  Host->device copies, the solve and
 * the device->host copy all happen inside this call. */
pf_status pf_solve_outer_host(pf_hierarchy* h, double* const* x_host, const double* const* b_host,
                              const pf_multigrid_config* cfg, pf_solve_stats* stats,
                              double* residuals, int max_residuals);

/* ----------------------------------------------------------- device assembly -- */
/* The finest level's Q1 stiffness system assembled on the device (assemble_system +
 * apply_dirichlet_rows, assembly.cpp:103-142, :162-170): each
 * stored entry (p, q) sums, over the rank's local cells containing both vertices in
 * ascending global cell number, kappa_c * K_e(c)[slot p][slot q]; Dirichlet rows become
 * identity.  Same products and order as the host assembly, so the values are identical. */
typedef struct {
  int32_t dim;
  int32_t n_cells;             /* N: cells per axis */
  int32_t n_dofs;
  int32_t n_coarse;            /* for the global cell number (gcn) */
  int32_t level;               /* refinement level of this grid (N = n_coarse 2^level) */
  const int32_t* lattice;      /* [3 * n_dofs] */
  const uint8_t* cell_mask;    /* [n_dofs] bit k: cell with low corner = vertex along axis a
                                * iff bit a of k, is local to the rank */
  const uint8_t* is_dirichlet; /* [n_dofs] */
  const double* kappa;         /* [N^d] per cell, lexicographic, or NULL (kappa = 1) */
  const double* elem;          /* [n_classes^d][8][8] element stiffness per extent class */
  const int32_t* elem_class;   /* [3][N] extent class of each cell index along each axis */
  int32_t n_classes;
} pf_assembly_desc;

typedef struct pf_operator pf_operator;
typedef struct pf_assembly pf_assembly;
pf_status pf_assembly_create(pf_hierarchy* h, int level, pf_assembly** out);
pf_status pf_assembly_set(pf_assembly* a, int subdomain, const pf_assembly_desc* desc);
/* Assemble into `op` (a value set on the level's pattern, pf_operator_create). */
pf_status pf_assemble_operator(pf_assembly* a, pf_operator* op);
pf_status pf_assembly_destroy(pf_assembly* a);
/* An operator's values of one subdomain, in the CSR entry order of its level desc. */
pf_status pf_operator_get_values(const pf_operator* op, int subdomain, double* values, int64_t nnz);

/* ----------------------------------------------------- heat (Crank-Nicolson) -- */
/* The reference's heat run (heat_rank_body, app.cpp:146-230) on the
 * device.  Per time step t_{k+1}:
 *   load_next = assemble_load(f, t_{k+1})                 assembly.cpp:144-160
 *   b = (M - dt/2 K) u + dt/2 (load_now + load_next)      app.cpp:191-194
 *   b_D = g(t_{k+1}), u_D = b_D                           app.cpp:195-200
 *   solve_outer(h, u, b)                                  app.cpp:202-209
 * Scalars that involve exp() are computed by the caller with the host libm (the
 * reference's), so each device product equals the reference's. */

typedef struct pf_operator pf_operator;
/* A second matrix on the sparsity pattern of `level` (all local subdomains), e.g. the CN
 * right-hand-side operator M - dt/2 K (app.cpp:185-189). */
pf_status pf_operator_create(pf_hierarchy* h, int level, pf_operator** out);
/* Values of one subdomain in the CSR entry order of its pf_level_desc. */
pf_status pf_operator_set_values(pf_operator* op, int subdomain, const double* values, int64_t nnz);
/* spmv (linalg.cpp:45-57) with this operator: y = Op x on every local row. */
pf_status pf_operator_apply(pf_operator* op, const pf_vector* x, pf_vector* y);
pf_status pf_operator_destroy(pf_operator* op);

typedef struct pf_load pf_load;
pf_status pf_load_create(pf_hierarchy* h, int level, pf_load** out);
pf_status pf_load_set(pf_load* ld, int subdomain, const pf_load_desc* desc);
/* assemble_load (assembly.cpp:144-160) with f = source_scale * profile: own-cell Gauss
 * quadrature per dof, then update_master_slave(AccumulateThenScatter). */
pf_status pf_load_assemble(pf_load* ld, double source_scale, pf_vector* out);
/* apply_dirichlet_rhs (assembly.cpp:172-179) with g = dirichlet_scale * profile
 * (has_dirichlet = 0: g = 0); with u != NULL also u_D = b_D (app.cpp:196-200). */
pf_status pf_load_apply_dirichlet(pf_load* ld, int has_dirichlet, double dirichlet_scale, pf_vector* b,
                                  pf_vector* u);
pf_status pf_load_destroy(pf_load* ld);

/* b = Op u + half_dt (load_now + load_next) on every local row, then the Dirichlet rows
 * of b and u as pf_load_apply_dirichlet (app.cpp:191-200); one pass over the matrix. */
pf_status pf_cn_rhs(pf_operator* op, pf_load* ld, const pf_vector* u_in, const pf_vector* load_now,
                    const pf_vector* load_next, double half_dt, int has_dirichlet, double dirichlet_scale,
                    pf_vector* b, pf_vector* u);

/* The whole loop (app.cpp:180-213): steps first_step+1 .. first_step+steps from u (in:
 * u(t_first), out: u(t_last)); load_now in: load(t_first), out: load(t_last).
 * source_scale[k] / dirichlet_scale[k] belong to step first_step+k+1.  stats / residuals:
 * the last step's solve.  A step that does not converge returns PF_ERR_NO_CONVERGENCE
 * with *failed_step = its 1-based index (app.cpp:205-207). */
pf_status pf_heat_run(pf_hierarchy* h, pf_operator* op, pf_load* ld, pf_vector* u, pf_vector* load_now,
                      int first_step, int steps, double half_dt, const double* source_scale, int has_dirichlet,
                      const double* dirichlet_scale, const pf_multigrid_config* cfg,
                      pf_solve_stats* stats, double* residuals, int max_residuals, int* failed_step);

/* ------------------------------------------------------------- profiling -- */

/* Number of this library's kernels launched since the last reset (graph nodes
 * count once per graph launch). */
pf_status pf_launch_count(const pf_hierarchy* h, int64_t* out);
pf_status pf_reset_launch_count(pf_hierarchy* h);

/* Times `iters` back-to-back launches of one smoother sweep of `kind` on `level`
 * (subdomain 0) with CUDA events on the library stream; writes the mean kernel time
 * in milliseconds and the algorithmic bytes one sweep moves. */
pf_status pf_time_sweep(pf_hierarchy* h, int level, int kind, int iters, double* mean_ms,
                        double* algorithmic_bytes);

/* Mean time of one full V-cycle (graph replay) over `iters` cycles, CUDA events. */
pf_status pf_time_vcycle(pf_hierarchy* h, pf_vector* x, const pf_vector* b,
                         const pf_multigrid_config* cfg, int iters, double* mean_ms);

/* The cudaStream_t (as void*) every operation of this hierarchy is issued on, so a
 * caller can bracket work with its own CUDA events on the right stream. */
pf_status pf_hierarchy_stream(const pf_hierarchy* h, void** stream);

/* Level geometry as uploaded (for diagnostics and tests). */
pf_status pf_level_info(const pf_hierarchy* h, int level, int subdomain, int64_t* n_dofs,
                        int64_t* n_own, int64_t* nnz, int64_t* n_colors);

#ifdef __cplusplus
}
#endif

#endif /* PF_GPU_H */
