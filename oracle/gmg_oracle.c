/*
 * ORACLE / TEST INFRASTRUCTURE — CPU restatement of the reference GMG hot path.
 *
 * Restates /root/reference/proj/src/{linalg,solvers,multigrid,fecomm,transport}.cpp for
 * K subdomains held in one process (the reference's K logical ranks), in the
 * reference's host order and with its exact expression order, compiled with
 * -ffp-contract=off so every product and sum rounds like the reference's x86-64
 * build.  See gmg_oracle.h.  Never linked into the product.
 */
#include "gmg_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* orc_last_error(void) { return g_err; }

typedef struct {
  int kind, peer, ns, nr;
  int32_t* send;
  int32_t* recv;
} OCh;

typedef struct {
  int set, n, n_own, nch, ncolors;
  int64_t* rp;
  int32_t* ci;
  double* v;
  uint8_t* owns;
  uint8_t* isdir;
  int32_t* color; /* n_own */
  OCh* ch;
  int64_t* po;
  int32_t* pc;
  double* pw;
  double *x, *b, *r; /* MultigridLevel::x, b, r (multigrid.hpp:30) */
} OLev;

struct orc_hier {
  int nl, ns;
  OLev* lev;   /* [level * ns + sub] */
  double* cinv; /* orc_set_coarse_direct: inverse of level 0's own block, or NULL */
  int colorwise; /* orc_set_colorwise */
};

static OLev* L_(orc_hier* h, int l, int s) { return &h->lev[l * h->ns + s]; }

static void* dup(const void* p, size_t bytes) {
  if (!p || bytes == 0) return calloc(1, 8);
  void* q = malloc(bytes);
  memcpy(q, p, bytes);
  return q;
}

int orc_create(int n_levels, int n_sub, orc_hier** out) {
  if (n_levels < 1 || n_sub < 1) return fail(1, "bad hierarchy shape");
  orc_hier* h = calloc(1, sizeof *h);
  h->nl = n_levels;
  h->ns = n_sub;
  h->lev = calloc((size_t)n_levels * n_sub, sizeof(OLev));
  *out = h;
  return 0;
}

void orc_destroy(orc_hier* h) {
  if (!h) return;
  free(h->cinv);
  for (int i = 0; i < h->nl * h->ns; ++i) {
    OLev* L = &h->lev[i];
    free(L->rp); free(L->ci); free(L->v); free(L->owns); free(L->isdir); free(L->color);
    for (int c = 0; c < L->nch; ++c) { free(L->ch[c].send); free(L->ch[c].recv); }
    free(L->ch); free(L->po); free(L->pc); free(L->pw); free(L->x); free(L->b); free(L->r);
  }
  free(h->lev);
  free(h);
}

int orc_n_dofs(const orc_hier* h, int level, int sub) { return h->lev[level * h->ns + sub].n; }

int orc_set_level(orc_hier* h, int level, int sub, const pf_level_desc* d) {
  OLev* L = L_(h, level, sub);
  const int n = d->n_dofs;
  const int64_t nnz = d->row_offsets[n];
  L->set = 1;
  L->n = n;
  L->n_own = d->n_own_dofs;
  L->rp = dup(d->row_offsets, sizeof(int64_t) * (n + 1));
  L->ci = dup(d->col_indices, sizeof(int32_t) * nnz);
  L->v = dup(d->values, sizeof(double) * nnz);
  L->owns = dup(d->owns_row, n);
  L->isdir = d->is_dirichlet ? dup(d->is_dirichlet, n) : calloc(n + 1, 1);
  L->color = calloc(L->n_own + 1, sizeof(int32_t));
  if (d->color) {
    memcpy(L->color, d->color, sizeof(int32_t) * L->n_own);
  } else {
    /* greedy colouring in host order: smallest colour unused by lower own neighbours */
    int* seen = calloc(64, sizeof(int));
    for (int i = 0; i < L->n_own; ++i) {
      memset(seen, 0, 64 * sizeof(int));
      for (int64_t k = L->rp[i]; k < L->rp[i + 1]; ++k)
        if (L->ci[k] < i && L->color[L->ci[k]] < 64) seen[L->color[L->ci[k]]] = 1;
      int c = 0;
      while (c < 64 && seen[c]) ++c;
      L->color[i] = c;
    }
    free(seen);
  }
  L->ncolors = 0;
  for (int i = 0; i < L->n_own; ++i)
    if (L->color[i] + 1 > L->ncolors) L->ncolors = L->color[i] + 1;
  L->nch = d->n_channels;
  L->ch = calloc(d->n_channels + 1, sizeof(OCh));
  for (int c = 0; c < d->n_channels; ++c) {
    const pf_channel_desc* s = &d->channels[c];
    L->ch[c].kind = s->kind;
    L->ch[c].peer = s->peer;
    L->ch[c].ns = s->n_send;
    L->ch[c].nr = s->n_recv;
    L->ch[c].send = dup(s->send_dofs, sizeof(int32_t) * s->n_send);
    L->ch[c].recv = dup(s->recv_dofs, sizeof(int32_t) * s->n_recv);
  }
  /* channels by (kind, peer) ascending: the reference iterates std::map<peer, Channel> */
  for (int a = 1; a < L->nch; ++a)
    for (int b = a; b > 0; --b) {
      OCh *p = &L->ch[b - 1], *q = &L->ch[b];
      if (p->kind > q->kind || (p->kind == q->kind && p->peer > q->peer)) {
        OCh t = *p; *p = *q; *q = t;
      }
    }
  if (level > 0 && d->p_offsets) {
    L->po = dup(d->p_offsets, sizeof(int64_t) * (n + 1));
    L->pc = dup(d->p_cols, sizeof(int32_t) * L->po[n]);
    L->pw = dup(d->p_weights, sizeof(double) * L->po[n]);
  }
  L->x = calloc(n + 1, sizeof(double));
  L->b = calloc(n + 1, sizeof(double));
  L->r = calloc(n + 1, sizeof(double));
  return 0;
}

int orc_finalize(orc_hier* h) {
  for (int i = 0; i < h->nl * h->ns; ++i)
    if (!h->lev[i].set) return fail(6, "level not set");
  return 0;
}

static OCh* find_ch(OLev* L, int kind, int peer) {
  for (int c = 0; c < L->nch; ++c)
    if (L->ch[c].kind == kind && L->ch[c].peer == peer) return &L->ch[c];
  return NULL;
}

/* ParFECommunicator::scatter (fecomm.cpp:25-39): every rank packs v[send_dofs] for each
 * peer from the values before the exchange, then unpacks into v[recv_dofs]. */
static int scatter(orc_hier* h, int level, int kind, double* const* v) {
  const int K = h->ns;
  double** msg = calloc((size_t)K * K, sizeof(double*));
  for (int s = 0; s < K; ++s) {
    OLev* L = L_(h, level, s);
    for (int c = 0; c < L->nch; ++c) {
      OCh* ch = &L->ch[c];
      if (ch->kind != kind || ch->ns == 0) continue;
      double* m = malloc(sizeof(double) * ch->ns);
      for (int i = 0; i < ch->ns; ++i) m[i] = v[s][ch->send[i]];
      msg[s * K + ch->peer] = m;
    }
  }
  int rc = 0;
  for (int s = 0; s < K && !rc; ++s) {
    OLev* L = L_(h, level, s);
    for (int c = 0; c < L->nch; ++c) {
      OCh* ch = &L->ch[c];
      if (ch->kind != kind || ch->nr == 0) continue;
      double* m = msg[ch->peer * K + s];
      OCh* pc = find_ch(L_(h, level, ch->peer), kind, s);
      if (!m || !pc || pc->ns != ch->nr) { rc = fail(4, "channel lists do not pair up"); break; }
      for (int i = 0; i < ch->nr; ++i) v[s][ch->recv[i]] = m[i];
    }
  }
  for (int i = 0; i < K * K; ++i) free(msg[i]);
  free(msg);
  return rc;
}

/* update_master_slave (fecomm.cpp:41-62): slaves push v[recv_dofs] to their master,
 * masters add them in ascending peer order, then scatter. */
int orc_update_master_slave(orc_hier* h, int level, double* const* v, int mode) {
  const int K = h->ns;
  if (mode == PF_UPDATE_ACCUMULATE_THEN_SCATTER) {
    double** msg = calloc((size_t)K * K, sizeof(double*));
    for (int s = 0; s < K; ++s) {
      OLev* L = L_(h, level, s);
      for (int c = 0; c < L->nch; ++c) {
        OCh* ch = &L->ch[c];
        if (ch->kind != PF_CH_MASTER_SLAVE || ch->nr == 0) continue;
        double* m = malloc(sizeof(double) * ch->nr);
        for (int i = 0; i < ch->nr; ++i) m[i] = v[s][ch->recv[i]];
        msg[s * K + ch->peer] = m;
      }
    }
    int rc = 0;
    for (int s = 0; s < K && !rc; ++s) {
      OLev* L = L_(h, level, s);
      for (int c = 0; c < L->nch; ++c) { /* channels sorted by peer: ascending order */
        OCh* ch = &L->ch[c];
        if (ch->kind != PF_CH_MASTER_SLAVE || ch->ns == 0) continue;
        double* m = msg[ch->peer * K + s];
        if (!m) { rc = fail(4, "master/slave lists do not pair up"); break; }
        for (int i = 0; i < ch->ns; ++i) v[s][ch->send[i]] += m[i];
      }
    }
    for (int i = 0; i < K * K; ++i) free(msg[i]);
    free(msg);
    if (rc) return rc;
  }
  return scatter(h, level, PF_CH_MASTER_SLAVE, v);
}

int orc_update_halo(orc_hier* h, int level, int kind, double* const* v) { return scatter(h, level, kind, v); }

/* spmv (linalg.cpp:45-57) */
int orc_spmv(orc_hier* h, int level, double* const* x, double* const* y) {
  for (int s = 0; s < h->ns; ++s) {
    OLev* L = L_(h, level, s);
    for (int r = 0; r < L->n; ++r) {
      double acc = 0.0;
      for (int64_t k = L->rp[r]; k < L->rp[r + 1]; ++k) acc += L->v[k] * x[s][L->ci[k]];
      y[s][r] = acc;
    }
  }
  return 0;
}

/* r = b - A x on every row, the cycle's residual (multigrid.cpp:166-167) */
int orc_cycle_residual(orc_hier* h, int level, double* const* x, double* const* b, double* const* r) {
  for (int s = 0; s < h->ns; ++s) {
    OLev* L = L_(h, level, s);
    for (int i = 0; i < L->n; ++i) {
      double acc = 0.0;
      for (int64_t k = L->rp[i]; k < L->rp[i + 1]; ++k) acc += L->v[k] * x[s][L->ci[k]];
      r[s][i] = b[s][i] - acc;
    }
  }
  return 0;
}

/* residual_norm (linalg.cpp:59-74) + allreduce_sum in ascending rank order
 * (transport.cpp:139-149: out = 0.0; out += v_r for r ascending) */
int orc_residual_norm(orc_hier* h, int level, double* const* x, double* const* b, double* out) {
  double total = 0.0;
  for (int s = 0; s < h->ns; ++s) {
    OLev* L = L_(h, level, s);
    double local = 0.0;
    for (int r = 0; r < L->n_own; ++r) {
      double acc = b[s][r];
      for (int64_t k = L->rp[r]; k < L->rp[r + 1]; ++k) acc -= L->v[k] * x[s][L->ci[k]];
      local += acc * acc;
    }
    total += local;
  }
  *out = sqrt(total);
  return 0;
}

static int check_diagonal(OLev* L) { /* solvers.cpp:10-15 */
  for (int r = 0; r < L->n_own; ++r) {
    double d = 0.0;
    for (int64_t k = L->rp[r]; k < L->rp[r + 1]; ++k)
      if (L->ci[k] == r) d = L->v[k];
    if (d == 0.0) return fail(2, "zero diagonal at own dof");
  }
  return 0;
}

/* one row of one_local_sweep (solvers.cpp:21-51): acc = b - sum_{c != r} a x_src */
static double offdiag(const OLev* L, int r, const double* x, double b, double* diag) {
  double acc = b;
  *diag = 0.0;
  for (int64_t k = L->rp[r]; k < L->rp[r + 1]; ++k) {
    const int c = L->ci[k];
    if (c == r) *diag = L->v[k];
    else acc -= L->v[k] * x[c];
  }
  return acc;
}

static void one_local_sweep(OLev* L, double* x, const double* b, const pf_smoother_config* c,
                            double* scratch) {
  double diag;
  if (c->kind == ORC_SMOOTHER_LEX_GS) { /* solvers.cpp:21-34 */
    for (int r = 0; r < L->n_own; ++r) {
      const double acc = offdiag(L, r, x, b[r], &diag);
      x[r] = acc / diag;
    }
  } else if (c->kind == PF_SMOOTHER_JACOBI) { /* solvers.cpp:35-51 */
    memcpy(scratch, x, sizeof(double) * L->n);
    for (int r = 0; r < L->n_own; ++r) {
      const double acc = offdiag(L, r, scratch, b[r], &diag);
      x[r] = (1.0 - c->damping) * scratch[r] + c->damping * acc / diag;
    }
  } else { /* coloured Gauss-Seidel / SOR: colours ascending, rows of a colour in host order */
    const int sor = c->kind == PF_SMOOTHER_MULTICOLOR_SOR;
    for (int col = 0; col < L->ncolors; ++col)
      for (int r = 0; r < L->n_own; ++r) {
        if (L->color[r] != col) continue;
        const double acc = offdiag(L, r, x, b[r], &diag);
        x[r] = sor ? (1.0 - c->damping) * x[r] + c->damping * acc / diag : acc / diag;
      }
  }
}

/* smooth (solvers.cpp:56-68) */
int orc_smooth(orc_hier* h, int level, double* const* x, double* const* b, const pf_smoother_config* c) {
  for (int s = 0; s < h->ns; ++s) {
    int rc = check_diagonal(L_(h, level, s));
    if (rc) return rc;
  }
  int maxn = 1;
  for (int s = 0; s < h->ns; ++s)
    if (L_(h, level, s)->n > maxn) maxn = L_(h, level, s)->n;
  double* scratch = malloc(sizeof(double) * maxn);
  int rc = 0;
  const int colorwise = h->colorwise && (c->kind == PF_SMOOTHER_GAUSS_SEIDEL || c->kind == PF_SMOOTHER_MULTICOLOR_SOR);
  int maxcol = 0;
  for (int s = 0; s < h->ns; ++s)
    if (L_(h, level, s)->ncolors > maxcol) maxcol = L_(h, level, s)->ncolors;
  for (int sweep = 0; sweep < c->sweeps && !rc; ++sweep) {
    for (int loc = 0; loc < c->local_sweeps && !rc; ++loc) {
      if (!colorwise) {
        for (int s = 0; s < h->ns; ++s) one_local_sweep(L_(h, level, s), x[s], b[s], c, scratch);
        continue;
      }
      /* colour-wise exchange (B200 option, not in the reference): every subdomain sweeps
       * colour col, then the master/slave and halo1 scatters refresh every copy, so the
       * next colour sees the values a single-domain coloured sweep would */
      const int sor = c->kind == PF_SMOOTHER_MULTICOLOR_SOR;
      for (int col = 0; col < maxcol && !rc; ++col) {
        for (int s = 0; s < h->ns; ++s) {
          OLev* L = L_(h, level, s);
          double diag;
          for (int r = 0; r < L->n_own; ++r) {
            if (L->color[r] != col) continue;
            const double acc = offdiag(L, r, x[s], b[s][r], &diag);
            x[s][r] = sor ? (1.0 - c->damping) * x[s][r] + c->damping * acc / diag : acc / diag;
          }
        }
        if (loc + 1 == c->local_sweeps && col + 1 == maxcol) break; /* the sweep's own exchange follows */
        rc = orc_update_master_slave(h, level, x, PF_UPDATE_SCATTER);
        if (!rc) rc = scatter(h, level, PF_CH_HALO1, x);
      }
    }
    if (!rc) rc = orc_update_master_slave(h, level, x, PF_UPDATE_SCATTER);
    if (!rc) rc = scatter(h, level, PF_CH_HALO1, x);
  }
  free(scratch);
  return rc;
}

/* Direct coarse solve of the B200 build (pf_hierarchy_set_coarse_direct): the inverse of
 * the own-own block by Gauss-Jordan elimination with partial pivoting (first row of
 * maximal |pivot|), pivot rows scaled by division. */
int orc_set_colorwise(orc_hier* h, int on) {
  h->colorwise = on != 0;
  return 0;
}

int orc_set_coarse_direct(orc_hier* h, int on) {
  free(h->cinv);
  h->cinv = NULL;
  if (!on) return 0;
  if (h->ns != 1) return fail(1, "direct coarse solve needs one subdomain");
  OLev* L = L_(h, 0, 0);
  const int n = L->n_own;
  double* M = calloc((size_t)n * n + 1, sizeof(double));
  double* I = calloc((size_t)n * n + 1, sizeof(double));
  for (int i = 0; i < n; ++i) {
    I[(size_t)i * n + i] = 1.0;
    for (int64_t e = L->rp[i]; e < L->rp[i + 1]; ++e)
      if (L->ci[e] < n) M[(size_t)i * n + L->ci[e]] = L->v[e];
  }
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = fabs(M[(size_t)k * n + k]);
    for (int i = k + 1; i < n; ++i)
      if (fabs(M[(size_t)i * n + k]) > best) { best = fabs(M[(size_t)i * n + k]); p = i; }
    if (best == 0.0) { free(M); free(I); return fail(2, "singular coarse matrix"); }
    if (p != k)
      for (int j = 0; j < n; ++j) {
        double t = M[(size_t)p * n + j]; M[(size_t)p * n + j] = M[(size_t)k * n + j]; M[(size_t)k * n + j] = t;
        t = I[(size_t)p * n + j]; I[(size_t)p * n + j] = I[(size_t)k * n + j]; I[(size_t)k * n + j] = t;
      }
    const double piv = M[(size_t)k * n + k];
    for (int j = 0; j < n; ++j) { M[(size_t)k * n + j] /= piv; I[(size_t)k * n + j] /= piv; }
    for (int i = 0; i < n; ++i) {
      if (i == k) continue;
      const double f = M[(size_t)i * n + k];
      if (f == 0.0) continue;
      for (int j = 0; j < n; ++j) {
        M[(size_t)i * n + j] = M[(size_t)i * n + j] - f * M[(size_t)k * n + j];
        I[(size_t)i * n + j] = I[(size_t)i * n + j] - f * I[(size_t)k * n + j];
      }
    }
  }
  free(M);
  h->cinv = I;
  return 0;
}

/* coarse_solve (solvers.cpp:70-92) with the reference's lexicographic Gauss-Seidel, or
 * the direct solve x_own = inv (b_own - A_o,rest x_rest) when set */
int orc_coarse_solve(orc_hier* h, int level, double* const* x, double* const* b, double tol, int max_iter,
                     pf_solve_stats* st) {
  pf_solve_stats s;
  memset(&s, 0, sizeof s);
  s.converged = 1;
  orc_residual_norm(h, level, x, b, &s.initial_residual);
  s.final_residual = s.initial_residual;
  if (h->cinv && level == 0 && s.initial_residual != 0.0) {
    OLev* L = L_(h, 0, 0);
    const int n = L->n_own;
    double* r = malloc(sizeof(double) * (size_t)(n + 1));
    for (int i = 0; i < n; ++i) {
      double acc = b[0][i];
      for (int64_t e = L->rp[i]; e < L->rp[i + 1]; ++e)
        if (L->ci[e] >= n) acc -= L->v[e] * x[0][L->ci[e]];
      r[i] = acc;
    }
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int j = 0; j < n; ++j) acc += h->cinv[(size_t)i * n + j] * r[j];
      x[0][i] = acc;
    }
    free(r);
    s.iterations = 1;
    orc_residual_norm(h, level, x, b, &s.final_residual);
    s.converged = s.final_residual <= tol * s.initial_residual;
  } else if (s.initial_residual != 0.0) {
    pf_smoother_config gs = {ORC_SMOOTHER_LEX_GS, 1, 1, 0.8};
    const double target = tol * s.initial_residual;
    s.converged = 0;
    while (s.iterations < max_iter) {
      int rc = orc_smooth(h, level, x, b, &gs);
      if (rc) return rc;
      ++s.iterations;
      orc_residual_norm(h, level, x, b, &s.final_residual);
      if (s.final_residual <= target) { s.converged = 1; break; }
    }
  }
  if (st) *st = s;
  return 0;
}

/* prolongate (multigrid.cpp:121-129) */
int orc_prolongate(orc_hier* h, int fine, double* const* xc, double* const* out) {
  for (int s = 0; s < h->ns; ++s) {
    OLev* F = L_(h, fine, s);
    for (int i = 0; i < F->n; ++i) {
      double acc = 0;
      for (int64_t e = F->po[i]; e < F->po[i + 1]; ++e) acc += F->pw[e] * xc[s][F->pc[e]];
      out[s][i] = acc;
    }
  }
  return 0;
}

/* restrict_residual (multigrid.cpp:131-146) */
int orc_restrict_residual(orc_hier* h, int fine, double* const* r, double* const* rc) {
  for (int s = 0; s < h->ns; ++s) {
    OLev* F = L_(h, fine, s);
    OLev* Cl = L_(h, fine - 1, s);
    memset(rc[s], 0, sizeof(double) * Cl->n);
    for (int f = 0; f < F->n; ++f) {
      if (!F->owns[f]) continue;
      const double rv = r[s][f];
      for (int64_t e = F->po[f]; e < F->po[f + 1]; ++e) rc[s][F->pc[e]] += F->pw[e] * rv;
    }
  }
  return orc_update_master_slave(h, fine - 1, rc, PF_UPDATE_ACCUMULATE_THEN_SCATTER);
}

/* cycle (multigrid.cpp:150-190) */
static int cycle(orc_hier* h, int level, double* const* x, double* const* b, const pf_multigrid_config* c,
                 pf_solve_stats* cst) {
  const int K = h->ns;
  double* xv[64];
  double* bv[64];
  double* rv[64];
  int rc;
  if (K > 64) return fail(1, "too many subdomains");
  if (level == 0) {
    rc = orc_coarse_solve(h, 0, x, b, c->coarse_tol, c->coarse_max_iter, cst);
    if (!rc) rc = scatter(h, 0, PF_CH_HALO2, x);
    return rc;
  }
  pf_smoother_config pre = c->smoother;
  pre.sweeps = c->pre_smooth;
  if ((rc = orc_smooth(h, level, x, b, &pre))) return rc;
  if ((rc = scatter(h, level, PF_CH_HALO2, x))) return rc;
  for (int s = 0; s < K; ++s) rv[s] = L_(h, level, s)->r;
  orc_cycle_residual(h, level, x, b, rv);
  for (int s = 0; s < K; ++s) {
    bv[s] = L_(h, level - 1, s)->b;
    xv[s] = L_(h, level - 1, s)->x;
  }
  if ((rc = orc_restrict_residual(h, level, rv, bv))) return rc;
  for (int s = 0; s < K; ++s) {
    OLev* Cl = L_(h, level - 1, s);
    for (int d = Cl->n_own; d < Cl->n; ++d)
      if (Cl->isdir[d]) Cl->b[d] = 0.0;
    memset(Cl->x, 0, sizeof(double) * Cl->n);
  }
  if ((rc = cycle(h, level - 1, xv, bv, c, cst))) return rc;
  for (int s = 0; s < K; ++s) {
    OLev* F = L_(h, level, s);
    for (int i = 0; i < F->n; ++i) {
      double acc = 0;
      for (int64_t e = F->po[i]; e < F->po[i + 1]; ++e) acc += F->pw[e] * xv[s][F->pc[e]];
      x[s][i] += acc;
    }
  }
  pf_smoother_config post = c->smoother;
  post.sweeps = c->post_smooth;
  if ((rc = orc_smooth(h, level, x, b, &post))) return rc;
  return scatter(h, level, PF_CH_HALO2, x);
}

/* v_cycle (multigrid.cpp:194-208) */
int orc_v_cycle(orc_hier* h, double* const* x, double* const* b, const pf_multigrid_config* c,
                pf_solve_stats* st) {
  pf_solve_stats cst;
  memset(&cst, 0, sizeof cst);
  int rc = scatter(h, h->nl - 1, PF_CH_HALO2, x);
  if (!rc) rc = cycle(h, h->nl - 1, x, b, c, &cst);
  if (st) *st = cst;
  return rc;
}

/* solve_outer (multigrid.cpp:210-246) */
int orc_solve_outer(orc_hier* h, double* const* x, double* const* b, const pf_multigrid_config* c,
                    pf_solve_stats* st, double* residuals, int max_residuals) {
  pf_solve_stats s;
  memset(&s, 0, sizeof s);
  const int top = h->nl - 1;
  orc_residual_norm(h, top, x, b, &s.initial_residual);
  const double r0 = s.initial_residual;
  s.final_residual = r0;
  s.converged = 1;
  if (r0 != 0.0) {
    s.converged = 0;
    for (int outer = 1; outer <= c->outer_max_cycles; ++outer) {
      for (int j = 0; j < c->cycles; ++j) {
        int rc = orc_v_cycle(h, x, b, c, NULL);
        if (rc) return rc;
      }
      double r;
      orc_residual_norm(h, top, x, b, &r);
      s.iterations = outer;
      if (residuals && outer <= max_residuals) residuals[outer - 1] = r;
      s.final_residual = r;
      if (r <= c->outer_tol * r0) { s.converged = 1; break; }
    }
  }
  if (st) *st = s;
  if (!s.converged) return fail(3, "multigrid stalled");
  return 0;
}
