// pf_fe_setup.cpp — Q2 and rotated-Q1 (Rannacher-Turek) hierarchies for the V-cycle
// (include/pf_fe.h; BASELINE configs[2] and configs[3]).
//
// Both families follow the reference's Q1 pipeline step for step:
//   element matrices by tensor Gauss quadrature         assembly.cpp:48-88
//   global sums over the cells of an entry in ascending cell order  assembly.cpp:90-142
//   Dirichlet rows kept with identity values            assembly.cpp:162-170
//   the load by the same quadrature, own cells only     assembly.cpp:144-160
//   prolongation as (coarse dof, weight) lists per fine dof         multigrid.cpp:35-72
// and every floating-point expression is written out so that the numpy restatement
// (oracle/fe_restated.py) reproduces it bit for bit.  One subdomain; rows are built in
// parallel (each row's sums are serial, so the result does not depend on the threads).
#include "pf_fe.h"

#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pf_coef.hpp"

std::vector<int> pf_coarse_partition(int d, int n, int k);  // pf_setup.cpp

namespace {

struct FeError : std::runtime_error {
  pf_status code;
  FeError(pf_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void invalid(const std::string& m) { throw FeError(PF_ERR_INVALID_ARGUMENT, m); }

thread_local std::string g_fe_err;

const double kPi = std::acos(-1.0);
constexpr uint8_t kIndep = 1, kSlaveCls = 4, kDirichlet = 7;  // DofClass (femapper.hpp:16-25)

// Gauss-Legendre rules on [0, 1]
struct Rule {
  int n;
  double t[3], w[3];
};
Rule gauss2() {
  const double r = 0.5 / std::sqrt(3.0);
  return {2, {0.5 - r, 0.5 + r, 0.0}, {0.5, 0.5, 0.0}};
}
Rule gauss3() {
  const double r = 0.5 * std::sqrt(0.6);
  return {3, {0.5 - r, 0.5, 0.5 + r}, {5.0 / 18.0, 8.0 / 18.0, 5.0 / 18.0}};
}

}  // namespace

struct FeLevel {
  int64_t N = 0;  // cells per axis
  int32_t n = 0, n_own = 0;
  std::vector<int64_t> rowptr;
  std::vector<int32_t> cols;
  std::vector<double> vals;
  std::vector<uint8_t> owns_row, is_dir, class_of;
  std::vector<int32_t> color;
  std::vector<int64_t> order, keys;  // keys: 4 per dof
  std::vector<int64_t> p_off;
  std::vector<int32_t> p_col;
  std::vector<double> p_w;
  std::vector<double> elem, kappa;  // element matrix (h included) and cell coefficients
  struct Chan {
    int32_t peer;
    std::vector<int32_t> send, recv;
  };
  std::vector<Chan> chans;               // master/slave channels, peers ascending
  std::vector<pf_channel_desc> descs;
  // lexicographic entity index <-> host index
  std::vector<int32_t> host_of;
  std::vector<int64_t> lex_of;
};

struct pf_fe_setup {
  int family = 0, n_coarse = 2, n_levels = 1, coefficient = 0, n_ranks = 1, rank = 0;
  std::vector<int> coarse_owner;
  uint64_t seed = 0;
  std::vector<std::unique_ptr<FeLevel>> levels;
  std::vector<double> b, x0, exact, kappa;
  double seconds = 0;
};

namespace {

// One rank's view of a level: the owner of every cell (coordinate bisection of the coarse
// cells, inherited by their descendants) and, per rank, its local cells = own cells plus
// the one-cell layer around them (the reference's subdomain: partition.cpp:156-365).
struct Region {
  int64_t N = 0;
  int rank = 0, n_ranks = 1;
  std::vector<int8_t> owner;                // [N^3]
  std::vector<std::vector<uint8_t>> local;  // [rank][N^3]
  bool is_local(int64_t cell) const { return local[static_cast<size_t>(rank)][static_cast<size_t>(cell)] != 0; }
};

Region make_region(const pf_fe_setup& s, int level) {
  Region R;
  const int64_t N = static_cast<int64_t>(s.n_coarse) << level, nc = s.n_coarse;
  R.N = N;
  R.rank = s.rank;
  R.n_ranks = s.n_ranks;
  R.owner.resize(static_cast<size_t>(N * N * N));
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < N * N * N; ++c) {
    const int64_t x = c / (N * N) >> level, y = (c / N) % N >> level, z = c % N >> level;
    R.owner[static_cast<size_t>(c)] = static_cast<int8_t>(s.coarse_owner[static_cast<size_t>((x * nc + y) * nc + z)]);
  }
  R.local.assign(static_cast<size_t>(s.n_ranks), std::vector<uint8_t>(static_cast<size_t>(N * N * N), 0));
  for (int r = 0; r < s.n_ranks; ++r) {
    auto& L = R.local[static_cast<size_t>(r)];
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < N * N * N; ++c) {
      const int64_t x = c / (N * N), y = (c / N) % N, z = c % N;
      uint8_t any = 0;
      for (int64_t dx = -1; dx <= 1 && !any; ++dx)
        for (int64_t dy = -1; dy <= 1 && !any; ++dy)
          for (int64_t dz = -1; dz <= 1 && !any; ++dz) {
            const int64_t u = x + dx, v = y + dy, w = z + dz;
            if (u < 0 || v < 0 || w < 0 || u >= N || v >= N || w >= N) continue;
            if (R.owner[static_cast<size_t>((u * N + v) * N + w)] == r) any = 1;
          }
      L[static_cast<size_t>(c)] = any;
    }
  }
  return R;
}

enum : int8_t { kNotLocal = -1, kOwn = 0, kSlave = 1, kDir = 2 };

// Host order: own entities first, then slaves (owned by another rank), then Dirichlet
// ones, each lexicographic.  cls[e]: kNotLocal / kOwn / kSlave / kDir; owner[e]: the
// lowest rank whose own cells contain e.
void number(FeLevel& L, int64_t n_lex, const std::vector<int8_t>& cls, const std::vector<int8_t>& owner, int rank) {
  L.host_of.assign(static_cast<size_t>(n_lex), -1);
  int64_t cnt[3] = {0, 0, 0};
  for (int64_t e = 0; e < n_lex; ++e)
    if (cls[static_cast<size_t>(e)] >= 0) ++cnt[cls[static_cast<size_t>(e)]];
  const int64_t n = cnt[0] + cnt[1] + cnt[2];
  if (n > INT32_MAX) invalid("level too large for int32 dof indices");
  int64_t next[3] = {0, cnt[0], cnt[0] + cnt[1]};
  L.lex_of.assign(static_cast<size_t>(n), 0);
  L.n = static_cast<int32_t>(n);
  L.n_own = static_cast<int32_t>(cnt[0]);
  L.owns_row.assign(static_cast<size_t>(n), 0);
  L.is_dir.assign(static_cast<size_t>(n), 0);
  L.class_of.assign(static_cast<size_t>(n), kIndep);
  for (int64_t e = 0; e < n_lex; ++e) {
    const int8_t c = cls[static_cast<size_t>(e)];
    if (c < 0) continue;
    const int64_t h = next[c]++;
    L.host_of[static_cast<size_t>(e)] = static_cast<int32_t>(h);
    L.lex_of[static_cast<size_t>(h)] = e;
    // authoritative rows (femapper.cpp:214-217): own ones and the Dirichlet ones this rank owns
    L.owns_row[static_cast<size_t>(h)] = (c == kOwn || (c == kDir && owner[static_cast<size_t>(e)] == rank)) ? 1 : 0;
    L.is_dir[static_cast<size_t>(h)] = c == kDir ? 1 : 0;
    L.class_of[static_cast<size_t>(h)] = c == kOwn ? kIndep : c == kSlave ? kSlaveCls : kDirichlet;
  }
  L.order.assign(L.lex_of.begin(), L.lex_of.end());
}

// Classify every entity of a level and build the master/slave channels: an entity is
// local when one of its cells is; its owner is the lowest rank whose own cells contain
// it; every local non-own, non-Dirichlet copy is a Slave of its owner, refreshed by the
// master/slave scatter after each sweep (so no halo channels are needed) and accumulated
// into the owner by AccumulateThenScatter after the restriction.
template <typename CellsOf>
void classify(FeLevel& L, const Region& R, int64_t n_lex, CellsOf cells_of, const std::vector<uint8_t>& boundary) {
  std::vector<int8_t> cls(static_cast<size_t>(n_lex), kNotLocal), owner(static_cast<size_t>(n_lex), 0);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < n_lex; ++e) {
    int64_t cells[8];
    const int nc = cells_of(e, cells);
    bool local = false;
    int own = 127;
    for (int k = 0; k < nc; ++k) {
      local = local || R.is_local(cells[k]);
      own = std::min<int>(own, R.owner[static_cast<size_t>(cells[k])]);
    }
    owner[static_cast<size_t>(e)] = static_cast<int8_t>(own);
    if (!local) continue;
    cls[static_cast<size_t>(e)] = boundary[static_cast<size_t>(e)] ? kDir : own == R.rank ? kOwn : kSlave;
  }
  number(L, n_lex, cls, owner, R.rank);
  // channels: to peer p, my own entities that p holds (one of their cells is local to p);
  // from p, my slaves owned by p; both in lexicographic order, so the i-th entries match
  L.chans.clear();
  for (int p = 0; p < R.n_ranks; ++p) {
    if (p == R.rank) continue;
    FeLevel::Chan ch;
    ch.peer = p;
    const auto& lp = R.local[static_cast<size_t>(p)];
    for (int64_t h = 0; h < L.n; ++h) {
      const int64_t e = L.lex_of[static_cast<size_t>(h)];
      if (h < L.n_own) {
        int64_t cells[8];
        const int nc = cells_of(e, cells);
        for (int k = 0; k < nc; ++k)
          if (lp[static_cast<size_t>(cells[k])]) {
            ch.send.push_back(static_cast<int32_t>(h));
            break;
          }
      } else if (!L.is_dir[static_cast<size_t>(h)] && owner[static_cast<size_t>(e)] == p) {
        ch.recv.push_back(static_cast<int32_t>(h));
      }
    }
    if (!ch.send.empty() || !ch.recv.empty()) L.chans.push_back(std::move(ch));
  }
  L.descs.clear();
  for (const auto& c : L.chans)
    L.descs.push_back(pf_channel_desc{PF_CH_MASTER_SLAVE, c.peer, static_cast<int32_t>(c.send.size()),
                                      static_cast<int32_t>(c.recv.size()), c.send.data(), c.recv.data()});
}

// Rows as (column, value) lists sorted by host column; row_fn(h, out) appends a row.
template <typename RowFn>
void build_csr(FeLevel& L, RowFn row_fn) {
  const int64_t n = L.n;
  std::vector<int32_t> len(static_cast<size_t>(n), 0);
#pragma omp parallel
  {
    std::vector<std::pair<int32_t, double>> row;
#pragma omp for schedule(static)
    for (int64_t h = 0; h < n; ++h) {
      row.clear();
      row_fn(h, row, /*values=*/false);
      len[static_cast<size_t>(h)] = static_cast<int32_t>(row.size());
    }
  }
  L.rowptr.assign(static_cast<size_t>(n) + 1, 0);
  for (int64_t h = 0; h < n; ++h) L.rowptr[static_cast<size_t>(h) + 1] = L.rowptr[static_cast<size_t>(h)] + len[static_cast<size_t>(h)];
  L.cols.resize(static_cast<size_t>(L.rowptr.back()));
  L.vals.resize(static_cast<size_t>(L.rowptr.back()));
#pragma omp parallel
  {
    std::vector<std::pair<int32_t, double>> row;
#pragma omp for schedule(static)
    for (int64_t h = 0; h < n; ++h) {
      row.clear();
      row_fn(h, row, /*values=*/true);
      std::sort(row.begin(), row.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
      int64_t k = L.rowptr[static_cast<size_t>(h)];
      for (const auto& [c, v] : row) {
        L.cols[static_cast<size_t>(k)] = c;
        L.vals[static_cast<size_t>(k)] = v;
        ++k;
      }
    }
  }
}

template <typename RowFn>
void build_p(FeLevel& L, RowFn row_fn) {
  const int64_t n = L.n;
  std::vector<int32_t> len(static_cast<size_t>(n), 0);
  std::vector<std::vector<std::pair<int32_t, double>>> rows(static_cast<size_t>(omp_get_max_threads()));
#pragma omp parallel for schedule(static)
  for (int64_t h = 0; h < n; ++h) {
    auto& row = rows[static_cast<size_t>(omp_get_thread_num())];
    row.clear();
    row_fn(h, row);
    len[static_cast<size_t>(h)] = static_cast<int32_t>(row.size());
  }
  L.p_off.assign(static_cast<size_t>(n) + 1, 0);
  for (int64_t h = 0; h < n; ++h) L.p_off[static_cast<size_t>(h) + 1] = L.p_off[static_cast<size_t>(h)] + len[static_cast<size_t>(h)];
  L.p_col.resize(static_cast<size_t>(L.p_off.back()));
  L.p_w.resize(static_cast<size_t>(L.p_off.back()));
#pragma omp parallel for schedule(static)
  for (int64_t h = 0; h < n; ++h) {
    auto& row = rows[static_cast<size_t>(omp_get_thread_num())];
    row.clear();
    row_fn(h, row);
    std::sort(row.begin(), row.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    int64_t k = L.p_off[static_cast<size_t>(h)];
    for (const auto& [c, w] : row) {
      L.p_col[static_cast<size_t>(k)] = c;
      L.p_w[static_cast<size_t>(k)] = w;
      ++k;
    }
  }
}

// ------------------------------------------------------------------------ Q2 --

// 1D Q2 basis on [0, 1] (nodes 0, 1/2, 1) and its derivative
double q2_phi(int i, double t) {
  return i == 0 ? (1.0 - t) * (1.0 - 2.0 * t) : i == 1 ? (4.0 * t) * (1.0 - t) : t * (2.0 * t - 1.0);
}
double q2_dphi(int i, double t) { return i == 0 ? 4.0 * t - 3.0 : i == 1 ? 4.0 - 8.0 * t : 4.0 * t - 1.0; }

// Stiffness of the unit cube, 27 x 27, local node a = (ax * 3 + ay) * 3 + az.
std::vector<double> q2_kref() {
  const Rule g = gauss3();
  double V[3][3], D[3][3];
  for (int i = 0; i < 3; ++i)
    for (int q = 0; q < 3; ++q) {
      V[i][q] = q2_phi(i, g.t[q]);
      D[i][q] = q2_dphi(i, g.t[q]);
    }
  std::vector<double> K(27 * 27, 0.0);
  for (int a = 0; a < 27; ++a)
    for (int b = 0; b < 27; ++b) {
      const int ax = a / 9, ay = (a / 3) % 3, az = a % 3, bx = b / 9, by = (b / 3) % 3, bz = b % 3;
      double s = 0.0;
      for (int qx = 0; qx < 3; ++qx)
        for (int qy = 0; qy < 3; ++qy)
          for (int qz = 0; qz < 3; ++qz) {
            const double w = (g.w[qx] * g.w[qy]) * g.w[qz];
            const double ga0 = (D[ax][qx] * V[ay][qy]) * V[az][qz], gb0 = (D[bx][qx] * V[by][qy]) * V[bz][qz];
            const double ga1 = (V[ax][qx] * D[ay][qy]) * V[az][qz], gb1 = (V[bx][qx] * D[by][qy]) * V[bz][qz];
            const double ga2 = (V[ax][qx] * V[ay][qy]) * D[az][qz], gb2 = (V[bx][qx] * V[by][qy]) * D[bz][qz];
            s += w * ((ga0 * gb0 + ga1 * gb1) + ga2 * gb2);
          }
      K[static_cast<size_t>(a * 27 + b)] = s;
    }
  return K;
}

// cells along one axis containing node i (at most 2, ascending)
int q2_cells(int64_t i, int64_t N, int64_t* out) {
  if (i & 1) {
    out[0] = (i - 1) / 2;
    return 1;
  }
  int n = 0;
  if (i / 2 - 1 >= 0) out[n++] = i / 2 - 1;
  if (i / 2 < N) out[n++] = i / 2;
  return n;
}


// The row of entity e: the entities of its local cells, each entry summed over the local
// cells containing both entities in ascending cell order (own rows: all their cells are
// local, so the sum is the global one); Dirichlet rows keep the pattern with identity values.
void q2_level(FeLevel& L, const Region& R, const std::vector<double>& Ke) {
  const int64_t N = R.N, M = 2 * N + 1;
  L.N = N;
  auto cells_of = [N, M](int64_t e, int64_t* cells) {
    const int64_t p[3] = {e / (M * M), (e / M) % M, e % M};
    int64_t pc[3][2];
    int np[3];
    for (int t = 0; t < 3; ++t) np[t] = q2_cells(p[t], N, pc[t]);
    int n = 0;
    for (int x = 0; x < np[0]; ++x)
      for (int y = 0; y < np[1]; ++y)
        for (int z = 0; z < np[2]; ++z) cells[n++] = (pc[0][x] * N + pc[1][y]) * N + pc[2][z];
    return n;
  };
  std::vector<uint8_t> bnd(static_cast<size_t>(M * M * M));
  for (int64_t i = 0; i < M; ++i)
    for (int64_t j = 0; j < M; ++j)
      for (int64_t k = 0; k < M; ++k)
        bnd[static_cast<size_t>((i * M + j) * M + k)] =
            (i == 0 || j == 0 || k == 0 || i == M - 1 || j == M - 1 || k == M - 1) ? 1 : 0;
  classify(L, R, M * M * M, cells_of, bnd);
  L.keys.resize(static_cast<size_t>(L.n) * 4);
  L.color.resize(static_cast<size_t>(L.n_own));
  auto cls = [](int64_t i) { return (i & 1) ? 2 : ((i & 3) == 0 ? 0 : 1); };
  for (int64_t h = 0; h < L.n; ++h) {
    const int64_t e = L.lex_of[static_cast<size_t>(h)];
    const int64_t i = e / (M * M), j = (e / M) % M, k = e % M;
    int64_t* key = &L.keys[static_cast<size_t>(h) * 4];
    key[0] = 0;
    key[1] = i;
    key[2] = j;
    key[3] = k;
    if (h < L.n_own) L.color[static_cast<size_t>(h)] = (cls(i) * 3 + cls(j)) * 3 + cls(k);
  }
  build_csr(L, [&](int64_t h, std::vector<std::pair<int32_t, double>>& row, bool values) {
    const int64_t e = L.lex_of[static_cast<size_t>(h)];
    const int64_t p[3] = {e / (M * M), (e / M) % M, e % M};
    int64_t cells[8];
    const int nall = cells_of(e, cells);
    int nc = 0;
    for (int k = 0; k < nall; ++k)
      if (R.is_local(cells[k])) cells[nc++] = cells[k];
    if (h < L.n_own && nc != nall) invalid("own row with a non-local cell");
    const bool dir = L.is_dir[static_cast<size_t>(h)] != 0;
    // the nodes of the local cells, each once, lexicographic
    int64_t cand[216];
    int nn = 0;
    for (int k = 0; k < nc; ++k) {
      const int64_t cx = cells[k] / (N * N), cy = (cells[k] / N) % N, cz = cells[k] % N;
      for (int q = 0; q < 27; ++q)
        cand[nn++] = ((2 * cx + q / 9) * M + 2 * cy + (q / 3) % 3) * M + 2 * cz + q % 3;
    }
    std::sort(cand, cand + nn);
    nn = static_cast<int>(std::unique(cand, cand + nn) - cand);
    for (int u = 0; u < nn; ++u) {
      const int64_t f = cand[u];
      const int32_t col = L.host_of[static_cast<size_t>(f)];
      double v = 0.0;
      if (values) {
        if (dir) {
          v = col == h ? 1.0 : 0.0;
        } else {
          const int64_t q[3] = {f / (M * M), (f / M) % M, f % M};
          for (int k = 0; k < nc; ++k) {
            const int64_t cc[3] = {cells[k] / (N * N), (cells[k] / N) % N, cells[k] % N};
            bool in = true;
            for (int t = 0; t < 3; ++t) in = in && q[t] >= 2 * cc[t] && q[t] <= 2 * cc[t] + 2;
            if (!in) continue;
            const int la = static_cast<int>(((p[0] - 2 * cc[0]) * 3 + (p[1] - 2 * cc[1])) * 3 + (p[2] - 2 * cc[2]));
            const int lb = static_cast<int>(((q[0] - 2 * cc[0]) * 3 + (q[1] - 2 * cc[1])) * 3 + (q[2] - 2 * cc[2]));
            v += Ke[static_cast<size_t>(la * 27 + lb)];
          }
        }
      }
      row.emplace_back(col, v);
    }
  });
}

// (coarse index, weight) of fine node i along one axis
int q2_pw(int64_t i, int64_t* c, double* w) {
  if ((i & 1) == 0) {
    c[0] = i / 2;
    w[0] = 1.0;
    return 1;
  }
  const int64_t cell = i / 4;
  const bool first = (i & 3) == 1;
  c[0] = 2 * cell;
  c[1] = 2 * cell + 1;
  c[2] = 2 * cell + 2;
  w[0] = first ? 0.375 : -0.125;
  w[1] = 0.75;
  w[2] = first ? -0.125 : 0.375;
  return 3;
}

void q2_prolongation(FeLevel& F, const FeLevel& Cl) {
  const int64_t Mf = 2 * F.N + 1, Mc = 2 * Cl.N + 1;
  build_p(F, [&](int64_t h, std::vector<std::pair<int32_t, double>>& row) {
    const int64_t e = F.lex_of[static_cast<size_t>(h)];
    const int64_t p[3] = {e / (Mf * Mf), (e / Mf) % Mf, e % Mf};
    int64_t c[3][3];
    double w[3][3];
    int n[3];
    for (int a = 0; a < 3; ++a) n[a] = q2_pw(p[a], c[a], w[a]);
    for (int x = 0; x < n[0]; ++x)
      for (int y = 0; y < n[1]; ++y)
        for (int z = 0; z < n[2]; ++z) {
          const int32_t col = Cl.host_of[static_cast<size_t>((c[0][x] * Mc + c[1][y]) * Mc + c[2][z])];
          if (col < 0) invalid("prolongation reaches a non-local coarse node");
          row.emplace_back(col, (w[0][x] * w[1][y]) * w[2][z]);
        }
  });
}

void q2_rhs(pf_fe_setup& s) {
  const FeLevel& L = *s.levels.back();
  const int64_t N = L.N, M = 2 * N + 1;
  const Rule g = gauss3();
  const double h = 1.0 / static_cast<double>(N);
  const double vol = (h * h) * h, K3 = (3.0 * kPi) * kPi;
  // sin(pi x) at the Gauss points of every cell interval
  std::vector<double> S(static_cast<size_t>(N * 3));
  for (int64_t c = 0; c < N; ++c)
    for (int q = 0; q < 3; ++q) S[static_cast<size_t>(c * 3 + q)] = std::sin(kPi * ((static_cast<double>(c) + g.t[q]) * h));
  double V[3][3];
  for (int i = 0; i < 3; ++i)
    for (int q = 0; q < 3; ++q) V[i][q] = q2_phi(i, g.t[q]);
  std::vector<double> le(static_cast<size_t>(N * N * N * 27));
#pragma omp parallel for schedule(static)
  for (int64_t cell = 0; cell < N * N * N; ++cell) {
    const int64_t cx = cell / (N * N), cy = (cell / N) % N, cz = cell % N;
    double* out = &le[static_cast<size_t>(cell * 27)];
    for (int a = 0; a < 27; ++a) out[a] = 0.0;
    for (int qx = 0; qx < 3; ++qx)
      for (int qy = 0; qy < 3; ++qy)
        for (int qz = 0; qz < 3; ++qz) {
          const double w = (g.w[qx] * g.w[qy]) * g.w[qz];
          const double f = ((K3 * S[static_cast<size_t>(cx * 3 + qx)]) * S[static_cast<size_t>(cy * 3 + qy)]) *
                           S[static_cast<size_t>(cz * 3 + qz)];
          const double wf = (w * vol) * f;
          for (int a = 0; a < 27; ++a) out[a] += wf * ((V[a / 9][qx] * V[(a / 3) % 3][qy]) * V[a % 3][qz]);
        }
  }
  s.b.assign(static_cast<size_t>(L.n), 0.0);
  s.x0.assign(static_cast<size_t>(L.n), 0.0);
  s.exact.assign(static_cast<size_t>(L.n), 0.0);
#pragma omp parallel for schedule(static)
  for (int64_t hh = 0; hh < L.n; ++hh) {
    const int64_t e = L.lex_of[static_cast<size_t>(hh)];
    const int64_t p[3] = {e / (M * M), (e / M) % M, e % M};
    double u = 1.0;
    for (int a = 0; a < 3; ++a) u *= std::sin(kPi * (static_cast<double>(p[a]) / static_cast<double>(2 * N)));
    s.exact[static_cast<size_t>(hh)] = u;
    if (hh >= L.n_own) continue;
    int64_t pc[3][2];
    int np[3];
    for (int a = 0; a < 3; ++a) np[a] = q2_cells(p[a], N, pc[a]);
    double acc = 0.0;
    for (int x = 0; x < np[0]; ++x)
      for (int y = 0; y < np[1]; ++y)
        for (int z = 0; z < np[2]; ++z) {
          const int64_t cell = (pc[0][x] * N + pc[1][y]) * N + pc[2][z];
          const int la = static_cast<int>(((p[0] - 2 * pc[0][x]) * 3 + (p[1] - 2 * pc[1][y])) * 3 + (p[2] - 2 * pc[2][z]));
          acc += le[static_cast<size_t>(cell * 27 + la)];
        }
    s.b[static_cast<size_t>(hh)] = acc;
  }
}

// ---------------------------------------------------------------- rotated Q1 --

// Face entity (o, a0, a1, a2): a_o in [0, N], the others in [0, N).
struct Faces {
  int64_t N, per;  // per orientation: N^2 (N + 1)
  int64_t lex(int o, const int64_t* a) const {
    const int64_t e1 = N + (o == 1), e2 = N + (o == 2);
    return o * per + (a[0] * e1 + a[1]) * e2 + a[2];
  }
  void unlex(int64_t e, int* o, int64_t* a) const {
    *o = static_cast<int>(e / per);
    const int64_t r = e % per, e1 = N + (*o == 1), e2 = N + (*o == 2);
    a[0] = r / (e1 * e2);
    a[1] = (r / e2) % e1;
    a[2] = r % e2;
  }
};

// basis of the face (o, sigma) on the unit cube in X = 2 t - 1 coordinates:
//   phi = 1/6 + sigma X_o / 2 + (2 X_o^2 - X_p^2 - X_q^2) / 4     (p < q the other axes)
double rt_phi(int o, double sigma, const double* X) {
  const int p = o == 0 ? 1 : 0, q = o == 2 ? 1 : 2;
  return (1.0 / 6.0 + (0.5 * sigma) * X[o]) + 0.25 * ((2.0 * X[o] * X[o] - X[p] * X[p]) - X[q] * X[q]);
}
// its gradient in t: d/dt_o = sigma + 2 X_o, d/dt_p = -X_p
void rt_grad(int o, double sigma, const double* X, double* g) {
  for (int a = 0; a < 3; ++a) g[a] = a == o ? sigma + 2.0 * X[a] : -X[a];
}

// Stiffness of the unit cube, 6 x 6, local face s = 2 o + (sigma > 0).
std::vector<double> rt_kref() {
  const Rule g = gauss2();
  std::vector<double> K(36, 0.0);
  for (int a = 0; a < 6; ++a)
    for (int b = 0; b < 6; ++b) {
      double s = 0.0;
      for (int qx = 0; qx < 2; ++qx)
        for (int qy = 0; qy < 2; ++qy)
          for (int qz = 0; qz < 2; ++qz) {
            const double X[3] = {2.0 * g.t[qx] - 1.0, 2.0 * g.t[qy] - 1.0, 2.0 * g.t[qz] - 1.0};
            const double w = (g.w[qx] * g.w[qy]) * g.w[qz];
            double ga[3], gb[3];
            rt_grad(a / 2, (a & 1) ? 1.0 : -1.0, X, ga);
            rt_grad(b / 2, (b & 1) ? 1.0 : -1.0, X, gb);
            s += w * ((ga[0] * gb[0] + ga[1] * gb[1]) + ga[2] * gb[2]);
          }
      K[static_cast<size_t>(a * 6 + b)] = s;
    }
  return K;
}

// the cells of a face (ascending) and the face's local slot in each
int rt_cells(const Faces& Fc, int o, const int64_t* a, int64_t* cell, int* slot) {
  const int64_t N = Fc.N;
  int n = 0;
  for (int side = 0; side < 2; ++side) {
    const int64_t co = a[o] - 1 + side;
    if (co < 0 || co >= N) continue;
    int64_t c[3] = {a[0], a[1], a[2]};
    c[o] = co;
    cell[n] = (c[0] * N + c[1]) * N + c[2];
    slot[n] = 2 * o + (side == 0 ? 1 : 0);  // the + face of the lower cell, the - face of the upper
    ++n;
  }
  return n;
}
// face lex of local slot s of cell (cx, cy, cz)
int64_t rt_face_of(const Faces& Fc, int64_t cell, int s) {
  const int64_t N = Fc.N;
  int64_t a[3] = {cell / (N * N), (cell / N) % N, cell % N};
  const int o = s / 2;
  a[o] += s & 1;
  return Fc.lex(o, a);
}

void rt_level(FeLevel& L, const Region& R, const std::vector<double>& Kref, const std::vector<double>& kappa) {
  const int64_t N = R.N;
  L.N = N;
  const Faces Fc{N, N * N * (N + 1)};
  const int64_t n_lex = 3 * Fc.per;
  auto cells_of = [&Fc](int64_t e, int64_t* cells) {
    int o;
    int64_t a[3];
    Fc.unlex(e, &o, a);
    int slot[2];
    return rt_cells(Fc, o, a, cells, slot);
  };
  std::vector<uint8_t> bnd(static_cast<size_t>(n_lex));
  for (int64_t e = 0; e < n_lex; ++e) {
    int o;
    int64_t a[3];
    Fc.unlex(e, &o, a);
    bnd[static_cast<size_t>(e)] = (a[o] == 0 || a[o] == N) ? 1 : 0;
  }
  classify(L, R, n_lex, cells_of, bnd);
  L.keys.resize(static_cast<size_t>(L.n) * 4);
  L.color.resize(static_cast<size_t>(L.n_own));
  for (int64_t h = 0; h < L.n; ++h) {
    int o;
    int64_t a[3];
    Fc.unlex(L.lex_of[static_cast<size_t>(h)], &o, a);
    int64_t* key = &L.keys[static_cast<size_t>(h) * 4];
    key[0] = o;
    key[1] = a[0];
    key[2] = a[1];
    key[3] = a[2];
    if (h < L.n_own) L.color[static_cast<size_t>(h)] = 2 * o + static_cast<int32_t>(a[o] & 1);
  }
  const double hx = 1.0 / static_cast<double>(N);
  std::vector<double> Ke(36);
  for (int i = 0; i < 36; ++i) Ke[static_cast<size_t>(i)] = hx * Kref[static_cast<size_t>(i)];
  build_csr(L, [&](int64_t h, std::vector<std::pair<int32_t, double>>& row, bool values) {
    int o;
    int64_t a[3];
    Fc.unlex(L.lex_of[static_cast<size_t>(h)], &o, a);
    int64_t cell[2];
    int slot[2];
    const int nall = rt_cells(Fc, o, a, cell, slot);
    int nc = 0;
    for (int k = 0; k < nall; ++k)
      if (R.is_local(cell[k])) {
        cell[nc] = cell[k];
        slot[nc] = slot[k];
        ++nc;
      }
    if (h < L.n_own && nc != nall) invalid("own row with a non-local cell");
    const bool dir = L.is_dir[static_cast<size_t>(h)] != 0;
    // the faces of the face's local cells, each once: cell 0's six, then cell 1's other five
    for (int k = 0; k < nc; ++k)
      for (int s2 = 0; s2 < 6; ++s2) {
        if (k == 1 && s2 == slot[1]) continue;  // the face itself, already listed by cell 0
        const int32_t col = L.host_of[static_cast<size_t>(rt_face_of(Fc, cell[k], s2))];
        double v = 0.0;
        if (values) {
          if (dir) {
            v = col == h ? 1.0 : 0.0;
          } else if (col == h) {
            for (int u = 0; u < nc; ++u)
              v += kappa[static_cast<size_t>(cell[u])] * Ke[static_cast<size_t>(slot[u] * 6 + slot[u])];
          } else {
            v += kappa[static_cast<size_t>(cell[k])] * Ke[static_cast<size_t>(slot[k] * 6 + s2)];
          }
        }
        row.emplace_back(col, v);
      }
  });
}

// Fine face means of the coarse function, averaged over the two sides of a coarse face;
// no entries for Dirichlet fine faces (the correction keeps their values).
void rt_prolongation(FeLevel& F, const FeLevel& Cl) {
  const Faces Ff{F.N, F.N * F.N * (F.N + 1)}, Fcn{Cl.N, Cl.N * Cl.N * (Cl.N + 1)};
  const int64_t Nc = Cl.N;
  build_p(F, [&](int64_t h, std::vector<std::pair<int32_t, double>>& row) {
    if (F.is_dir[static_cast<size_t>(h)]) return;
    int o;
    int64_t a[3];
    Ff.unlex(F.lex_of[static_cast<size_t>(h)], &o, a);
    // coarse cells containing the fine face and the face's normal coordinate X_o in each
    int64_t cells[2];
    double Xo[2];
    int nc = 0;
    if (a[o] & 1) {
      cells[0] = (a[o] - 1) / 2;
      Xo[0] = 0.0;
      nc = 1;
    } else {
      const int64_t pl = a[o] / 2;
      if (pl - 1 >= 0) {
        cells[nc] = pl - 1;
        Xo[nc++] = 1.0;
      }
      if (pl < Nc) {
        cells[nc] = pl;
        Xo[nc++] = -1.0;
      }
    }
    const double scale = nc == 2 ? 0.5 : 1.0;
    for (int k = 0; k < nc; ++k) {
      int64_t c[3];
      double m[3];  // mean of X_t over the fine face along each tangential axis
      for (int t = 0; t < 3; ++t) {
        if (t == o) {
          c[t] = cells[k];
          m[t] = 0.0;
        } else {
          c[t] = a[t] / 2;
          m[t] = (a[t] & 1) ? 0.5 : -0.5;
        }
      }
      const int64_t cell = (c[0] * Nc + c[1]) * Nc + c[2];
      for (int s2 = 0; s2 < 6; ++s2) {
        const int o2 = s2 / 2;
        const double sg = (s2 & 1) ? 1.0 : -1.0;
        double w;
        if (o2 == o)
          w = Xo[k] == 0.0 ? 0.0 : (sg == Xo[k] ? 1.0 : 0.0);
        else
          w = (Xo[k] == 0.0 ? 0.25 : 0.0) + 0.5 * (sg * m[o2]);
        if (w == 0.0) continue;
        const int32_t col = Cl.host_of[static_cast<size_t>(rt_face_of(Fcn, cell, s2))];
        if (col < 0) invalid("prolongation reaches a non-local coarse face");
        const double ws = scale * w;
        bool merged = false;
        for (auto& [cc, ww] : row)
          if (cc == col) {
            ww += ws;
            merged = true;
          }
        if (!merged) row.emplace_back(col, ws);
      }
    }
  });
}

void rt_rhs(pf_fe_setup& s) {
  const FeLevel& L = *s.levels.back();
  const int64_t N = L.N;
  const Faces Fc{N, N * N * (N + 1)};
  const Rule g = gauss3();
  const double h = 1.0 / static_cast<double>(N);
  const double vol = (h * h) * h, K3 = (3.0 * kPi) * kPi;
  std::vector<double> S(static_cast<size_t>(N * 3));
  for (int64_t c = 0; c < N; ++c)
    for (int q = 0; q < 3; ++q) S[static_cast<size_t>(c * 3 + q)] = std::sin(kPi * ((static_cast<double>(c) + g.t[q]) * h));
  double phi[27][6];
  for (int q = 0; q < 27; ++q) {
    const double X[3] = {2.0 * g.t[q / 9] - 1.0, 2.0 * g.t[(q / 3) % 3] - 1.0, 2.0 * g.t[q % 3] - 1.0};
    for (int a = 0; a < 6; ++a) phi[q][a] = rt_phi(a / 2, (a & 1) ? 1.0 : -1.0, X);
  }
  std::vector<double> le(static_cast<size_t>(N * N * N * 6));
#pragma omp parallel for schedule(static)
  for (int64_t cell = 0; cell < N * N * N; ++cell) {
    const int64_t cx = cell / (N * N), cy = (cell / N) % N, cz = cell % N;
    double* out = &le[static_cast<size_t>(cell * 6)];
    for (int a = 0; a < 6; ++a) out[a] = 0.0;
    for (int q = 0; q < 27; ++q) {
      const int qx = q / 9, qy = (q / 3) % 3, qz = q % 3;
      const double w = (g.w[qx] * g.w[qy]) * g.w[qz];
      const double f = ((K3 * S[static_cast<size_t>(cx * 3 + qx)]) * S[static_cast<size_t>(cy * 3 + qy)]) *
                       S[static_cast<size_t>(cz * 3 + qz)];
      const double wf = (w * vol) * f;
      for (int a = 0; a < 6; ++a) out[a] += wf * phi[q][a];
    }
  }
  s.b.assign(static_cast<size_t>(L.n), 0.0);
  s.x0.assign(static_cast<size_t>(L.n), 0.0);
  s.exact.assign(static_cast<size_t>(L.n), 0.0);
  const double ph = kPi * h;
#pragma omp parallel for schedule(static)
  for (int64_t hh = 0; hh < L.n; ++hh) {
    int o;
    int64_t a[3];
    Fc.unlex(L.lex_of[static_cast<size_t>(hh)], &o, a);
    double u = 1.0;
    for (int t = 0; t < 3; ++t) {
      const double x0 = static_cast<double>(a[t]) * h;
      u *= t == o ? std::sin(kPi * x0) : (std::cos(kPi * x0) - std::cos(kPi * (static_cast<double>(a[t] + 1) * h))) / ph;
    }
    s.exact[static_cast<size_t>(hh)] = u;
    if (hh >= L.n_own) continue;
    int64_t cell[2];
    int slot[2];
    const int nc = rt_cells(Fc, o, a, cell, slot);
    double acc = 0.0;
    for (int k = 0; k < nc; ++k) acc += le[static_cast<size_t>(cell[k] * 6 + slot[k])];
    s.b[static_cast<size_t>(hh)] = acc;
  }
}

// ------------------------------------------------------------------- create --

void create(pf_fe_setup& s) {
  const int nl = s.n_levels;
  s.coarse_owner = pf_coarse_partition(3, s.n_coarse, s.n_ranks);
  s.levels.clear();
  for (int l = 0; l < nl; ++l) s.levels.push_back(std::make_unique<FeLevel>());
  const int64_t Nf = static_cast<int64_t>(s.n_coarse) << (nl - 1);
  if (s.family == PF_FE_Q2) {
    const std::vector<double> Kref = q2_kref();
    s.kappa.assign(static_cast<size_t>(Nf * Nf * Nf), 1.0);
    for (int l = 0; l < nl; ++l) {
      const int64_t N = static_cast<int64_t>(s.n_coarse) << l;
      const double h = 1.0 / static_cast<double>(N);
      std::vector<double> Ke(Kref.size());
      for (size_t i = 0; i < Kref.size(); ++i) Ke[i] = h * Kref[i];
      q2_level(*s.levels[static_cast<size_t>(l)], make_region(s, l), Ke);
      s.levels[static_cast<size_t>(l)]->elem = Ke;
      if (l > 0) q2_prolongation(*s.levels[static_cast<size_t>(l)], *s.levels[static_cast<size_t>(l) - 1]);
    }
    q2_rhs(s);
  } else {
    const std::vector<double> Kref = rt_kref();
    // coefficients: finest by the generator, each coarser cell the mean of its 8 children
    std::vector<std::vector<double>> kap(static_cast<size_t>(nl));
    kap.back().resize(static_cast<size_t>(Nf * Nf * Nf));
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < Nf * Nf * Nf; ++c)
      kap.back()[static_cast<size_t>(c)] = s.coefficient == PF_COEF_LOGNORMAL ? pf::lognormal_kappa(s.seed, c) : 1.0;
    for (int l = nl - 2; l >= 0; --l) {
      const int64_t N = static_cast<int64_t>(s.n_coarse) << l, N2 = 2 * N;
      auto& kc = kap[static_cast<size_t>(l)];
      const auto& kf = kap[static_cast<size_t>(l) + 1];
      kc.resize(static_cast<size_t>(N * N * N));
#pragma omp parallel for schedule(static)
      for (int64_t c = 0; c < N * N * N; ++c) {
        const int64_t cx = c / (N * N), cy = (c / N) % N, cz = c % N;
        double sum = 0.0;
        for (int d = 0; d < 8; ++d)
          sum += kf[static_cast<size_t>(((2 * cx + (d >> 2)) * N2 + 2 * cy + ((d >> 1) & 1)) * N2 + 2 * cz + (d & 1))];
        kc[static_cast<size_t>(c)] = 0.125 * sum;
      }
    }
    for (int l = 0; l < nl; ++l) {
      FeLevel& L = *s.levels[static_cast<size_t>(l)];
      rt_level(L, make_region(s, l), Kref, kap[static_cast<size_t>(l)]);
      const double hx = 1.0 / static_cast<double>(static_cast<int64_t>(s.n_coarse) << l);
      L.elem.resize(36);
      for (int i = 0; i < 36; ++i) L.elem[static_cast<size_t>(i)] = hx * Kref[static_cast<size_t>(i)];
      if (l + 1 < nl) L.kappa = kap[static_cast<size_t>(l)];
      if (l > 0) rt_prolongation(*s.levels[static_cast<size_t>(l)], *s.levels[static_cast<size_t>(l) - 1]);
    }
    s.kappa = std::move(kap.back());
    rt_rhs(s);
  }
  for (auto& L : s.levels) {
    L->host_of.clear();
    L->host_of.shrink_to_fit();
    L->lex_of.clear();
    L->lex_of.shrink_to_fit();
  }
}

template <typename F>
pf_status guard(F&& f) {
  try {
    f();
    return PF_OK;
  } catch (const FeError& e) {
    g_fe_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_fe_err = e.what();
    return PF_ERR_STATE;
  }
}

}  // namespace

extern "C" {

const char* pf_fe_last_error(void) { return g_fe_err.c_str(); }

pf_status pf_fe_setup_create_part(int family, int n_coarse, int n_levels, int coefficient, uint64_t seed,
                                  int n_ranks, int rank, pf_fe_setup** out) {
  return guard([&] {
    if (!out) invalid("null argument");
    *out = nullptr;
    if (family != PF_FE_Q2 && family != PF_FE_ROTATED_Q1) invalid("unknown element family");
    if (coefficient != PF_COEF_CONSTANT && coefficient != PF_COEF_LOGNORMAL) invalid("unknown coefficient");
    if (family == PF_FE_Q2 && coefficient != PF_COEF_CONSTANT) invalid("Q2 takes the constant coefficient only");
    if (n_coarse < 2 || n_levels < 1 || n_levels > 12) invalid("need n_coarse >= 2 and 1 <= n_levels <= 12");
    if (n_ranks < 1 || n_ranks > n_coarse * n_coarse * n_coarse || n_ranks > 127 || rank < 0 || rank >= n_ranks)
      invalid("need 1 <= n_ranks <= coarse cells and 0 <= rank < n_ranks");
    auto s = std::make_unique<pf_fe_setup>();
    s->family = family;
    s->n_coarse = n_coarse;
    s->n_levels = n_levels;
    s->coefficient = coefficient;
    s->seed = seed;
    s->n_ranks = n_ranks;
    s->rank = rank;
    const auto t0 = std::chrono::steady_clock::now();
    create(*s);
    s->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = s.release();
  });
}

pf_status pf_fe_setup_create(int family, int n_coarse, int n_levels, int coefficient, uint64_t seed,
                             pf_fe_setup** out) {
  return pf_fe_setup_create_part(family, n_coarse, n_levels, coefficient, seed, 1, 0, out);
}

pf_status pf_fe_setup_destroy(pf_fe_setup* s) {
  delete s;
  return PF_OK;
}

pf_status pf_fe_setup_level(const pf_fe_setup* s, int level, pf_level_desc* out) {
  return guard([&] {
    if (!s || !out) invalid("null argument");
    if (level < 0 || level >= s->n_levels) invalid("level out of range");
    const FeLevel& L = *s->levels[static_cast<size_t>(level)];
    std::memset(out, 0, sizeof *out);
    out->n_dofs = L.n;
    out->n_own_dofs = L.n_own;
    out->row_offsets = L.rowptr.data();
    out->col_indices = L.cols.data();
    out->values = L.vals.data();
    out->owns_row = L.owns_row.data();
    out->is_dirichlet = L.is_dir.data();
    out->color = L.color.data();
    out->row_order = L.order.data();
    out->n_channels = static_cast<int32_t>(L.descs.size());
    out->channels = L.descs.data();
    if (level > 0) {
      out->p_offsets = L.p_off.data();
      out->p_cols = L.p_col.data();
      out->p_weights = L.p_w.data();
    }
  });
}

pf_status pf_fe_setup_level_keys(const pf_fe_setup* s, int level, const int64_t** keys4, const uint8_t** class_of) {
  return guard([&] {
    if (!s || !keys4 || !class_of) invalid("null argument");
    if (level < 0 || level >= s->n_levels) invalid("level out of range");
    *keys4 = s->levels[static_cast<size_t>(level)]->keys.data();
    *class_of = s->levels[static_cast<size_t>(level)]->class_of.data();
  });
}

pf_status pf_fe_setup_rhs(const pf_fe_setup* s, const double** b, const double** x0, const double** exact,
                          int64_t* n) {
  return guard([&] {
    if (!s || !b || !x0 || !exact || !n) invalid("null argument");
    *b = s->b.data();
    *x0 = s->x0.data();
    *exact = s->exact.data();
    *n = static_cast<int64_t>(s->b.size());
  });
}

pf_status pf_fe_setup_kappa(const pf_fe_setup* s, const double** kappa, int64_t* n) {
  return guard([&] {
    if (!s || !kappa || !n) invalid("null argument");
    *kappa = s->kappa.data();
    *n = static_cast<int64_t>(s->kappa.size());
  });
}

pf_status pf_fe_setup_assembly_desc(const pf_fe_setup* s, int level, pf_fe_assembly_desc* out) {
  return guard([&] {
    if (!s || !out) invalid("null argument");
    if (level < 0 || level >= s->n_levels) invalid("level out of range");
    const FeLevel& L = *s->levels[static_cast<size_t>(level)];
    std::memset(out, 0, sizeof *out);
    out->family = s->family;
    out->n_cells = static_cast<int32_t>(L.N);
    out->n_dofs = L.n;
    out->keys4 = L.keys.data();
    out->is_dirichlet = L.is_dir.data();
    out->elem = L.elem.data();
    if (s->family == PF_FE_ROTATED_Q1)
      out->kappa = level + 1 == s->n_levels ? s->kappa.data() : L.kappa.data();
  });
}

pf_status pf_fe_setup_seconds(const pf_fe_setup* s, double* out) {
  return guard([&] {
    if (!s || !out) invalid("null argument");
    *out = s->seconds;
  });
}

}  // extern "C"
