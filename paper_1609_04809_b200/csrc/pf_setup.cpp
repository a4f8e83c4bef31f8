// pf_setup.cpp — structured, communication-free hierarchy setup (see include/pf_setup.h).
//
// Everything the reference derives with std::map lookups and a cross-rank handshake is a
// closed-form function of the lattice here:
//   owner(cell)            = coarse owner of (cell >> level)          partition.cpp:255-265
//   local(rank, cell)      = cell owned by rank or sharing a vertex with one it owns
//                                                                    partition.cpp:156-240
//   dependent(rank, cell)  = owned cell sharing a vertex with a foreign cell
//   interface carriers     = vertices whose cells have >= 2 owners; masters by the greedy
//                            "fewest so far, ties to the lowest rank" rule in key order
//                                                                    femapper.cpp:84-121
//   dof classes / channels = femapper.cpp:123-165, :222-351 evaluated per vertex
// so a rank can classify its own vertices and its neighbours' vertices (to know what
// they will request) without any message.
#include "pf_setup.h"

#include <omp.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace {

struct SetupError : std::runtime_error {
  pf_status code;
  SetupError(pf_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void invalid(const std::string& m) { throw SetupError(PF_ERR_INVALID_ARGUMENT, m); }

thread_local std::string g_setup_err;

const double kPi = std::acos(-1.0);

enum Cls : uint8_t { kMaster = 0, kIndep = 1, kDep1 = 2, kDep2 = 3, kSlave = 4, kHalo1 = 5, kHalo2 = 6, kDirichlet = 7 };

// Ring order of cell corners (mesh.cpp:16-21).
constexpr int kRing[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                             {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};

// ------------------------------------------------------------ coarse partition --

// Coordinate bisection of the coarse cells (partition.cpp:35-74, :104-142), restated.
std::vector<int> coarse_partition(int d, int n, int k) {
  const int64_t nz = d == 3 ? n : 1;
  const int64_t total = static_cast<int64_t>(n) * n * nz;
  if (k < 1) invalid("partition needs k >= 1");
  if (k > total)
    invalid("partition needs at least one cell per rank: k=" + std::to_string(k) +
            ", cells=" + std::to_string(total));
  std::vector<int64_t> targets(static_cast<size_t>(k), total / k);
  for (int i = 0; i < static_cast<int>(total % k); ++i) ++targets[static_cast<size_t>(i)];
  auto corner = [&](int64_t c, int a) -> int64_t {
    const int64_t ix = c / (n * nz), iy = (c / nz) % n, iz = c % nz;
    return a == 0 ? ix : a == 1 ? iy : iz;
  };
  std::vector<int> owner(static_cast<size_t>(total), -1);
  std::vector<int64_t> ids(static_cast<size_t>(total));
  std::iota(ids.begin(), ids.end(), 0);
  struct Rec {
    static void go(std::vector<int64_t>& cells, int r0, int r1, int d, const std::vector<int64_t>& targets,
                   std::vector<int>& owner, const decltype(corner)& corner) {
      if (r1 - r0 == 1) {
        for (int64_t c : cells) owner[static_cast<size_t>(c)] = r0;
        return;
      }
      const int mid = r0 + (r1 - r0) / 2;
      int64_t left = 0;
      for (int r = r0; r < mid; ++r) left += targets[static_cast<size_t>(r)];
      int axis = 0;
      int64_t best = -1;
      for (int a = 0; a < d; ++a) {
        int64_t lo = corner(cells.front(), a), hi = lo;
        for (int64_t c : cells) {
          lo = std::min(lo, corner(c, a));
          hi = std::max(hi, corner(c, a));
        }
        if (hi - lo > best) {
          best = hi - lo;
          axis = a;
        }
      }
      std::stable_sort(cells.begin(), cells.end(), [&](int64_t a, int64_t b) {
        const int64_t ca = corner(a, axis), cb = corner(b, axis);
        if (ca != cb) return ca < cb;
        return a < b;  // gcn == index at level 0
      });
      std::vector<int64_t> L(cells.begin(), cells.begin() + left), R(cells.begin() + left, cells.end());
      go(L, r0, mid, d, targets, owner, corner);
      go(R, mid, r1, d, targets, owner, corner);
    }
  };
  Rec::go(ids, 0, k, d, targets, owner, corner);
  return owner;
}

// ------------------------------------------------------------------- geometry --

struct Geo {
  int d = 3;
  int n_coarse = 2;
  int level = 0;
  int64_t N = 0;       // cells per axis
  int64_t S = 1;       // fine cells per coarse cell per axis
  int nranks = 1;
  const std::vector<int>* coarse_owner = nullptr;
  std::unordered_map<int64_t, int> master;  // interface vertex -> master rank

  int64_t nzc() const { return d == 3 ? N : 1; }     // cells along z
  int64_t nzv() const { return d == 3 ? N + 1 : 1; } // vertices along z
  int64_t vkey(int64_t x, int64_t y, int64_t z) const { return (x * (N + 1) + y) * nzv() + z; }
  bool cell_in(int64_t x, int64_t y, int64_t z) const {
    return x >= 0 && y >= 0 && z >= 0 && x < N && y < N && z < nzc();
  }
  int owner(int64_t x, int64_t y, int64_t z) const {
    const int64_t n = n_coarse, nz = d == 3 ? n : 1;
    return (*coarse_owner)[static_cast<size_t>(((x / S) * n + (y / S)) * nz + (z / S))];
  }
  bool boundary(int64_t x, int64_t y, int64_t z) const {
    return x == 0 || x == N || y == 0 || y == N || (d == 3 && (z == 0 || z == N));
  }
  int master_of(int64_t x, int64_t y, int64_t z) const {
    // interface carriers lie on coarse-cell planes
    if (x % S && y % S && (d == 2 || z % S)) return -1;
    auto it = master.find(vkey(x, y, z));
    return it == master.end() ? -1 : it->second;
  }
  // distinct owners of the in-domain cells around a vertex, ascending
  int owners_around(int64_t x, int64_t y, int64_t z, int* out) const {
    int n = 0;
    const int zlo = d == 3 ? -1 : 0;
    for (int dx = -1; dx <= 0; ++dx)
      for (int dy = -1; dy <= 0; ++dy)
        for (int dz = zlo; dz <= 0; ++dz) {
          if (!cell_in(x + dx, y + dy, z + dz)) continue;
          const int o = owner(x + dx, y + dy, z + dz);
          bool seen = false;
          for (int i = 0; i < n; ++i) seen = seen || out[i] == o;
          if (!seen) out[n++] = o;
        }
    for (int i = 1; i < n; ++i)
      for (int j = i; j > 0 && out[j - 1] > out[j]; --j) std::swap(out[j - 1], out[j]);
    return n;
  }
};

// Global interface carriers and their masters (femapper.cpp:84-121): candidates are the
// vertices on coarse-cell planes; key order is lexicographic (x, y, z) = vkey order.
void assign_masters(Geo& g) {
  std::vector<int64_t> keys;
  const int64_t nzv = g.nzv();
  for (int a = 0; a < g.d; ++a)
    for (int64_t m = 0; m <= g.n_coarse; ++m) {
      int64_t lo[3] = {0, 0, 0}, hi[3] = {g.N + 1, g.N + 1, nzv};
      lo[a] = m * g.S;
      hi[a] = m * g.S + 1;
      for (int64_t x = lo[0]; x < hi[0]; ++x)
        for (int64_t y = lo[1]; y < hi[1]; ++y)
          for (int64_t z = lo[2]; z < hi[2]; ++z) {
            int own[8];
            if (g.owners_around(x, y, z, own) >= 2) keys.push_back(g.vkey(x, y, z));
          }
    }
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  std::vector<int64_t> assigned(static_cast<size_t>(g.nranks), 0);
  g.master.reserve(keys.size() * 2);
  for (int64_t k : keys) {
    const int64_t z = k % nzv, y = (k / nzv) % (g.N + 1), x = k / (nzv * (g.N + 1));
    int own[8];
    const int n = g.owners_around(x, y, z, own);
    int best = own[0];
    for (int i = 0; i < n; ++i)
      if (assigned[static_cast<size_t>(own[i])] < assigned[static_cast<size_t>(best)]) best = own[i];
    g.master.emplace(k, best);
    ++assigned[static_cast<size_t>(best)];
  }
}

struct Box {
  int64_t lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};  // [lo, hi)
  int64_t ext(int a) const { return hi[a] - lo[a]; }
  int64_t size() const { return ext(0) * ext(1) * ext(2); }
  bool in(int64_t x, int64_t y, int64_t z) const {
    return x >= lo[0] && x < hi[0] && y >= lo[1] && y < hi[1] && z >= lo[2] && z < hi[2];
  }
  int64_t idx(int64_t x, int64_t y, int64_t z) const {
    return ((x - lo[0]) * ext(1) + (y - lo[1])) * ext(2) + (z - lo[2]);
  }
};

// One rank's cell flags over a region of cells.
struct RankView {
  const Geo* g = nullptr;
  int q = 0;
  Box R;
  std::vector<uint8_t> local, dep, hasm;

  void build(const Geo& geo, int rank, const Box& region) {
    g = &geo;
    q = rank;
    R = region;
    const int64_t n = R.size();
    local.assign(static_cast<size_t>(n), 0);
    dep.assign(static_cast<size_t>(n), 0);
    hasm.assign(static_cast<size_t>(n), 0);
    const int d = geo.d;
    const int64_t S = geo.S;
#pragma omp parallel for schedule(static) collapse(2)
    for (int64_t x = R.lo[0]; x < R.hi[0]; ++x)
      for (int64_t y = R.lo[1]; y < R.hi[1]; ++y)
        for (int64_t z = R.lo[2]; z < R.hi[2]; ++z) {
          const int64_t i = R.idx(x, y, z);
          const int o = geo.owner(x, y, z);
          const bool interior = (x % S) > 0 && (x % S) < S - 1 && (y % S) > 0 && (y % S) < S - 1 &&
                                (d == 2 || ((z % S) > 0 && (z % S) < S - 1));
          bool has_q = o == q, has_foreign = o != q;
          if (!interior) {
            const int zr = d == 3 ? 1 : 0;
            for (int dx = -1; dx <= 1; ++dx)
              for (int dy = -1; dy <= 1; ++dy)
                for (int dz = -zr; dz <= zr; ++dz) {
                  if (!geo.cell_in(x + dx, y + dy, z + dz)) continue;
                  const int oo = geo.owner(x + dx, y + dy, z + dz);
                  if (oo == q) has_q = true;
                  else has_foreign = true;
                }
          }
          local[i] = has_q;
          dep[i] = (o == q) && has_foreign;
          bool hm = false;
          if (!interior) {
            const int nv = 1 << d;
            for (int v = 0; v < nv && !hm; ++v) {
              const int64_t vx = x + kRing[v][0], vy = y + kRing[v][1], vz = z + (d == 3 ? kRing[v][2] : 0);
              if (geo.boundary(vx, vy, vz)) continue;
              hm = geo.master_of(vx, vy, vz) == q;
            }
          }
          hasm[i] = hm;
        }
  }
  bool cell_local(int64_t x, int64_t y, int64_t z) const {
    return g->cell_in(x, y, z) && R.in(x, y, z) && local[R.idx(x, y, z)];
  }
};

struct VInfo {
  bool local = false;
  uint8_t cls = 0;
  int target = -1, kind = -1;  // request this rank makes for the vertex
  int owners_front = -1;
  int diri_authority = -1;
};

// femapper.cpp:123-165 (classes) and :237-264 (requests) for one vertex of rank q.
VInfo classify(const RankView& V, int64_t x, int64_t y, int64_t z) {
  const Geo& g = *V.g;
  VInfo info;
  int owners[8];
  int n_owners = 0;
  bool on_own = false, on_halo = false, any_dep = false, any_hasm = false;
  const int zlo = g.d == 3 ? -1 : 0;
  for (int dx = -1; dx <= 0; ++dx)
    for (int dy = -1; dy <= 0; ++dy)
      for (int dz = zlo; dz <= 0; ++dz) {
        const int64_t cx = x + dx, cy = y + dy, cz = z + dz;
        if (!V.cell_local(cx, cy, cz)) continue;
        const int64_t i = V.R.idx(cx, cy, cz);
        const int o = g.owner(cx, cy, cz);
        bool seen = false;
        for (int k = 0; k < n_owners; ++k) seen = seen || owners[k] == o;
        if (!seen) owners[n_owners++] = o;
        (o == V.q ? on_own : on_halo) = true;
        any_dep = any_dep || V.dep[i];
        any_hasm = any_hasm || V.hasm[i];
      }
  if (n_owners == 0) return info;
  for (int i = 1; i < n_owners; ++i)
    for (int j = i; j > 0 && owners[j - 1] > owners[j]; --j) std::swap(owners[j - 1], owners[j]);
  info.local = true;
  info.owners_front = owners[0];
  const bool interface = on_own && on_halo;
  const int master = g.master_of(x, y, z);
  if (g.boundary(x, y, z)) {
    info.cls = kDirichlet;
    info.diri_authority = master >= 0 ? master : owners[0];
  } else if (interface) {
    info.cls = master == V.q ? kMaster : kSlave;
  } else if (on_halo) {
    info.cls = any_hasm ? kHalo1 : kHalo2;
  } else {
    info.cls = any_dep ? (any_hasm ? kDep2 : kDep1) : kIndep;
  }
  if (interface && master != V.q) {
    info.kind = PF_CH_MASTER_SLAVE;
    info.target = master;
  } else if (info.cls == kHalo1 || info.cls == kHalo2) {
    info.kind = info.cls == kHalo1 ? PF_CH_HALO1 : PF_CH_HALO2;
    info.target = owners[0];
  }
  return info;
}

struct OwnedChannel {
  int kind = 0, peer = 0;
  std::vector<int32_t> send, recv;
};

struct SetupLevel {
  Geo geo;
  int32_t n = 0, n_own = 0;
  Box vbox;                       // vertex box of the local vertices
  std::vector<int32_t> index;     // over vbox: local index or -1
  std::vector<int64_t> vert;      // per local dof: packed vertex key
  std::vector<int64_t> rowptr;
  std::vector<int32_t> cols;
  std::vector<double> vals;
  std::vector<uint8_t> owns_row, is_dir, class_of;
  std::vector<int32_t> color;
  std::vector<int64_t> keys4;
  std::vector<OwnedChannel> channels;
  std::vector<pf_channel_desc> descs;
  std::vector<int64_t> p_off;
  std::vector<int32_t> p_col;
  std::vector<double> p_w;
  int32_t lookup(int64_t x, int64_t y, int64_t z) const {
    return vbox.in(x, y, z) ? index[vbox.idx(x, y, z)] : -1;
  }
};

// Q1 element stiffness on a cube of side h, 2-point Gauss (assembly.cpp:11-92).
struct Element {
  int nv = 8;
  double K[8][8] = {};
  double qp[8][3] = {};   // quadrature points (reference cell)
  double qw[8] = {};      // weight * volume
  double phi[8][8] = {};  // phi[q][v]
};

Element make_element(int d, double h) {
  Element E;
  E.nv = 1 << d;
  const double off = 0.5 / std::sqrt(3.0);
  const double pts[2] = {0.5 - off, 0.5 + off};
  double hh[3] = {1.0, 1.0, 1.0}, volume = 1.0;
  for (int a = 0; a < d; ++a) {
    hh[a] = h;
    volume *= hh[a];
  }
  int q = 0;
  const int nz = d == 3 ? 2 : 1;
  for (int ix = 0; ix < 2; ++ix)
    for (int iy = 0; iy < 2; ++iy)
      for (int iz = 0; iz < nz; ++iz, ++q) {
        const double p[3] = {pts[ix], pts[iy], d == 3 ? pts[iz] : 0.0};
        double w = 0.5 * 0.5;
        if (d == 3) w *= 0.5;
        E.qw[q] = w * volume;
        for (int a = 0; a < 3; ++a) E.qp[q][a] = p[a];
        double grad[8][3];
        for (int v = 0; v < E.nv; ++v) {
          double factor[3] = {1.0, 1.0, 1.0}, dfactor[3] = {0.0, 0.0, 0.0};
          for (int a = 0; a < d; ++a) {
            const bool high = kRing[v][a] == 1;
            factor[a] = high ? p[a] : 1.0 - p[a];
            dfactor[a] = high ? 1.0 : -1.0;
          }
          double value = 1.0;
          for (int a = 0; a < d; ++a) value *= factor[a];
          for (int a = 0; a < d; ++a) {
            double gg = dfactor[a];
            for (int b = 0; b < d; ++b)
              if (b != a) gg *= factor[b];
            grad[v][a] = gg;
          }
          E.phi[q][v] = value;
        }
        for (int i = 0; i < E.nv; ++i)
          for (int j = 0; j < E.nv; ++j) {
            double gsum = 0.0;
            for (int a = 0; a < d; ++a) gsum += grad[i][a] * grad[j][a] / (hh[a] * hh[a]);
            E.K[i][j] += E.qw[q] * gsum;
          }
      }
  return E;
}

int ring_slot(int d, int ox, int oy, int oz) {
  for (int v = 0; v < (1 << d); ++v)
    if (kRing[v][0] == ox && kRing[v][1] == oy && (d == 2 || kRing[v][2] == oz)) return v;
  return -1;
}

struct Problem {
  int kind = 0, d = 3;
  double f(const double* x) const {
    if (kind == PF_PROBLEM_UNIT_SOURCE) return 1.0;
    if (kind == PF_PROBLEM_BASELINE) {
      double u = std::sin(kPi * x[0]) * std::sin(kPi * x[1]);
      if (d == 3) u *= std::sin(kPi * x[2]);
      return d * kPi * kPi * u;
    }
    double u = std::sin(kPi * x[0]) * std::cos(kPi * x[1]);  // model.cpp:12-16
    if (d == 3) u *= std::cos(kPi * x[2]);
    return d * kPi * kPi * u;
  }
  double g(const double* x) const {
    if (kind != PF_PROBLEM_REFERENCE_POISSON) return 0.0;
    double u = std::sin(kPi * x[0]) * std::cos(kPi * x[1]);
    if (d == 3) u *= std::cos(kPi * x[2]);
    return u;
  }
};

}  // namespace

struct pf_setup {
  int d = 3, n_coarse = 2, n_levels = 1, n_ranks = 1, rank = 0;
  Problem prob;
  std::vector<int> coarse_owner;
  std::vector<std::unique_ptr<SetupLevel>> levels;
  std::vector<double> b, x0;
  double seconds = 0;
};

namespace {

Box own_cell_box(const pf_setup& s, const Geo& g) {
  Box b;
  const int n = s.n_coarse;
  const int nz = s.d == 3 ? n : 1;
  int64_t lo[3] = {1 << 30, 1 << 30, 1 << 30}, hi[3] = {-1, -1, -1};
  for (int ix = 0; ix < n; ++ix)
    for (int iy = 0; iy < n; ++iy)
      for (int iz = 0; iz < nz; ++iz)
        if (s.coarse_owner[static_cast<size_t>((ix * n + iy) * nz + iz)] == s.rank) {
          const int64_t c[3] = {ix, iy, iz};
          for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], c[a]);
            hi[a] = std::max(hi[a], c[a] + 1);
          }
        }
  if (hi[0] < 0) invalid("rank owns no cells");
  for (int a = 0; a < 3; ++a) {
    const int64_t S = (a < s.d) ? g.S : 1;
    b.lo[a] = lo[a] * S;
    b.hi[a] = hi[a] * S;
  }
  return b;
}

Box expand(const Box& b, int64_t by, const Geo& g, bool vertices) {
  Box o;
  for (int a = 0; a < 3; ++a) {
    if (a == 2 && g.d == 2) {
      o.lo[a] = 0;
      o.hi[a] = 1;
      continue;
    }
    const int64_t top = vertices ? g.N + 1 : g.N;
    o.lo[a] = std::max<int64_t>(0, b.lo[a] - by);
    o.hi[a] = std::min<int64_t>(top, b.hi[a] + by);
  }
  return o;
}

void build_level(pf_setup& s, int l) {
  auto L = std::make_unique<SetupLevel>();
  Geo& g = L->geo;
  g.d = s.d;
  g.n_coarse = s.n_coarse;
  g.level = l;
  g.S = int64_t(1) << l;
  g.N = static_cast<int64_t>(s.n_coarse) * g.S;
  g.nranks = s.n_ranks;
  g.coarse_owner = &s.coarse_owner;
  assign_masters(g);
  const int d = s.d;
  const int me = s.rank;

  const Box own = own_cell_box(s, g);
  const Box region = expand(own, 2, g, false);
  // vertex box: vertices of cells within one layer of the own box
  Box vb;
  for (int a = 0; a < 3; ++a) {
    if (a == 2 && d == 2) {
      vb.lo[a] = 0;
      vb.hi[a] = 1;
      continue;
    }
    vb.lo[a] = std::max<int64_t>(0, own.lo[a] - 1);
    vb.hi[a] = std::min<int64_t>(g.N + 1, own.hi[a] + 2);
  }
  L->vbox = vb;
  RankView V;
  V.build(g, me, region);

  // --- classify local vertices
  const int64_t nvb = vb.size();
  std::vector<VInfo> info(static_cast<size_t>(nvb));
#pragma omp parallel for schedule(static) collapse(2)
  for (int64_t x = vb.lo[0]; x < vb.hi[0]; ++x)
    for (int64_t y = vb.lo[1]; y < vb.hi[1]; ++y)
      for (int64_t z = vb.lo[2]; z < vb.hi[2]; ++z) info[vb.idx(x, y, z)] = classify(V, x, y, z);

  // --- numbering: own (lexicographic), then Slave, Halo1, Halo2, Dirichlet
  L->index.assign(static_cast<size_t>(nvb), -1);
  int64_t count[8] = {};
  for (const VInfo& v : info)
    if (v.local) ++count[v.cls];
  const int64_t n_own = count[kMaster] + count[kIndep] + count[kDep1] + count[kDep2];
  int64_t total = 0;
  for (int64_t c : count) total += c;
  if (total >= (int64_t(1) << 31)) invalid("local level too large for int32 indices");
  int64_t next[5] = {0, n_own, n_own + count[kSlave], n_own + count[kSlave] + count[kHalo1],
                     n_own + count[kSlave] + count[kHalo1] + count[kHalo2]};
  auto group = [](uint8_t c) { return c <= kDep2 ? 0 : c - 3; };
  L->n = static_cast<int32_t>(total);
  L->n_own = static_cast<int32_t>(n_own);
  L->vert.resize(static_cast<size_t>(total));
  L->class_of.resize(static_cast<size_t>(total));
  L->owns_row.resize(static_cast<size_t>(total));
  L->is_dir.resize(static_cast<size_t>(total));
  L->keys4.resize(static_cast<size_t>(4 * total));
  for (int64_t x = vb.lo[0]; x < vb.hi[0]; ++x)
    for (int64_t y = vb.lo[1]; y < vb.hi[1]; ++y)
      for (int64_t z = vb.lo[2]; z < vb.hi[2]; ++z) {
        const int64_t bi = vb.idx(x, y, z);
        const VInfo& v = info[static_cast<size_t>(bi)];
        if (!v.local) continue;
        const int64_t li = next[group(v.cls)]++;
        L->index[static_cast<size_t>(bi)] = static_cast<int32_t>(li);
        L->vert[static_cast<size_t>(li)] = g.vkey(x, y, z);
        L->class_of[static_cast<size_t>(li)] = v.cls;
        L->is_dir[static_cast<size_t>(li)] = v.cls == kDirichlet;
        L->owns_row[static_cast<size_t>(li)] = v.cls <= kDep2 || (v.cls == kDirichlet && v.diri_authority == me);
        int64_t* k4 = &L->keys4[static_cast<size_t>(4 * li)];
        k4[0] = 0;
        k4[1] = x;
        k4[2] = y;
        k4[3] = d == 3 ? z : 0;
      }
  const int32_t n = L->n;
  auto unpack = [&](int64_t key, int64_t& x, int64_t& y, int64_t& z) {
    const int64_t nzv = g.nzv();
    z = key % nzv;
    y = (key / nzv) % (g.N + 1);
    x = key / (nzv * (g.N + 1));
  };
  // lattice-parity colour of own rows: 2^d independent sets of the Q1 stencil
  L->color.resize(static_cast<size_t>(n_own));
  for (int32_t i = 0; i < L->n_own; ++i) {
    int64_t x, y, z;
    unpack(L->vert[i], x, y, z);
    L->color[i] = static_cast<int32_t>(d == 3 ? ((x & 1) << 2) | ((y & 1) << 1) | (z & 1)
                                              : ((x & 1) << 1) | (y & 1));
  }

  // --- stiffness (assembly over own + halo cells, Dirichlet rows -> identity)
  const double h = 1.0 / static_cast<double>(g.N);
  const Element E = make_element(d, h);
  const int zr = d == 3 ? 1 : 0;
  std::vector<int64_t> rowlen(static_cast<size_t>(n) + 1, 0);
  auto shared_cells = [&](int64_t x, int64_t y, int64_t z, int dx, int dy, int dz, int64_t* cells) {
    // min corners of local cells containing both (x,y,z) and (x+dx,y+dy,z+dz), lex order
    int nc = 0;
    const int64_t jx = x + dx, jy = y + dy, jz = z + dz;
    for (int64_t cx = std::max(x, jx) - 1; cx <= std::min(x, jx); ++cx)
      for (int64_t cy = std::max(y, jy) - 1; cy <= std::min(y, jy); ++cy)
        for (int64_t cz = (d == 3 ? std::max(z, jz) - 1 : 0); cz <= (d == 3 ? std::min(z, jz) : 0); ++cz) {
          if (!V.cell_local(cx, cy, cz)) continue;
          cells[3 * nc] = cx;
          cells[3 * nc + 1] = cy;
          cells[3 * nc + 2] = cz;
          ++nc;
        }
    return nc;
  };
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < n; ++i) {
    int64_t x, y, z;
    unpack(L->vert[i], x, y, z);
    int64_t cells[24];
    int64_t cnt = 0;
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -zr; dz <= zr; ++dz)
          if (L->lookup(x + dx, y + dy, z + dz) >= 0 && shared_cells(x, y, z, dx, dy, dz, cells) > 0) ++cnt;
    rowlen[static_cast<size_t>(i) + 1] = cnt;
  }
  L->rowptr.assign(static_cast<size_t>(n) + 1, 0);
  for (int32_t i = 0; i < n; ++i) L->rowptr[i + 1] = L->rowptr[i] + rowlen[i + 1];
  L->cols.resize(static_cast<size_t>(L->rowptr[n]));
  L->vals.resize(static_cast<size_t>(L->rowptr[n]));
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < n; ++i) {
    int64_t x, y, z;
    unpack(L->vert[i], x, y, z);
    std::pair<int32_t, double> row[27];
    int nr = 0;
    int64_t cells[24];
    const bool dir = L->is_dir[i];
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -zr; dz <= zr; ++dz) {
          const int32_t j = L->lookup(x + dx, y + dy, z + dz);
          if (j < 0) continue;
          const int nc = shared_cells(x, y, z, dx, dy, dz, cells);
          if (nc == 0) continue;
          double v = 0.0;
          for (int c = 0; c < nc; ++c) {
            const int si = ring_slot(d, static_cast<int>(x - cells[3 * c]), static_cast<int>(y - cells[3 * c + 1]),
                                     static_cast<int>(z - cells[3 * c + 2]));
            const int sj = ring_slot(d, static_cast<int>(x + dx - cells[3 * c]), static_cast<int>(y + dy - cells[3 * c + 1]),
                                     static_cast<int>(z + dz - cells[3 * c + 2]));
            v += E.K[si][sj];
          }
          if (dir) v = (j == i) ? 1.0 : 0.0;  // apply_dirichlet_rows, assembly.cpp:162-170
          row[nr++] = {j, v};
        }
    std::sort(row, row + nr, [](const auto& a, const auto& b) { return a.first < b.first; });
    for (int k = 0; k < nr; ++k) {
      L->cols[static_cast<size_t>(L->rowptr[i] + k)] = row[k].first;
      L->vals[static_cast<size_t>(L->rowptr[i] + k)] = row[k].second;
    }
  }

  // --- channels: my requests (recv lists), then every other rank's requests to me
  std::vector<OwnedChannel> chans;
  auto chan = [&](int kind, int peer) -> OwnedChannel& {
    for (OwnedChannel& c : chans)
      if (c.kind == kind && c.peer == peer) return c;
    chans.push_back(OwnedChannel{kind, peer, {}, {}});
    return chans.back();
  };
  for (int64_t x = vb.lo[0]; x < vb.hi[0]; ++x)
    for (int64_t y = vb.lo[1]; y < vb.hi[1]; ++y)
      for (int64_t z = vb.lo[2]; z < vb.hi[2]; ++z) {
        const VInfo& v = info[static_cast<size_t>(vb.idx(x, y, z))];
        if (v.local && v.target >= 0) chan(v.kind, v.target).recv.push_back(L->lookup(x, y, z));
      }
  for (int r = 0; r < s.n_ranks; ++r) {
    if (r == me) continue;
    RankView W;
    W.build(g, r, region);
    for (int64_t x = vb.lo[0]; x < vb.hi[0]; ++x)
      for (int64_t y = vb.lo[1]; y < vb.hi[1]; ++y)
        for (int64_t z = vb.lo[2]; z < vb.hi[2]; ++z) {
          const VInfo v = classify(W, x, y, z);
          if (!v.local || v.target != me) continue;
          const int32_t li = L->lookup(x, y, z);
          if (li < 0) throw SetupError(PF_ERR_STATE, "request from a neighbour resolves to no local dof");
          chan(v.kind, r).send.push_back(li);
        }
  }
  std::sort(chans.begin(), chans.end(), [](const OwnedChannel& a, const OwnedChannel& b) {
    return a.kind != b.kind ? a.kind < b.kind : a.peer < b.peer;
  });
  L->channels = std::move(chans);
  for (OwnedChannel& c : L->channels)
    L->descs.push_back(pf_channel_desc{c.kind, c.peer, static_cast<int32_t>(c.send.size()),
                                       static_cast<int32_t>(c.recv.size()), c.send.data(), c.recv.data()});

  // --- prolongation from level l-1 (multigrid.cpp:35-72)
  if (l > 0) {
    const SetupLevel& C = *s.levels[static_cast<size_t>(l - 1)];
    L->p_off.assign(static_cast<size_t>(n) + 1, 0);
    std::vector<std::array<std::pair<int32_t, double>, 8>> rows(static_cast<size_t>(n));
    std::vector<int> cnt(static_cast<size_t>(n), 0);
    bool bad = false;
#pragma omp parallel for schedule(static)
    for (int32_t i = 0; i < n; ++i) {
      int64_t X[3];
      unpack(L->vert[i], X[0], X[1], X[2]);
      int64_t c[3] = {0, 0, 0};
      for (int a = 0; a < d; ++a)
        c[a] = (X[a] & 1) ? (X[a] - 1) / 2 : std::min<int64_t>(X[a] / 2, C.geo.N - 1);
      for (int v = 0; v < (1 << d); ++v) {
        double w = 1.0;
        int64_t corner[3] = {0, 0, 0};
        for (int a = 0; a < d; ++a) {
          corner[a] = c[a] + kRing[v][a];
          const double f = (X[a] & 1) ? 0.5 : (2 * corner[a] == X[a] ? 1.0 : 0.0);
          w *= f;
        }
        if (w == 0.0) continue;
        const int32_t cd = C.lookup(corner[0], corner[1], corner[2]);
        if (cd < 0) bad = true;
        rows[i][cnt[i]++] = {cd, w};
      }
    }
    if (bad) throw SetupError(PF_ERR_STATE, "prolongation parent dof is not local on the coarse level");
    for (int32_t i = 0; i < n; ++i) L->p_off[i + 1] = L->p_off[i] + cnt[i];
    L->p_col.resize(static_cast<size_t>(L->p_off[n]));
    L->p_w.resize(static_cast<size_t>(L->p_off[n]));
    for (int32_t i = 0; i < n; ++i)
      for (int k = 0; k < cnt[i]; ++k) {
        L->p_col[static_cast<size_t>(L->p_off[i] + k)] = rows[i][k].first;
        L->p_w[static_cast<size_t>(L->p_off[i] + k)] = rows[i][k].second;
      }
  }

  // --- finest level: load (own cells + master/slave accumulate) and rhs
  if (l == s.n_levels - 1) {
    s.b.assign(static_cast<size_t>(n), 0.0);
    s.x0.assign(static_cast<size_t>(n), 0.0);
    const double denom = static_cast<double>(g.N);
    auto partial = [&](int q, int64_t x, int64_t y, int64_t z) {
      // sum over cells around (x,y,z) owned by q, lexicographic, of the element load
      double acc = 0.0;
      const int zlo = d == 3 ? -1 : 0;
      for (int dx = -1; dx <= 0; ++dx)
        for (int dy = -1; dy <= 0; ++dy)
          for (int dz = zlo; dz <= 0; ++dz) {
            const int64_t cx = x + dx, cy = y + dy, cz = z + dz;
            if (!g.cell_in(cx, cy, cz) || g.owner(cx, cy, cz) != q) continue;
            const int slot = ring_slot(d, -dx, -dy, -dz);
            const double lo[3] = {static_cast<double>(cx) / denom, static_cast<double>(cy) / denom,
                                  d == 3 ? static_cast<double>(cz) / denom : 0.0};
            double load = 0.0;
            for (int q2 = 0; q2 < (1 << d); ++q2) {
              double xq[3] = {0.0, 0.0, 0.0};
              for (int a = 0; a < 3; ++a) xq[a] = lo[a] + E.qp[q2][a] * (a < d ? h : 1.0);
              const double fq = s.prob.f(xq);
              load += E.qw[q2] * fq * E.phi[q2][slot];
            }
            acc += load;
          }
      return acc;
    };
#pragma omp parallel for schedule(static)
    for (int32_t i = 0; i < n; ++i) {
      int64_t x, y, z;
      unpack(L->vert[i], x, y, z);
      const uint8_t c = L->class_of[i];
      double bi = 0.0;
      if (c == kDirichlet) {
        const double xc[3] = {static_cast<double>(x) / denom, static_cast<double>(y) / denom,
                              d == 3 ? static_cast<double>(z) / denom : 0.0};
        bi = s.prob.g(xc);  // apply_dirichlet_rhs, assembly.cpp:172-179
        s.x0[i] = bi;
      } else if (c == kMaster || c == kSlave) {
        const int m = g.master_of(x, y, z);
        int owners[8];
        const int no = g.owners_around(x, y, z, owners);
        bi = partial(m, x, y, z);
        for (int k = 0; k < no; ++k)
          if (owners[k] != m) bi += partial(owners[k], x, y, z);
      } else if (c <= kDep2) {
        bi = partial(me, x, y, z);
      }
      s.b[i] = bi;
    }
  }
  s.levels.push_back(std::move(L));
}

template <typename F>
pf_status guard(F&& f) {
  try {
    f();
    return PF_OK;
  } catch (const SetupError& e) {
    g_setup_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_setup_err = e.what();
    return PF_ERR_STATE;
  }
}

}  // namespace

extern "C" {

const char* pf_setup_last_error(void) { return g_setup_err.c_str(); }

pf_status pf_setup_create(int dim, int n_coarse, int n_levels, int n_ranks, int rank, int problem,
                          pf_setup** out) {
  return guard([&] {
    if (!out) invalid("null output");
    if (dim != 2 && dim != 3) invalid("dimension must be 2 or 3, got " + std::to_string(dim));
    if (n_coarse < 1) invalid("n_coarse must be >= 1");
    if (n_levels < 1) invalid("hierarchy needs at least one level");
    if (rank < 0 || rank >= n_ranks) invalid("rank out of range");
    if (problem < 0 || problem > 2) invalid("unknown problem");
    const auto t0 = std::chrono::steady_clock::now();
    auto s = std::make_unique<pf_setup>();
    s->d = dim;
    s->n_coarse = n_coarse;
    s->n_levels = n_levels;
    s->n_ranks = n_ranks;
    s->rank = rank;
    s->prob.kind = problem;
    s->prob.d = dim;
    s->coarse_owner = coarse_partition(dim, n_coarse, n_ranks);
    for (int l = 0; l < n_levels; ++l) build_level(*s, l);
    s->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = s.release();
  });
}

pf_status pf_setup_destroy(pf_setup* s) {
  delete s;
  return PF_OK;
}

pf_status pf_setup_level(const pf_setup* s, int level, pf_level_desc* out) {
  return guard([&] {
    if (!s || !out) invalid("null argument");
    if (level < 0 || level >= s->n_levels) invalid("level out of range");
    const SetupLevel& L = *s->levels[static_cast<size_t>(level)];
    std::memset(out, 0, sizeof *out);
    out->n_dofs = L.n;
    out->n_own_dofs = L.n_own;
    out->row_offsets = L.rowptr.data();
    out->col_indices = L.cols.data();
    out->values = L.vals.data();
    out->owns_row = L.owns_row.data();
    out->is_dirichlet = L.is_dir.data();
    out->color = L.color.data();
    out->n_channels = static_cast<int32_t>(L.descs.size());
    out->channels = L.descs.data();
    if (level > 0) {
      out->p_offsets = L.p_off.data();
      out->p_cols = L.p_col.data();
      out->p_weights = L.p_w.data();
    }
  });
}

pf_status pf_setup_level_keys(const pf_setup* s, int level, const int64_t** keys4, const uint8_t** class_of) {
  return guard([&] {
    if (!s) invalid("null setup");
    if (level < 0 || level >= s->n_levels) invalid("level out of range");
    const SetupLevel& L = *s->levels[static_cast<size_t>(level)];
    if (keys4) *keys4 = L.keys4.data();
    if (class_of) *class_of = L.class_of.data();
  });
}

pf_status pf_setup_rhs(const pf_setup* s, const double** b, const double** x0, int64_t* n) {
  return guard([&] {
    if (!s) invalid("null setup");
    if (b) *b = s->b.data();
    if (x0) *x0 = s->x0.data();
    if (n) *n = static_cast<int64_t>(s->b.size());
  });
}

pf_status pf_setup_counts(const pf_setup* s, int level, int64_t* n_global, int64_t* n_dofs, int64_t* n_own,
                          int64_t* nnz) {
  return guard([&] {
    if (!s) invalid("null setup");
    if (level < 0 || level >= s->n_levels) invalid("level out of range");
    const SetupLevel& L = *s->levels[static_cast<size_t>(level)];
    const int64_t nv = L.geo.N + 1;
    if (n_global) *n_global = s->d == 3 ? nv * nv * nv : nv * nv;
    if (n_dofs) *n_dofs = L.n;
    if (n_own) *n_own = L.n_own;
    if (nnz) *nnz = L.rowptr.empty() ? 0 : L.rowptr.back();
  });
}

pf_status pf_setup_seconds(const pf_setup* s, double* out) {
  return guard([&] {
    if (!s || !out) invalid("null argument");
    *out = s->seconds;
  });
}

}  // extern "C"
