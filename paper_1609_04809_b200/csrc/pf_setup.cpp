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

#include "pf_runtime.hpp"

#include <algorithm>
#include <parallel/algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "pf_coef.hpp"

namespace {

struct SetupError : std::runtime_error {
  pf_status code;
  SetupError(pf_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void invalid(const std::string& m) { throw SetupError(PF_ERR_INVALID_ARGUMENT, m); }
[[noreturn]] void state_error(const std::string& m) { throw SetupError(PF_ERR_STATE, m); }

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

  // Vertex coordinate along one axis as the reference stores it: level 0 from the unit
  // mesh (mesh.cpp:73,87: i * (1/n)), refined levels from the lattice (partition.cpp:331).
  double coord(int64_t i) const {
    return level == 0 ? static_cast<double>(i) * (1.0 / static_cast<double>(N))
                      : static_cast<double>(i) / static_cast<double>(N);
  }
  // Cell extent (element_matrices takes hi - lo per axis, assembly.cpp:51-58).
  double extent(int64_t c) const { return coord(c + 1) - coord(c); }
  // Global cell number: coarse cells lexicographic (mesh.cpp:93-100), children
  // nc * parent + child index with child offset (c/4, c/2 % 2, c % 2) (mesh.cpp:36-42,
  // :170-176).  Local cells are visited in ascending gcn (partition.cpp:184-186, :296-298),
  // which fixes the order every assembled sum is accumulated in.
  int64_t gcn(int64_t x, int64_t y, int64_t z) const {
    const int64_t n = n_coarse;
    int64_t g = d == 3 ? ((x / S) * n + (y / S)) * n + (z / S) : (x / S) * n + (y / S);
    for (int b = level - 1; b >= 0; --b) {
      const int64_t ci = d == 3 ? (((x >> b) & 1) << 2) | (((y >> b) & 1) << 1) | ((z >> b) & 1)
                                : (((x >> b) & 1) << 1) | ((y >> b) & 1);
      g = g * (int64_t(1) << d) + ci;
    }
    return g;
  }
  int64_t nzc() const { return d == 3 ? N : 1; }     // cells along z
  int64_t nzv() const { return d == 3 ? N + 1 : 1; } // vertices along z
  int64_t vkey(int64_t x, int64_t y, int64_t z) const { return (x * (N + 1) + y) * nzv() + z; }
  void unpack(int64_t key, int64_t& x, int64_t& y, int64_t& z) const {
    z = key % nzv();
    y = (key / nzv()) % (N + 1);
    x = key / (nzv() * (N + 1));
  }
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
// direct: halo requests for a carrier the owner holds as Slave go to its Master instead
// (the value the Slave would forward after the master/slave scatter), so the Halo1/Halo2
// exchanges no longer depend on the master/slave one and can share its message group.
VInfo classify(const RankView& V, int64_t x, int64_t y, int64_t z, bool direct = false) {
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
    if (direct && master >= 0 && master != owners[0]) info.target = master;
  }
  return info;
}

struct OwnedChannel {
  int kind = 0, peer = 0;
  std::vector<int32_t> send, recv;
};

// Q1 element matrices on an axis-aligned cell with extents h[0..d), 2-point Gauss
// (assembly.cpp:11-92): stiffness K, mass M, and what the load needs per quadrature point.
struct Element {
  int nv = 8, nq = 8;
  double K[8][8] = {};
  double M[8][8] = {};
  double qp[8][3] = {};   // quadrature points (reference cell)
  double qw[8] = {};      // weight * volume
  double phi[8][8] = {};  // phi[q][v]
  double h[3] = {1.0, 1.0, 1.0};
};

Element make_element(int d, const double* hx) {
  Element E;
  E.nv = 1 << d;
  E.nq = 1 << d;
  const double off = 0.5 / std::sqrt(3.0);
  const double pts[2] = {0.5 - off, 0.5 + off};
  double volume = 1.0;
  for (int a = 0; a < d; ++a) {
    E.h[a] = hx[a];
    volume *= E.h[a];
  }
  const double* hh = E.h;
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
            E.M[i][j] += E.qw[q] * E.phi[q][i] * E.phi[q][j];
          }
      }
  return E;
}

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
  // per local dof: which of the 2^d cells around the vertex are local (finest level; bit k
  // <-> cell with low corner = vertex along axis a iff bit a of k), for device assembly
  std::vector<uint8_t> cell_mask;
  // element matrices per distinct cell shape (extents differ in the last bit across cells
  // unless N is a power of two)
  std::vector<Element> elems;
  std::vector<int> hid;  // per cell index along an axis: its extent's slot
  int nh = 0;
  int32_t lookup(int64_t x, int64_t y, int64_t z) const {
    return vbox.in(x, y, z) ? index[vbox.idx(x, y, z)] : -1;
  }
  const Element& elem(int64_t cx, int64_t cy, int64_t cz) const {
    const int e = geo.d == 3 ? (hid[cx] * nh + hid[cy]) * nh + hid[cz] : hid[cx] * nh + hid[cy];
    return elems[static_cast<size_t>(e)];
  }
};

int ring_slot(int d, int ox, int oy, int oz) {
  for (int v = 0; v < (1 << d); ++v)
    if (kRing[v][0] == ox && kRing[v][1] == oy && (d == 2 || kRing[v][2] == oz)) return v;
  return -1;
}

// The manufactured fields as the reference evaluates them.  Every source and boundary
// field here is "scalar(t) * profile(x)" with profile = F0(pi x) * F1(pi y) [* F2(pi z)]
// multiplied left to right, so a device kernel holding per-axis factor tables and the
// host-computed scalar reproduces each product bit for bit.
struct Problem {
  int kind = 0, d = 3;
  double dt = 0.0;
  uint64_t seed = 0;  // PF_PROBLEM_LOGNORMAL
  bool unit() const { return kind == PF_PROBLEM_UNIT_SOURCE; }
  // axis factor a of the profile: sin for axis 0 (and every axis of BASELINE), else cos
  bool axis_sin(int a) const { return a == 0 || kind == PF_PROBLEM_BASELINE || kind == PF_PROBLEM_LOGNORMAL; }
  double profile(const double* x) const {
    if (unit()) return 1.0;
    double u = (axis_sin(0) ? std::sin(kPi * x[0]) : std::cos(kPi * x[0])) *
               (axis_sin(1) ? std::sin(kPi * x[1]) : std::cos(kPi * x[1]));  // model.cpp:12-16
    if (d == 3) u *= axis_sin(2) ? std::sin(kPi * x[2]) : std::cos(kPi * x[2]);
    return u;
  }
  // f(t, x) = source_scale(t) * profile(x)
  double source_scale(double t) const {
    if (unit()) return 1.0;
    if (kind == PF_PROBLEM_HEAT) return (-0.1 + d * kPi * kPi) * std::exp(-0.1 * t);  // model.cpp:24-29
    return d * kPi * kPi;                                                                // model.cpp:38-41
  }
  // g(t, x) = dirichlet_scale(t) * profile(x), or exactly 0 when !has_dirichlet()
  bool has_dirichlet() const { return kind == PF_PROBLEM_REFERENCE_POISSON || kind == PF_PROBLEM_HEAT; }
  double dirichlet_scale(double t) const { return kind == PF_PROBLEM_HEAT ? std::exp(-0.1 * t) : 1.0; }
  double f(double t, const double* x) const { return source_scale(t) * profile(x); }
  double g(double t, const double* x) const {
    if (!has_dirichlet()) return 0.0;
    if (kind == PF_PROBLEM_HEAT) return std::exp(-0.1 * t) * profile(x);  // model.cpp:19-22
    return profile(x);
  }
};

}  // namespace

struct pf_setup {
  int d = 3, n_coarse = 2, n_levels = 1, n_ranks = 1, rank = 0;
  bool direct_halos = false;  // pf_setup_options::direct_halos
  Problem prob;
  std::vector<int> coarse_owner;
  std::vector<std::unique_ptr<SetupLevel>> levels;
  std::vector<double> b, x0;
  std::vector<double> rhs_op;  // heat: finest-level M - dt/2 K in the system's CSR order
  // device load description of the finest level (pf_load_desc)
  std::vector<int32_t> ld_lattice;
  std::vector<uint32_t> ld_cells;
  std::vector<double> ld_factor, ld_extent, ld_phi, ld_boundary;
  // PF_PROBLEM_LOGNORMAL: kappa of every finest cell (lexicographic), and the element
  // matrices (8 x 8, row-major) of every cell of each coarser level
  std::vector<double> kappa;
  std::vector<std::vector<double>> coef_elem;
  // device assembly description of the finest level (pf_assembly_desc)
  std::vector<double> asm_elem;
  std::vector<int32_t> asm_hid;
  bool matrices_released = false;  // pf_setup_release_matrices
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

// ------------------------------------------------------- lognormal coefficient --
//
// PF_PROBLEM_LOGNORMAL (BASELINE configs 3-4; not in the reference):
// kappa_c = exp(z_c), z_c ~ N(0, 1) drawn per finest cell from a counter-based generator
// keyed by (seed, finest gcn) — independent of the partition.  The finest element matrix
// is kappa_c * K_e; a coarse cell's element matrix is the Galerkin product of its
// children's, E_C = sum_{children c, child index order} P_c^T E_c P_c, with P_c the exact
// trilinear interpolation of the coarse cell's basis at the child's vertices (for nested
// conforming Q1 spaces this is the rediscretisation with the fine coefficient).

using pf::lognormal_kappa;

Geo geo_of(int d, int n_coarse, int level) {
  Geo g;
  g.d = d;
  g.n_coarse = n_coarse;
  g.level = level;
  g.S = int64_t(1) << level;
  g.N = static_cast<int64_t>(n_coarse) * g.S;
  return g;
}

void build_coefficients(pf_setup& s) {
  const int d = s.d, nv = 1 << d, L = s.n_levels;
  const Geo gf = geo_of(d, s.n_coarse, L - 1);
  const int64_t N = gf.N, nz = d == 3 ? N : 1;
  s.kappa.assign(static_cast<size_t>(N * N * nz), 0.0);
#pragma omp parallel for schedule(static) collapse(2)
  for (int64_t x = 0; x < N; ++x)
    for (int64_t y = 0; y < N; ++y)
      for (int64_t z = 0; z < nz; ++z)
        s.kappa[static_cast<size_t>((x * N + y) * nz + z)] = lognormal_kappa(s.prob.seed, gf.gcn(x, y, z));
  // interpolation of the parent's ring basis at child ci's ring vertices: P[ci][k][i]
  std::vector<double> P(static_cast<size_t>(8 * 8 * 8), 0.0);
  for (int ci = 0; ci < nv; ++ci) {
    const int o[3] = {d == 3 ? ci >> 2 : ci >> 1, d == 3 ? (ci >> 1) & 1 : ci & 1, d == 3 ? ci & 1 : 0};
    for (int k = 0; k < nv; ++k)
      for (int i = 0; i < nv; ++i) {
        double w = 1.0;
        for (int a = 0; a < d; ++a) {
          const double xi = static_cast<double>(o[a] + kRing[k][a]) / 2.0;
          w *= kRing[i][a] ? xi : 1.0 - xi;
        }
        P[static_cast<size_t>((ci * 8 + k) * 8 + i)] = w;
      }
  }
  s.coef_elem.assign(static_cast<size_t>(L), {});
  for (int l = L - 2; l >= 0; --l) {
    const Geo gc = geo_of(d, s.n_coarse, l);
    const int64_t Nc = gc.N, nzc = d == 3 ? Nc : 1, nzf = d == 3 ? 2 * Nc : 1;
    std::vector<double>& EC = s.coef_elem[static_cast<size_t>(l)];
    EC.assign(static_cast<size_t>(Nc * Nc * nzc * 64), 0.0);
    const bool child_finest = l + 1 == L - 1;
    // the finest children's K_e depends on their extents (last bit, N not a power of two)
    std::vector<double> hv;
    std::vector<int> hidf;
    std::vector<Element> ef;
    if (child_finest) {
      hidf.assign(static_cast<size_t>(N), 0);
      for (int64_t c = 0; c < N; ++c) {
        const double e = gf.extent(c);
        size_t k = 0;
        while (k < hv.size() && hv[k] != e) ++k;
        if (k == hv.size()) hv.push_back(e);
        hidf[static_cast<size_t>(c)] = static_cast<int>(k);
      }
      const int nh = static_cast<int>(hv.size());
      for (int a = 0; a < nh; ++a)
        for (int b = 0; b < nh; ++b)
          for (int c = 0; c < (d == 3 ? nh : 1); ++c) {
            const double hx[3] = {hv[a], hv[b], d == 3 ? hv[c] : 1.0};
            ef.push_back(make_element(d, hx));
          }
    }
    const int nh = static_cast<int>(hv.size());
    const std::vector<double>& EF = child_finest ? s.kappa : s.coef_elem[static_cast<size_t>(l + 1)];
#pragma omp parallel for schedule(static) collapse(2)
    for (int64_t X = 0; X < Nc; ++X)
      for (int64_t Y = 0; Y < Nc; ++Y)
        for (int64_t Z = 0; Z < nzc; ++Z) {
          double* out = &EC[static_cast<size_t>(((X * Nc + Y) * nzc + Z) * 64)];
          for (int ci = 0; ci < nv; ++ci) {
            const int o[3] = {d == 3 ? ci >> 2 : ci >> 1, d == 3 ? (ci >> 1) & 1 : ci & 1, d == 3 ? ci & 1 : 0};
            const int64_t cx = 2 * X + o[0], cy = 2 * Y + o[1], cz = d == 3 ? 2 * Z + o[2] : 0;
            const int64_t cidx = (cx * (2 * Nc) + cy) * nzf + cz;
            double E[64];
            if (child_finest) {
              const int e = d == 3 ? (hidf[cx] * nh + hidf[cy]) * nh + hidf[cz] : hidf[cx] * nh + hidf[cy];
              const double kap = EF[static_cast<size_t>(cidx)];
              for (int k = 0; k < nv; ++k)
                for (int m = 0; m < nv; ++m) E[k * 8 + m] = kap * ef[static_cast<size_t>(e)].K[k][m];
            } else {
              for (int q = 0; q < 64; ++q) E[q] = EF[static_cast<size_t>(cidx * 64 + q)];
            }
            const double* Pc = &P[static_cast<size_t>(ci * 64)];
            double T[64];
            for (int k = 0; k < nv; ++k)
              for (int j = 0; j < nv; ++j) {
                double t = 0.0;
                for (int m = 0; m < nv; ++m) t += E[k * 8 + m] * Pc[m * 8 + j];
                T[k * 8 + j] = t;
              }
            for (int i = 0; i < nv; ++i)
              for (int j = 0; j < nv; ++j) {
                double u = 0.0;
                for (int k = 0; k < nv; ++k) u += Pc[k * 8 + i] * T[k * 8 + j];
                out[i * 8 + j] += u;
              }
          }
        }
  }
}

// Element-matrix entry (si, sj) of cell (cx, cy, cz) of level l for the coefficient problem.
double coef_entry(const pf_setup& s, const SetupLevel& L, int l, int64_t cx, int64_t cy, int64_t cz, int si,
                  int sj) {
  const int64_t N = L.geo.N, nz = s.d == 3 ? N : 1;
  const int64_t c = (cx * N + cy) * nz + cz;
  if (l == s.n_levels - 1) return s.kappa[static_cast<size_t>(c)] * L.elem(cx, cy, cz).K[si][sj];
  return s.coef_elem[static_cast<size_t>(l)][static_cast<size_t>(c * 64 + si * 8 + sj)];
}

// Cells given as (x, y, z) triples, reordered by ascending gcn (at most 8).
void sort_cells_by_gcn(const Geo& g, int64_t* cells, int nc) {
  int64_t key[8];
  for (int c = 0; c < nc; ++c) key[c] = g.gcn(cells[3 * c], cells[3 * c + 1], cells[3 * c + 2]);
  for (int i = 1; i < nc; ++i)
    for (int j = i; j > 0 && key[j - 1] > key[j]; --j) {
      std::swap(key[j - 1], key[j]);
      for (int a = 0; a < 3; ++a) std::swap(cells[3 * (j - 1) + a], cells[3 * j + a]);
    }
}

// The cells around vertex (x, y, z) owned by rank q, in gcn order; returns the count.
int owned_cells_around(const Geo& g, int q, int64_t x, int64_t y, int64_t z, int64_t* cells) {
  int nc = 0;
  const int zlo = g.d == 3 ? -1 : 0;
  for (int dx = -1; dx <= 0; ++dx)
    for (int dy = -1; dy <= 0; ++dy)
      for (int dz = zlo; dz <= 0; ++dz) {
        const int64_t cx = x + dx, cy = y + dy, cz = z + dz;
        if (!g.cell_in(cx, cy, cz) || g.owner(cx, cy, cz) != q) continue;
        cells[3 * nc] = cx;
        cells[3 * nc + 1] = cy;
        cells[3 * nc + 2] = cz;
        ++nc;
      }
  sort_cells_by_gcn(g, cells, nc);
  return nc;
}

// Rank q's share of the load at vertex (x, y, z) at time t: its own cells in gcn order,
// each cell's element load summed over the quadrature points (assembly.cpp:60-88,
// :144-160).
double load_partial(const Problem& P, const SetupLevel& L, int q, int64_t x, int64_t y, int64_t z, double t) {
  const Geo& g = L.geo;
  const int d = g.d;
  int64_t cells[24];
  const int nc = owned_cells_around(g, q, x, y, z, cells);
  double acc = 0.0;
  for (int c = 0; c < nc; ++c) {
    const int64_t* cc = &cells[3 * c];
    const Element& E = L.elem(cc[0], cc[1], cc[2]);
    const int slot = ring_slot(d, static_cast<int>(x - cc[0]), static_cast<int>(y - cc[1]),
                               static_cast<int>(z - cc[2]));
    const double lo[3] = {g.coord(cc[0]), g.coord(cc[1]), d == 3 ? g.coord(cc[2]) : 0.0};
    double load = 0.0;
    for (int q2 = 0; q2 < E.nq; ++q2) {
      double xq[3];
      for (int a = 0; a < 3; ++a) xq[a] = lo[a] + E.qp[q2][a] * E.h[a];
      const double fq = P.f(t, xq);
      load += E.qw[q2] * fq * E.phi[q2][slot];
    }
    acc += load;
  }
  return acc;
}

// Finest-level load at time t after the master/slave accumulate-then-scatter
// (fecomm.cpp:41-62: masters add the slaves' parts in ascending rank order, slaves take
// the sum).  Dirichlet rows are left 0: the caller overwrites them with boundary data.
void finest_load(const pf_setup& s, double t, double* out);
void finish_finest(pf_setup& s);

void build_level(pf_setup& s, int l) {
  const bool timing = std::getenv("PF_TIMING") != nullptr;
  auto tick = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[pf_timing]   setup level %d %-16s %8.3f s\n", l, what,
                 std::chrono::duration<double>(now - tick).count());
    tick = now;
  };
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
      for (int64_t z = vb.lo[2]; z < vb.hi[2]; ++z) info[vb.idx(x, y, z)] = classify(V, x, y, z, s.direct_halos);

  lap("classify");
  // --- numbering: the reference's own.  build_fespace numbers vertices at first touch
  // over the local cells in gcn order, ring-slot order inside a cell (fespace.cpp:47-85);
  // build_parfemapper then stable-sorts that numbering by DofClass value
  // (femapper.cpp:167-199).  So local index order = (class, gcn of the lowest local cell
  // containing the vertex, the vertex's slot in it) — which makes every row's column
  // order, the restriction's scatter-add order and the coarse Gauss-Seidel order the
  // reference's, and with them the floating-point results.
  L->index.assign(static_cast<size_t>(nvb), -1);
  int64_t count[8] = {};
  for (const VInfo& v : info)
    if (v.local) ++count[v.cls];
  const int64_t n_own = count[kMaster] + count[kIndep] + count[kDep1] + count[kDep2];
  int64_t total = 0;
  for (int64_t c : count) total += c;
  if (total >= (int64_t(1) << 31)) invalid("local level too large for int32 indices");
  struct Order {
    int64_t key;  // class << 60 | first-touch rank
    int64_t bi;
  };
  std::vector<Order> order;
  order.reserve(static_cast<size_t>(total));
  for (int64_t bi = 0; bi < nvb; ++bi)
    if (info[static_cast<size_t>(bi)].local) order.push_back({0, bi});
  const int zlo = d == 3 ? -1 : 0;
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < static_cast<int64_t>(order.size()); ++k) {
    const int64_t bi = order[static_cast<size_t>(k)].bi;
    const int64_t ez = vb.ext(2), ey = vb.ext(1);
    const int64_t x = vb.lo[0] + bi / (ey * ez), y = vb.lo[1] + (bi / ez) % ey, z = vb.lo[2] + bi % ez;
    int64_t best = -1;
    int slot = 0;
    for (int dx = -1; dx <= 0; ++dx)
      for (int dy = -1; dy <= 0; ++dy)
        for (int dz = zlo; dz <= 0; ++dz) {
          const int64_t cx = x + dx, cy = y + dy, cz = z + dz;
          if (!V.cell_local(cx, cy, cz)) continue;
          const int64_t gc = g.gcn(cx, cy, cz);
          if (best < 0 || gc < best) {
            best = gc;
            slot = ring_slot(d, -dx, -dy, -dz);
          }
        }
    order[static_cast<size_t>(k)].key =
        (static_cast<int64_t>(info[static_cast<size_t>(bi)].cls) << 59) | (best * 8 + slot);
  }
  __gnu_parallel::sort(order.begin(), order.end(), [](const Order& a, const Order& b) { return a.key < b.key; });
  L->n = static_cast<int32_t>(total);
  L->n_own = static_cast<int32_t>(n_own);
  L->vert.resize(static_cast<size_t>(total));
  L->class_of.resize(static_cast<size_t>(total));
  L->owns_row.resize(static_cast<size_t>(total));
  L->is_dir.resize(static_cast<size_t>(total));
  L->keys4.resize(static_cast<size_t>(4 * total));
#pragma omp parallel for schedule(static)
  for (int64_t li = 0; li < total; ++li) {
    const int64_t bi = order[static_cast<size_t>(li)].bi;
    const int64_t ez = vb.ext(2), ey = vb.ext(1);
    const int64_t x = vb.lo[0] + bi / (ey * ez), y = vb.lo[1] + (bi / ez) % ey, z = vb.lo[2] + bi % ez;
    const VInfo& v = info[static_cast<size_t>(bi)];
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
  auto unpack = [&](int64_t key, int64_t& x, int64_t& y, int64_t& z) { g.unpack(key, x, y, z); };
  // lattice-parity colour of own rows: 2^d independent sets of the Q1 stencil
  L->color.resize(static_cast<size_t>(n_own));
  for (int32_t i = 0; i < L->n_own; ++i) {
    int64_t x, y, z;
    unpack(L->vert[i], x, y, z);
    L->color[i] = static_cast<int32_t>(d == 3 ? ((x & 1) << 2) | ((y & 1) << 1) | (z & 1)
                                              : ((x & 1) << 1) | (y & 1));
  }

  lap("numbering");
  // --- element matrices per distinct cell shape
  std::vector<double> hvals;
  L->hid.assign(static_cast<size_t>(g.N), 0);
  for (int64_t c = 0; c < g.N; ++c) {
    const double e = g.extent(c);
    size_t k = 0;
    while (k < hvals.size() && hvals[k] != e) ++k;
    if (k == hvals.size()) hvals.push_back(e);
    L->hid[static_cast<size_t>(c)] = static_cast<int>(k);
  }
  L->nh = static_cast<int>(hvals.size());
  for (int a = 0; a < L->nh; ++a)
    for (int b = 0; b < L->nh; ++b)
      for (int c = 0; c < (d == 3 ? L->nh : 1); ++c) {
        const double hx[3] = {hvals[a], hvals[b], d == 3 ? hvals[c] : 1.0};
        L->elems.push_back(make_element(d, hx));
      }
  const SetupLevel& LC = *L;
  auto elem = [&](int64_t cx, int64_t cy, int64_t cz) -> const Element& { return LC.elem(cx, cy, cz); };
  auto sort_by_gcn = [&](int64_t* cells, int nc) { sort_cells_by_gcn(g, cells, nc); };
  const bool heat = s.prob.kind == PF_PROBLEM_HEAT;
  const bool coef = s.prob.kind == PF_PROBLEM_LOGNORMAL;
  const bool finest = l == s.n_levels - 1;
  const double half_dt = 0.5 * s.prob.dt;

  lap("elements");
  // --- system (assembly over own + halo cells in gcn order, assembly.cpp:114-131);
  // heat: M + dt/2 K (multigrid.cpp:18-28); Dirichlet rows -> identity (:162-170)
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
    sort_by_gcn(cells, nc);
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
  if (finest) {
    L->cell_mask.assign(static_cast<size_t>(n), 0);
#pragma omp parallel for schedule(static)
    for (int32_t i = 0; i < n; ++i) {
      int64_t x, y, z;
      unpack(L->vert[i], x, y, z);
      uint8_t m = 0;
      for (int k = 0; k < (1 << d); ++k) {
        const int64_t cx = x - 1 + (k & 1), cy = y - 1 + ((k >> 1) & 1), cz = d == 3 ? z - 1 + ((k >> 2) & 1) : 0;
        if (V.cell_local(cx, cy, cz)) m |= static_cast<uint8_t>(1u << k);
      }
      L->cell_mask[static_cast<size_t>(i)] = m;
    }
  }
  const int64_t nnz = L->rowptr[n];
  L->cols.resize(static_cast<size_t>(nnz));
  L->vals.resize(static_cast<size_t>(nnz));
  if (heat && finest) s.rhs_op.resize(static_cast<size_t>(nnz));
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < n; ++i) {
    int64_t x, y, z;
    unpack(L->vert[i], x, y, z);
    struct Ent {
      int32_t j;
      double sys, rhs;
    } row[27];
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
          double k = 0.0, m = 0.0;
          for (int c = 0; c < nc; ++c) {
            const int64_t* cc = &cells[3 * c];
            const int si = ring_slot(d, static_cast<int>(x - cc[0]), static_cast<int>(y - cc[1]),
                                     static_cast<int>(z - cc[2]));
            const int sj = ring_slot(d, static_cast<int>(x + dx - cc[0]), static_cast<int>(y + dy - cc[1]),
                                     static_cast<int>(z + dz - cc[2]));
            const Element& E = elem(cc[0], cc[1], cc[2]);
            k += coef ? coef_entry(s, LC, l, cc[0], cc[1], cc[2], si, sj) : E.K[si][sj];
            if (heat) m += E.M[si][sj];
          }
          double v = heat ? m + half_dt * k : k;
          // heat rhs operator M - dt/2 K on raw rows (app.cpp:185-189)
          const double r = heat ? m - half_dt * k : 0.0;
          if (dir) v = (j == i) ? 1.0 : 0.0;  // apply_dirichlet_rows, assembly.cpp:162-170
          row[nr++] = {j, v, r};
        }
    std::sort(row, row + nr, [](const Ent& a, const Ent& b) { return a.j < b.j; });
    for (int e = 0; e < nr; ++e) {
      const size_t at = static_cast<size_t>(L->rowptr[i] + e);
      L->cols[at] = row[e].j;
      L->vals[at] = row[e].sys;
      if (heat && finest) s.rhs_op[at] = row[e].rhs;
    }
  }

  lap("system");
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
          const VInfo v = classify(W, x, y, z, s.direct_halos);
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

  lap("channels");
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
      // parent of the dof's home cell: the lowest-gcn local fine cell containing it
      // (multigrid.cpp:43-55); its ring order fixes the order of the row's entries
      int64_t home[3] = {0, 0, 0}, best = -1;
      for (int dx = -1; dx <= 0; ++dx)
        for (int dy = -1; dy <= 0; ++dy)
          for (int dz = (d == 3 ? -1 : 0); dz <= 0; ++dz) {
            const int64_t cx = X[0] + dx, cy = X[1] + dy, cz = X[2] + dz;
            if (!V.cell_local(cx, cy, cz)) continue;
            const int64_t gc = g.gcn(cx, cy, cz);
            if (best < 0 || gc < best) {
              best = gc;
              home[0] = cx;
              home[1] = cy;
              home[2] = cz;
            }
          }
      if (best < 0) bad = true;
      int64_t c[3] = {0, 0, 0};
      for (int a = 0; a < d; ++a) c[a] = home[a] >> 1;
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

  lap("prolongation");
  s.levels.push_back(std::move(L));
  if (l == s.n_levels - 1) finish_finest(s);
  lap("finish");
}

void finest_load(const pf_setup& s, double t, double* out) {
  const SetupLevel& L = *s.levels.back();
  const Geo& g = L.geo;
  const int me = s.rank;
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < L.n; ++i) {
    int64_t x, y, z;
    g.unpack(L.vert[i], x, y, z);
    const uint8_t c = L.class_of[i];
    double bi = 0.0;
    if (c == kMaster || c == kSlave) {
      const int m = g.master_of(x, y, z);
      int owners[8];
      const int no = g.owners_around(x, y, z, owners);
      bi = load_partial(s.prob, L, m, x, y, z, t);
      for (int k = 0; k < no; ++k)
        if (owners[k] != m) bi += load_partial(s.prob, L, owners[k], x, y, z, t);
    } else if (c <= kDep2) {
      bi = load_partial(s.prob, L, me, x, y, z, t);
    }
    out[i] = bi;
  }
}

// Finest level: rhs and start vector.  Poisson kinds: b = load with the Dirichlet rhs
// applied, x0 = boundary data on Dirichlet rows, 0 elsewhere (app.cpp:253-260).  Heat:
// b = the load at t = 0 (app.cpp:178), x0 = the exact solution at t = 0 on every dof
// (app.cpp:173-176).
void finish_finest(pf_setup& s) {
  const SetupLevel& L = *s.levels.back();
  const Geo& g = L.geo;
  const int32_t n = L.n;
  s.b.assign(static_cast<size_t>(n), 0.0);
  s.x0.assign(static_cast<size_t>(n), 0.0);
  finest_load(s, 0.0, s.b.data());
  const bool heat = s.prob.kind == PF_PROBLEM_HEAT;
  const double denom = static_cast<double>(g.N);
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < n; ++i) {
    int64_t x, y, z;
    g.unpack(L.vert[i], x, y, z);
    // dof coordinates key / denom (fespace.cpp:66-70)
    const double xc[3] = {static_cast<double>(x) / denom, static_cast<double>(y) / denom,
                          g.d == 3 ? static_cast<double>(z) / denom : 0.0};
    if (heat) {
      s.x0[i] = s.prob.g(0.0, xc);
    } else if (L.class_of[i] == kDirichlet) {
      s.b[i] = s.prob.g(0.0, xc);  // apply_dirichlet_rhs, assembly.cpp:172-179
      s.x0[i] = s.b[i];
    }
  }

  // --- device load description (pf_load_desc)
  const int d = g.d;
  const int64_t N = g.N;
  s.ld_lattice.resize(static_cast<size_t>(3 * n));
  s.ld_cells.assign(static_cast<size_t>(n), 0u);
  s.ld_boundary.assign(static_cast<size_t>(n), 0.0);
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < n; ++i) {
    int64_t x, y, z;
    g.unpack(L.vert[i], x, y, z);
    s.ld_lattice[3 * static_cast<size_t>(i)] = static_cast<int32_t>(x);
    s.ld_lattice[3 * static_cast<size_t>(i) + 1] = static_cast<int32_t>(y);
    s.ld_lattice[3 * static_cast<size_t>(i) + 2] = static_cast<int32_t>(z);
    const double xc[3] = {static_cast<double>(x) / denom, static_cast<double>(y) / denom,
                          d == 3 ? static_cast<double>(z) / denom : 0.0};
    s.ld_boundary[i] = s.prob.profile(xc);
    if (L.class_of[i] == kDirichlet) continue;
    int64_t cells[24];
    const int nc = owned_cells_around(g, s.rank, x, y, z, cells);
    uint32_t w = static_cast<uint32_t>(nc);
    for (int c = 0; c < nc; ++c) {
      const uint32_t bits = (cells[3 * c] == x ? 1u : 0u) | (cells[3 * c + 1] == y ? 2u : 0u) |
                            (d == 3 && cells[3 * c + 2] == z ? 4u : 0u);
      w |= bits << (4 + 3 * c);
    }
    s.ld_cells[i] = w;
  }
  s.ld_factor.assign(static_cast<size_t>(3 * N * 2), 1.0);
  s.ld_extent.assign(static_cast<size_t>(3 * N), 1.0);
  const Element& E0 = L.elems.front();
  for (int a = 0; a < d; ++a)
    for (int64_t c = 0; c < N; ++c) {
      const double lo = g.coord(c), h = g.extent(c);
      s.ld_extent[static_cast<size_t>(a * N + c)] = h;
      for (int k = 0; k < 2; ++k) {
        const double xq = lo + E0.qp[k == 0 ? 0 : E0.nq - 1][0] * h;  // Gauss point k (q = 0 / last)
        double f = 1.0;
        if (!s.prob.unit()) f = s.prob.axis_sin(a) ? std::sin(kPi * xq) : std::cos(kPi * xq);
        s.ld_factor[static_cast<size_t>((a * N + c) * 2 + k)] = f;
      }
    }
  s.ld_phi.assign(64, 0.0);
  for (int q = 0; q < E0.nq; ++q)
    for (int v = 0; v < E0.nv; ++v) s.ld_phi[static_cast<size_t>(q * 8 + v)] = E0.phi[q][v];
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

pf_status create(int dim, int n_coarse, int n_levels, int n_ranks, int rank, int problem, double dt,
                 uint64_t seed, pf_setup** out, bool direct_halos = false) {
  return guard([&] {
    if (!out) invalid("null output");
    if (dim != 2 && dim != 3) invalid("dimension must be 2 or 3, got " + std::to_string(dim));
    if (n_coarse < 1) invalid("n_coarse must be >= 1");
    if (n_levels < 1) invalid("hierarchy needs at least one level");
    if (rank < 0 || rank >= n_ranks) invalid("rank out of range");
    if (problem < 0 || problem > 4) invalid("unknown problem");
    if (problem == PF_PROBLEM_HEAT && !(dt > 0.0)) invalid("dt must be positive");  // config.cpp:86
    const auto t0 = std::chrono::steady_clock::now();
    auto s = std::make_unique<pf_setup>();
    s->d = dim;
    s->n_coarse = n_coarse;
    s->n_levels = n_levels;
    s->n_ranks = n_ranks;
    s->rank = rank;
    s->prob.kind = problem;
    s->prob.d = dim;
    s->prob.dt = problem == PF_PROBLEM_HEAT ? dt : 0.0;
    s->prob.seed = seed;
    s->direct_halos = direct_halos;
    s->coarse_owner = coarse_partition(dim, n_coarse, n_ranks);
    const bool timing = std::getenv("PF_TIMING") != nullptr;
    auto tick = std::chrono::steady_clock::now();
    auto lap = [&](const char* what, int l) {
      if (!timing) return;
      const auto now = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[pf_timing] setup level %d %-14s %8.3f s\n", l, what,
                   std::chrono::duration<double>(now - tick).count());
      tick = now;
    };
    if (problem == PF_PROBLEM_LOGNORMAL) build_coefficients(*s);
    lap("coefficients", -1);
    for (int l = 0; l < n_levels; ++l) {
      build_level(*s, l);
      lap("level", l);
    }
    s->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = s.release();
  });
}

}  // namespace

extern "C" {

const char* pf_setup_last_error(void) { return g_setup_err.c_str(); }

pf_status pf_setup_create(int dim, int n_coarse, int n_levels, int n_ranks, int rank, int problem,
                          pf_setup** out) {
  if (problem == PF_PROBLEM_HEAT || problem == PF_PROBLEM_LOGNORMAL) {
    g_setup_err = problem == PF_PROBLEM_HEAT ? "the heat problem needs dt: use pf_setup_create_heat"
                                              : "the lognormal problem needs a seed: use pf_setup_create_lognormal";
    return PF_ERR_INVALID_ARGUMENT;
  }
  return create(dim, n_coarse, n_levels, n_ranks, rank, problem, 0.0, 0, out);
}

pf_status pf_setup_create_heat(int dim, int n_coarse, int n_levels, int n_ranks, int rank, double dt,
                               pf_setup** out) {
  return create(dim, n_coarse, n_levels, n_ranks, rank, PF_PROBLEM_HEAT, dt, 0, out);
}

pf_status pf_setup_create_opts(const pf_setup_options* o, pf_setup** out) {
  if (!o) {
    g_setup_err = "null options";
    return PF_ERR_INVALID_ARGUMENT;
  }
  return create(o->dim, o->n_coarse, o->n_levels, o->n_ranks, o->rank, o->problem, o->dt, o->seed, out,
                o->direct_halos != 0);
}

pf_status pf_setup_create_lognormal(int dim, int n_coarse, int n_levels, int n_ranks, int rank, uint64_t seed,
                                    pf_setup** out) {
  return create(dim, n_coarse, n_levels, n_ranks, rank, PF_PROBLEM_LOGNORMAL, 0.0, seed, out);
}

pf_status pf_setup_kappa(const pf_setup* s, const double** kappa, int64_t* n) {
  return guard([&] {
    if (!s) invalid("null setup");
    if (s->prob.kind != PF_PROBLEM_LOGNORMAL) invalid("kappa exists for the lognormal problem only");
    if (kappa) *kappa = s->kappa.data();
    if (n) *n = static_cast<int64_t>(s->kappa.size());
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
    if (s->matrices_released) state_error("level matrices released (pf_setup_release_matrices)");
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
    out->row_order = L.vert.data();  // lexicographic lattice index: coalesced gathers
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

pf_status pf_setup_rhs_operator(const pf_setup* s, const double** values, int64_t* nnz) {
  return guard([&] {
    if (!s) invalid("null setup");
    if (s->prob.kind != PF_PROBLEM_HEAT) invalid("rhs operator exists for the heat problem only");
    if (values) *values = s->rhs_op.data();
    if (nnz) *nnz = static_cast<int64_t>(s->rhs_op.size());
  });
}

pf_status pf_setup_load_at(const pf_setup* s, double t, double* out, int64_t n) {
  return guard([&] {
    if (!s || !out) invalid("null argument");
    if (n != s->levels.back()->n) invalid("load length does not match the finest level");
    finest_load(*s, t, out);
  });
}

pf_status pf_setup_load_desc(const pf_setup* s, pf_load_desc* out) {
  return guard([&] {
    if (!s || !out) invalid("null argument");
    const SetupLevel& L = *s->levels.back();
    std::memset(out, 0, sizeof *out);
    out->dim = s->d;
    out->n_cells = static_cast<int32_t>(L.geo.N);
    out->n_dofs = L.n;
    out->lattice = s->ld_lattice.data();
    out->cells = s->ld_cells.data();
    out->factor = s->ld_factor.data();
    out->extent = s->ld_extent.data();
    out->phi = s->ld_phi.data();
    out->qweight = s->d == 3 ? (0.5 * 0.5) * 0.5 : 0.5 * 0.5;
    out->boundary = s->ld_boundary.data();
    out->is_dirichlet = L.is_dir.data();
  });
}

pf_status pf_setup_assembly_desc(pf_setup* s, pf_assembly_desc* out) {
  return guard([&] {
    if (!s || !out) invalid("null argument");
    if (s->prob.kind == PF_PROBLEM_HEAT) invalid("device assembly covers the stiffness systems (not the CN system)");
    const SetupLevel& L = *s->levels.back();
    const int d = s->d;
    const int64_t N = L.geo.N;
    if (s->asm_elem.empty()) {
      for (const Element& E : L.elems)
        for (int i = 0; i < 8; ++i)
          for (int j = 0; j < 8; ++j) s->asm_elem.push_back(E.K[i][j]);
      s->asm_hid.assign(static_cast<size_t>(3 * N), 0);
      for (int a = 0; a < d; ++a)
        for (int64_t c = 0; c < N; ++c) s->asm_hid[static_cast<size_t>(a * N + c)] = L.hid[static_cast<size_t>(c)];
    }
    std::memset(out, 0, sizeof *out);
    out->dim = d;
    out->n_cells = static_cast<int32_t>(N);
    out->n_dofs = L.n;
    out->n_coarse = s->n_coarse;
    out->level = s->n_levels - 1;
    out->lattice = s->ld_lattice.data();
    out->cell_mask = L.cell_mask.data();
    out->is_dirichlet = L.is_dir.data();
    out->kappa = s->prob.kind == PF_PROBLEM_LOGNORMAL ? s->kappa.data() : nullptr;
    out->elem = s->asm_elem.data();
    out->elem_class = s->asm_hid.data();
    out->n_classes = L.nh;
  });
}

pf_status pf_setup_scales(const pf_setup* s, double t, double* source_scale, int32_t* has_dirichlet,
                          double* dirichlet_scale) {
  return guard([&] {
    if (!s) invalid("null setup");
    if (source_scale) *source_scale = s->prob.source_scale(t);
    if (has_dirichlet) *has_dirichlet = s->prob.has_dirichlet() ? 1 : 0;
    if (dirichlet_scale) *dirichlet_scale = s->prob.has_dirichlet() ? s->prob.dirichlet_scale(t) : 0.0;
  });
}

pf_status pf_setup_export_matrixmarket(const pf_setup* const* setups, int n_ranks, const char* matrix_path,
                                       const char* rhs_path, int64_t* n_global, int64_t* nnz) {
  return guard([&] {
    if (!setups || n_ranks < 1 || !matrix_path || !rhs_path) invalid("null argument");
    for (int r = 0; r < n_ranks; ++r) {
      if (!setups[r]) invalid("null setup");
      if (setups[r]->rank != r || setups[r]->n_ranks != n_ranks)
        invalid("setups[r] must be rank r of one n_ranks decomposition");
      if (setups[r]->d != setups[0]->d || setups[r]->n_coarse != setups[0]->n_coarse ||
          setups[r]->n_levels != setups[0]->n_levels || setups[r]->prob.kind != setups[0]->prob.kind)
        invalid("setups of different problems");
    }
    // assign_global_numbers (femapper.cpp:353-472): own dofs rank by rank in local order,
    // then the Dirichlet dofs each rank is the authority of (owns_row), rank by rank; every
    // other local dof takes its carrier's number from the rank that numbered it.
    const Geo& g0 = setups[0]->levels.back()->geo;
    const int64_t nv = (g0.N + 1) * (g0.N + 1) * g0.nzv();
    std::vector<int64_t> gid_of_key(static_cast<size_t>(nv), -1);
    int64_t next = 0;
    for (int r = 0; r < n_ranks; ++r) {
      const SetupLevel& L = *setups[r]->levels.back();
      for (int32_t i = 0; i < L.n_own; ++i) gid_of_key[static_cast<size_t>(L.vert[i])] = next++;
    }
    const int64_t total_own = next;
    for (int r = 0; r < n_ranks; ++r) {
      const SetupLevel& L = *setups[r]->levels.back();
      for (int32_t i = 0; i < L.n; ++i)
        if (L.owns_row[i] && L.class_of[i] == kDirichlet) gid_of_key[static_cast<size_t>(L.vert[i])] = next++;
    }
    const int64_t n = next;
    (void)total_own;
    // export_matrixmarket (matrix_market.cpp:47-112): "%lld %lld %.17g" per entry of every
    // owned row, rank by rank in local order; the rhs as an array, own rows of all ranks
    // first, then the owned Dirichlet rows.
    int64_t total_nnz = 0;
    for (int r = 0; r < n_ranks; ++r) {
      const SetupLevel& L = *setups[r]->levels.back();
      for (int32_t i = 0; i < L.n; ++i)
        if (L.owns_row[i]) total_nnz += L.rowptr[i + 1] - L.rowptr[i];
    }
    std::FILE* fm = std::fopen(matrix_path, "wb");
    if (!fm) throw SetupError(PF_ERR_STATE, std::string("cannot open '") + matrix_path + "' for writing");
    std::fprintf(fm, "%%%%MatrixMarket matrix coordinate real general\n%lld %lld %lld\n", static_cast<long long>(n),
                 static_cast<long long>(n), static_cast<long long>(total_nnz));
    for (int r = 0; r < n_ranks; ++r) {
      const SetupLevel& L = *setups[r]->levels.back();
      // rows formatted in parallel blocks, written in order
      constexpr int32_t kRows = 1 << 14;
      for (int32_t r0 = 0; r0 < L.n; r0 += kRows * 16) {
        const int32_t r1 = std::min<int32_t>(L.n, r0 + kRows * 16);
        const int nb = (r1 - r0 + kRows - 1) / kRows;
        std::vector<std::string> out(static_cast<size_t>(nb));
#pragma omp parallel for schedule(dynamic)
        for (int b = 0; b < nb; ++b) {
          std::string& o = out[static_cast<size_t>(b)];
          char buf[128];
          for (int32_t i = r0 + b * kRows; i < std::min<int32_t>(r1, r0 + (b + 1) * kRows); ++i) {
            if (!L.owns_row[i]) continue;
            const long long grow = gid_of_key[static_cast<size_t>(L.vert[i])] + 1;
            for (int64_t k = L.rowptr[i]; k < L.rowptr[i + 1]; ++k) {
              const long long gcol = gid_of_key[static_cast<size_t>(L.vert[static_cast<size_t>(L.cols[k])])] + 1;
              const int len = std::snprintf(buf, sizeof buf, "%lld %lld %.17g\n", grow, gcol, L.vals[static_cast<size_t>(k)]);
              o.append(buf, static_cast<size_t>(len));
            }
          }
        }
        for (const std::string& o : out) std::fwrite(o.data(), 1, o.size(), fm);
      }
    }
    const bool ok_m = std::fflush(fm) == 0 && !std::ferror(fm);
    std::fclose(fm);
    if (!ok_m) throw SetupError(PF_ERR_STATE, std::string("write failed for '") + matrix_path + "'");
    std::FILE* fr = std::fopen(rhs_path, "wb");
    if (!fr) throw SetupError(PF_ERR_STATE, std::string("cannot open '") + rhs_path + "' for writing");
    std::fprintf(fr, "%%%%MatrixMarket matrix array real general\n%lld 1\n", static_cast<long long>(n));
    for (int pass = 0; pass < 2; ++pass)
      for (int r = 0; r < n_ranks; ++r) {
        const SetupLevel& L = *setups[r]->levels.back();
        const std::vector<double>& b = setups[r]->b;
        for (int32_t i = pass == 0 ? 0 : L.n_own; i < (pass == 0 ? L.n_own : L.n); ++i) {
          if (pass == 1 && !L.owns_row[i]) continue;
          std::fprintf(fr, "%.17g\n", b[static_cast<size_t>(i)]);
        }
      }
    const bool ok_r = std::fflush(fr) == 0 && !std::ferror(fr);
    std::fclose(fr);
    if (!ok_r) throw SetupError(PF_ERR_STATE, std::string("write failed for '") + rhs_path + "'");
    if (n_global) *n_global = n;
    if (nnz) *nnz = total_nnz;
  });
}

pf_status pf_setup_release_matrices(pf_setup* s) {
  return guard([&] {
    if (!s) invalid("null setup");
    for (auto& L : s->levels) {
      std::vector<int64_t>().swap(L->rowptr);
      std::vector<int32_t>().swap(L->cols);
      std::vector<double>().swap(L->vals);
      std::vector<int64_t>().swap(L->p_off);
      std::vector<int32_t>().swap(L->p_col);
      std::vector<double>().swap(L->p_w);
    }
    std::vector<double>().swap(s->rhs_op);
    s->matrices_released = true;
  });
}

}  // extern "C"

namespace pf {

// Hand one level of a setup to a hierarchy by moving its arrays (no second host copy of
// the matrices; pf_hierarchy_set_level_from_setup).  The setup's matrices of that level
// are gone afterwards.
void adopt_setup_level(pf_setup* s, int level, HostLevel& H) {
  if (!s) throw Error(PF_ERR_INVALID_ARGUMENT, "null setup");
  if (level < 0 || level >= s->n_levels) throw Error(PF_ERR_INVALID_ARGUMENT, "level out of range");
  SetupLevel& L = *s->levels[static_cast<size_t>(level)];
  if (L.rowptr.empty()) throw Error(PF_ERR_STATE, "level matrices already released or adopted");
  H = HostLevel{};
  H.set = true;
  H.n = L.n;
  H.n_own = L.n_own;
  H.rowptr = std::move(L.rowptr);
  H.cols = std::move(L.cols);
  H.vals = std::move(L.vals);
  H.owns_row = L.owns_row;
  H.is_dir = L.is_dir;
  H.color = L.color;
  H.order = L.vert;  // lexicographic lattice index: the device placement hint
  for (const OwnedChannel& c : L.channels) {
    HostChannel hc;
    hc.kind = c.kind;
    hc.peer = c.peer;
    hc.send = c.send;
    hc.recv = c.recv;
    H.channels.push_back(std::move(hc));
  }
  std::sort(H.channels.begin(), H.channels.end(), [](const HostChannel& a, const HostChannel& b) {
    return a.kind != b.kind ? a.kind < b.kind : a.peer < b.peer;
  });
  if (level > 0) {
    H.p_off = std::move(L.p_off);
    H.p_col = std::move(L.p_col);
    H.p_w = std::move(L.p_w);
  }
  s->matrices_released = true;  // pf_setup_level no longer describes this setup
}

}  // namespace pf

extern "C" {

pf_status pf_setup_seconds(const pf_setup* s, double* out) {
  return guard([&] {
    if (!s || !out) invalid("null argument");
    *out = s->seconds;
  });
}

}  // extern "C"

// Coordinate bisection of the coarse cells, for the element families (pf_fe_setup.cpp).
std::vector<int> pf_coarse_partition(int d, int n, int k) { return coarse_partition(d, n, k); }
