// parfem_gpu_bridge.cpp — see parfem_gpu_bridge.hpp.
#include "parfem_gpu_bridge.hpp"

#include <csignal>
#include <cstdio>
#include <execinfo.h>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

#include "parfem/errors.hpp"
#include "parfem_b200.hpp"

namespace parfem::gpu {

namespace {

void on_segv(int) {
  void* frames[64];
  const int n = backtrace(frames, 64);
  backtrace_symbols_fd(frames, n, 2);
  std::_Exit(139);
}

void trace(const char* what) {
  static const bool on = [] {
    const bool t = std::getenv("PF_BRIDGE_TRACE") != nullptr;
    if (t) std::signal(SIGSEGV, on_segv);
    return t;
  }();
  if (on) std::fprintf(stderr, "[parfem::gpu] %s\n", what);
}

// Plain storage behind one pf_level_desc.
struct LevelStore {
  int32_t n = 0, n_own = 0;
  std::vector<int64_t> rowptr;
  std::vector<int32_t> cols;
  std::vector<double> vals;
  std::vector<uint8_t> owns, isdir;
  struct Ch {
    int32_t kind, peer;
    std::vector<int32_t> send, recv;
  };
  std::vector<Ch> chans;
  std::vector<pf_channel_desc> descs;
  std::vector<int64_t> poff;
  std::vector<int32_t> pcol;
  std::vector<double> pw;

  pf_level_desc desc() {
    descs.clear();
    for (Ch& c : chans)
      descs.push_back({c.kind, c.peer, static_cast<int32_t>(c.send.size()), static_cast<int32_t>(c.recv.size()),
                       c.send.data(), c.recv.data()});
    pf_level_desc d{};
    d.n_dofs = n;
    d.n_own_dofs = n_own;
    d.row_offsets = rowptr.data();
    d.col_indices = cols.data();
    d.values = vals.data();
    d.owns_row = owns.data();
    d.is_dirichlet = isdir.data();
    d.color = nullptr;  // greedy colouring of the reference's own row graph
    d.n_channels = static_cast<int32_t>(descs.size());
    d.channels = descs.data();
    if (!poff.empty()) {
      d.p_offsets = poff.data();
      d.p_cols = pcol.data();
      d.p_weights = pw.data();
    }
    return d;
  }
};

// MultigridLevel (multigrid.hpp:15-31) -> plain arrays in the reference's host order.
LevelStore from_level(const MultigridLevel& L) {
  const ParFEMapper& m = *L.mapper;
  LevelStore s;
  s.n = m.n_dofs;
  s.n_own = m.n_own_dofs;
  s.rowptr.assign(L.system.row_offsets.begin(), L.system.row_offsets.end());
  s.cols = L.system.col_indices;
  s.vals = L.system.values;
  s.owns.assign(m.owns_row.begin(), m.owns_row.end());
  for (DofClass c : m.class_of) s.isdir.push_back(c == DofClass::Dirichlet ? 1 : 0);
  for (int k = 0; k < kNumChannelKinds; ++k)
    for (const auto& [peer, ch] : m.channels[static_cast<size_t>(k)])
      s.chans.push_back({k, peer, ch.send_dofs, ch.recv_dofs});
  if (!L.prolong_map.empty()) {
    s.poff.push_back(0);
    for (const auto& row : L.prolong_map) {
      for (const auto& [cd, w] : row) {
        s.pcol.push_back(cd);
        s.pw.push_back(w);
      }
      s.poff.push_back(static_cast<int64_t>(s.pcol.size()));
    }
  }
  return s;
}

template <typename T>
void put_vec(ByteWriter& w, const std::vector<T>& v) {
  w.put_i64(static_cast<std::int64_t>(v.size()));
  for (const T& x : v) {
    if constexpr (std::is_floating_point_v<T>) w.put_f64(x);
    else w.put_i64(static_cast<std::int64_t>(x));
  }
}

template <typename T>
std::vector<T> get_vec(ByteReader& r) {
  std::vector<T> v(static_cast<size_t>(r.get_i64()));
  for (T& x : v) {
    if constexpr (std::is_floating_point_v<T>) x = r.get_f64();
    else x = static_cast<T>(r.get_i64());
  }
  return v;
}

Bytes serialize(const LevelStore& s) {
  ByteWriter w;
  w.put_i64(s.n);
  w.put_i64(s.n_own);
  put_vec(w, s.rowptr);
  put_vec(w, s.cols);
  put_vec(w, s.vals);
  put_vec(w, s.owns);
  put_vec(w, s.isdir);
  w.put_i64(static_cast<std::int64_t>(s.chans.size()));
  for (const auto& c : s.chans) {
    w.put_i64(c.kind);
    w.put_i64(c.peer);
    put_vec(w, c.send);
    put_vec(w, c.recv);
  }
  return w.take();
}

LevelStore deserialize(Bytes b) {
  ByteReader r(std::move(b));
  LevelStore s;
  s.n = static_cast<int32_t>(r.get_i64());
  s.n_own = static_cast<int32_t>(r.get_i64());
  s.rowptr = get_vec<int64_t>(r);
  s.cols = get_vec<int32_t>(r);
  s.vals = get_vec<double>(r);
  s.owns = get_vec<uint8_t>(r);
  s.isdir = get_vec<uint8_t>(r);
  const std::int64_t nc = r.get_i64();
  for (std::int64_t i = 0; i < nc; ++i) {
    LevelStore::Ch c;
    c.kind = static_cast<int32_t>(r.get_i64());
    c.peer = static_cast<int32_t>(r.get_i64());
    c.send = get_vec<int32_t>(r);
    c.recv = get_vec<int32_t>(r);
    s.chans.push_back(std::move(c));
  }
  return s;
}

struct Mirror {
  std::unique_ptr<parfem_b200::Hierarchy> dev;
  std::unique_ptr<parfem_b200::DeviceVector> x, b;
  void* hub = nullptr;
  bool owns_hub = false;
  std::uint64_t fp = 0;  // fingerprint of the hierarchy the mirror was built from
};

std::mutex g_mu;
std::map<const MultigridHierarchy*, std::unique_ptr<Mirror>> g_mirrors;

// Sampled FNV-1a fingerprint of a hierarchy's level data (sizes, row offsets, columns,
// values, prolongation rows): a hierarchy rebuilt at the same address with other data
// must not reuse the old device mirror.
std::uint64_t fingerprint(const MultigridHierarchy& h) {
  std::uint64_t f = 1469598103934665603ull;
  auto mix = [&f](const void* p, size_t n) {
    const unsigned char* c = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) f = (f ^ c[i]) * 1099511628211ull;
  };
  auto sample = [&mix](const auto& v) {
    const size_t n = v.size();
    mix(&n, sizeof n);
    const size_t step = n > 1024 ? n / 1024 : 1;
    for (size_t i = 0; i < n; i += step) mix(&v[i], sizeof v[i]);
    if (n) mix(&v[n - 1], sizeof v[n - 1]);
  };
  const int K = h.tp->size();
  mix(&K, sizeof K);
  for (const MultigridLevel& L : h.levels) {
    mix(&L.mapper->n_dofs, sizeof L.mapper->n_dofs);
    mix(&L.mapper->n_own_dofs, sizeof L.mapper->n_own_dofs);
    sample(L.system.row_offsets);
    sample(L.system.col_indices);
    sample(L.system.values);
    const size_t np = L.prolong_map.size();
    mix(&np, sizeof np);
    const size_t step = np > 256 ? np / 256 : 1;
    for (size_t i = 0; i < np; i += step)
      for (const auto& [cd, w] : L.prolong_map[i]) {
        mix(&cd, sizeof cd);
        mix(&w, sizeof w);
      }
  }
  return f;
}

Mirror& mirror(MultigridHierarchy& h) {
  const std::uint64_t fp = fingerprint(h);
  bool found = false, stale = false;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    auto it = g_mirrors.find(&h);
    if (it != g_mirrors.end()) {
      found = true;
      stale = it->second->fp != fp;
    }
  }
  if (found && h.tp->size() > 1) {  // rebuilding is collective: any stale rank decides for all
    ByteWriter w;
    w.put_i64(stale ? 1 : 0);
    for (Bytes& b : allgather(*h.tp, w.take()))
      if (ByteReader(std::move(b)).get_i64()) stale = true;
  }
  if (found && !stale) {
    std::lock_guard<std::mutex> lock(g_mu);
    return *g_mirrors.find(&h)->second;
  }
  if (found) release(h);
  Transport& tp = *h.tp;
  const int K = tp.size(), rank = tp.rank(), L = static_cast<int>(h.levels.size());
  int n_dev = 0;
  if (pf_device_count(&n_dev) != PF_OK || n_dev < 1) throw Error("parfem::gpu: no CUDA device");
  auto m = std::make_unique<Mirror>();
  trace("create");
  m->dev = std::make_unique<parfem_b200::Hierarchy>(rank % n_dev, L, 1, rank, K);
  trace("created");
  std::vector<LevelStore> stores;
  for (const MultigridLevel& lv : h.levels) stores.push_back(from_level(lv));
  for (int l = 0; l < L; ++l) m->dev->set_level(l, 0, stores[static_cast<size_t>(l)].desc());
  trace("levels set");
  if (K > 1) {
    // every rank's coarse level, over the reference's own transport (setup only)
    std::vector<Bytes> all = allgather(tp, serialize(stores[0]));
    for (int q = 0; q < K; ++q) {
      LevelStore s = deserialize(std::move(all[static_cast<size_t>(q)]));
      m->dev->set_coarse_replica(q, s.desc());
    }
  }
  m->dev->finalize();
  trace("finalized");
  if (K > 1) {
    ByteWriter w;
    if (rank == 0) {
      parfem_b200::check(pf_loopback_create(K, &m->hub));
      m->owns_hub = true;
      w.put_i64(static_cast<std::int64_t>(reinterpret_cast<std::intptr_t>(m->hub)));
    }
    ByteReader r(broadcast(tp, 0, w.take()));
    m->hub = reinterpret_cast<void*>(static_cast<std::intptr_t>(r.get_i64()));
    m->dev->init_loopback(m->hub);
  }
  m->x = std::make_unique<parfem_b200::DeviceVector>(*m->dev, L - 1);
  m->b = std::make_unique<parfem_b200::DeviceVector>(*m->dev, L - 1);
  m->fp = fp;
  std::lock_guard<std::mutex> lock(g_mu);
  return *(g_mirrors[&h] = std::move(m));
}

}  // namespace

SolveStats solve_outer(MultigridHierarchy& h, DistributedVector& x, const DistributedVector& b,
                       const MultigridConfig& cfg) {
  if (h.levels.empty()) throw Error("empty hierarchy");
  if (x.size() != static_cast<size_t>(h.finest().mapper->n_dofs) || b.size() != x.size())
    throw std::invalid_argument("solve_outer: vector sizes do not match the mapper");
  Mirror& m = mirror(h);
  parfem_b200::MultigridConfig c;
  c.cycles = cfg.cycles;
  c.smoother.kind = cfg.smoother.kind == SmootherKind::Jacobi ? parfem_b200::SmootherKind::Jacobi
                                                              : parfem_b200::SmootherKind::GaussSeidel;
  c.smoother.sweeps = cfg.smoother.sweeps;
  c.smoother.local_sweeps = cfg.smoother.local_sweeps;
  c.smoother.damping = cfg.smoother.damping;
  c.pre_smooth = cfg.pre_smooth;
  c.post_smooth = cfg.post_smooth;
  c.coarse_tol = cfg.coarse_tol;
  c.coarse_max_iter = cfg.coarse_max_iter;
  c.outer_tol = cfg.outer_tol;
  c.outer_max_cycles = cfg.outer_max_cycles;
  trace("upload");
  m.x->upload(x.values);
  m.b->upload(b.values);
  trace("solve");
  SolveStats out;
  try {
    const parfem_b200::SolveStats s = parfem_b200::solve_outer(*m.dev, *m.x, *m.b, c);
    out.iterations = s.iterations;
    out.initial_residual = s.initial_residual;
    out.final_residual = s.final_residual;
    out.converged = s.converged;
    out.residuals = s.residuals;
    out.solve_seconds = s.solve_seconds;
    out.comm_seconds = s.comm_seconds;
  } catch (const parfem_b200::NoConvergenceError& e) {
    m.x->download(x.values);
    throw NoConvergenceError(e.what());
  } catch (const parfem_b200::TransportError& e) {
    throw TransportError(e.what());
  } catch (const parfem_b200::SingularDiagonalError& e) {
    throw SingularDiagonalError(e.what());
  }
  trace("download");
  m.x->download(x.values);
  x.state = ConsistencyState::Consistent;
  trace("done");
  return out;
}

void release(const MultigridHierarchy& h) {
  std::unique_ptr<Mirror> m;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    auto it = g_mirrors.find(&h);
    if (it == g_mirrors.end()) return;
    m = std::move(it->second);
    g_mirrors.erase(it);
  }
  barrier(*h.tp);  // nobody may still be using the shared hub
  void* hub = m->owns_hub ? m->hub : nullptr;
  m.reset();
  barrier(*h.tp);
  if (hub) pf_loopback_destroy(hub);
}

}  // namespace parfem::gpu
