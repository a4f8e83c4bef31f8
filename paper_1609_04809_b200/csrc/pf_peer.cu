// pf_peer.cu — peer-memory transport: IPC arena export/import and the exchange launches.
//
// Replaces the reference's Transport mailboxes (transport.cpp:33-104) under
// ParFECommunicator::scatter / update_master_slave (fecomm.cpp:25-62) and the allgather of
// allreduce_sum (transport.cpp:139-165) with stores into mapped peer memory
// (pf_peer.cuh).  See pf_peer.hpp for the setup sequence.
#include <unistd.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "pf_peer.hpp"

namespace pf {

// pf_runtime.cu
int64_t* launch_counter(pf_hierarchy* h);
bool pdl_on(const pf_hierarchy* h);

namespace {

// Stream-ordered upload: ranks that share a device (hierarchies of one process) may already
// be spinning in exchange kernels, which a legacy-stream copy or a device-wide
// synchronisation would wait for.
template <typename T>
void upload_on(DevBuf<T>& d, const std::vector<T>& v, cudaStream_t s) {
  d.alloc(static_cast<int64_t>(v.size()));
  if (!v.empty()) cuda_check(cudaMemcpyAsync(d.p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, s), "peer upload");
  cuda_check(cudaStreamSynchronize(s), "peer upload");
}

constexpr uint64_t kMagic = 0x31524545504650ull;  // "PFPEER1"
constexpr int64_t kAlign = 256;

int64_t align_up(int64_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

struct BlobHead {
  uint64_t magic;
  int32_t version, rank, world, device;
  int64_t pid;
  uint64_t arena_ptr;
  int64_t arena_bytes;
  cudaIpcMemHandle_t handle;
  int32_t ipc_ok, n_plans, n_sites, fused;
};
struct BlobSeg {
  int32_t peer, pad;
  int64_t stage_off, len;
};
struct BlobSite {
  int64_t stage_off, count;
};

// The hierarchy's remote exchange plans in a canonical order every rank shares.
std::vector<ExchangePlan*> remote_plans(pf_hierarchy* h, std::vector<bool>* is_acc = nullptr) {
  std::vector<ExchangePlan*> v;
  for (Level& L : h->levels) {
    for (ExchangePlan& P : L.scatter) v.push_back(&P);
    v.push_back(&L.accumulate);
    if (h->fused) {
      v.push_back(&L.fused_ms_h1);
      v.push_back(&L.fused_all);
    }
  }
  if (is_acc) {
    is_acc->assign(v.size(), false);
    for (size_t i = 0; i < v.size(); ++i)
      for (Level& L : h->levels)
        if (v[i] == &L.accumulate) (*is_acc)[i] = true;
  }
  return v;
}

struct SiteSpec {
  const double* send;
  double* recv;
  int64_t count;
};

// Every allgather the V-cycle issues (enq_allreduce, the replicated coarse solve and the
// replicated bottom), same order on every rank.
std::vector<SiteSpec> site_specs(pf_hierarchy* h) {
  std::vector<SiteSpec> v;
  for (Level& L : h->levels) v.push_back({L.sumsq.p, L.sumsq.p + 1, 1});
  if (h->rep.active) {
    for (auto& RL : h->rep.lv) v.push_back({h->rep.send.p, RL.b.p, RL.stride});
    v.push_back({h->rep.send.p, h->rep.lv[0].x.p, h->rep.lv[0].stride});
  }
  return v;
}

int64_t recv_total(const ExchangePlan& P) {
  int64_t n = 0;
  for (const auto& s : P.recv_segs) n = std::max(n, s.off + s.len);
  return n;
}

double watchdog_default() {
  const char* e = std::getenv("PF_WATCHDOG_S");
  return e ? std::atof(e) : 120.0;
}

}  // namespace

PeerArgs PeerTransport::args(const Op& o, bool wait_only) const {
  PeerArgs a{};
  a.sends = o.sends.p;
  a.recvs = o.recvs.p;
  a.segs = o.segs.p;
  a.n_sends = o.n_sends;
  a.n_recvs = o.n_recvs;
  a.me = rank;
  a.wait_only = wait_only ? 1 : 0;
  a.mine = ctl();
  a.remote = remote_ctl.p;
  a.timeout_ns = timeout_ns;
  return a;
}

void PeerTransport::launch_exchange(const Op& o, double* v, bool wait_only, cudaStream_t s) {
  if (!ready) throw Error(PF_ERR_STATE, "peer transport used before pf_hierarchy_init_peer");
  const int grid = o.n_sends + o.n_recvs;
  if (grid == 0) return;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(static_cast<unsigned>(grid));
  lc.blockDim = dim3(kPeerBlock);
  lc.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = pdl_on(h) ? 1 : 0;
  cuda_check(cudaLaunchKernelEx(&lc, k_peer_exchange, args(o, wait_only), v), "k_peer_exchange");
  ++*launch_counter(h);
}

void PeerTransport::run_plan(const ExchangePlan& P, double* v, bool wait_only, cudaStream_t s) {
  if (P.peer_id < 0 || P.peer_id >= static_cast<int>(plans.size()))
    throw Error(PF_ERR_STATE, "exchange plan unknown to the peer transport");
  launch_exchange(plans[static_cast<size_t>(P.peer_id)], v, wait_only, s);
}

const double* PeerTransport::staging(const ExchangePlan& P) const {
  const Op& o = plans.at(static_cast<size_t>(P.peer_id));
  return reinterpret_cast<const double*>(arena.p + o.stage_off);
}

void PeerTransport::ack_plan(const ExchangePlan& P, cudaStream_t s) {
  const Op& o = plans.at(static_cast<size_t>(P.peer_id));
  if (o.n_recvs == 0) return;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(static_cast<unsigned>((o.n_recvs + 31) / 32));
  lc.blockDim = dim3(32);
  lc.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = pdl_on(h) ? 1 : 0;
  cuda_check(cudaLaunchKernelEx(&lc, k_peer_ack, args(o, true)), "k_peer_ack");
  ++*launch_counter(h);
}

void PeerTransport::allgather(const double* send, double* recv, int64_t count, cudaStream_t s) {
  auto it = site_of.find(recv);
  if (it == site_of.end()) throw Error(PF_ERR_STATE, "allgather target not registered with the peer transport");
  const Op& o = sites[static_cast<size_t>(it->second)];
  if (o.send != send || o.count != count) throw Error(PF_ERR_STATE, "allgather differs from its registration");
  launch_exchange(o, nullptr, false, s);
}

void PeerTransport::group_start() { throw Error(PF_ERR_STATE, "the peer transport executes whole plans"); }
void PeerTransport::group_end(cudaStream_t) { throw Error(PF_ERR_STATE, "the peer transport executes whole plans"); }
void PeerTransport::send(const double*, int64_t, int, cudaStream_t) {
  throw Error(PF_ERR_STATE, "the peer transport executes whole plans");
}
void PeerTransport::recv(double*, int64_t, int, cudaStream_t) {
  throw Error(PF_ERR_STATE, "the peer transport executes whole plans");
}

// Called after the stream drained: a wait that hit the device watchdog left its mark.
void PeerTransport::check_async() {
  if (!ready) return;
  PeerCtl c;
  cuda_check(cudaMemcpyAsync(&c.error, &ctl()->error, sizeof(unsigned int) + sizeof(int), cudaMemcpyDeviceToHost,
                             h->stream),
             "peer error word");
  cuda_check(cudaStreamSynchronize(h->stream), "peer error word");
  if (c.error)
    throw Error(PF_ERR_TRANSPORT, "peer watchdog: rank " + std::to_string(c.error_peer) +
                                      " did not deliver (or acknowledge) an exchange within " +
                                      std::to_string(timeout_ns / 1e9) + " s");
}

PeerTransport::~PeerTransport() {
  for (void* p : opened) cudaIpcCloseMemHandle(p);
}

int64_t peer_export(pf_hierarchy* h, void* buf, int64_t cap) {
  auto* t = dynamic_cast<PeerTransport*>(h->xport.get());
  if (!t) {
    if (h->xport) throw Error(PF_ERR_STATE, "transport already initialized");
    if (h->world > kPeerMaxWorld) throw Error(PF_ERR_INVALID_ARGUMENT, "peer transport supports up to 64 ranks");
    auto nt = std::make_unique<PeerTransport>();
    nt->h = h;
    nt->rank = h->rank_base;
    nt->world = h->world;
    nt->timeout_ns = static_cast<unsigned long long>(watchdog_default() * 1e9);
    std::vector<bool> is_acc;
    auto ps = remote_plans(h, &is_acc);
    auto ss = site_specs(h);
    int64_t off = align_up(static_cast<int64_t>(sizeof(PeerCtl)));
    nt->plans.resize(ps.size());
    for (size_t i = 0; i < ps.size(); ++i) {
      ps[i]->peer_id = static_cast<int>(i);
      nt->plans[i].stage_off = off;
      off += align_up(8 * recv_total(*ps[i]));
    }
    nt->sites.resize(ss.size());
    for (size_t i = 0; i < ss.size(); ++i) {
      PeerTransport::Op& o = nt->sites[i];
      o.send = ss[i].send;
      o.recv = ss[i].recv;
      o.count = ss[i].count;
      o.stage_off = off;
      off += align_up(8 * ss[i].count * h->world);
      if (nt->site_of.count(o.recv)) throw Error(PF_ERR_STATE, "allgather target registered twice");
      nt->site_of[o.recv] = static_cast<int>(i);
    }
    nt->arena_bytes = off;
    nt->arena.alloc(off);
    cuda_check(cudaMemsetAsync(nt->arena.p, 0, static_cast<size_t>(off), h->stream), "peer arena");
    cuda_check(cudaStreamSynchronize(h->stream), "peer arena");
    t = nt.get();
    h->xport = std::move(nt);
  }
  // the blob
  std::vector<char> blob(sizeof(BlobHead));
  BlobHead head{};
  head.magic = kMagic;
  head.version = 1;
  head.rank = t->rank;
  head.world = t->world;
  head.device = h->device;
  head.pid = static_cast<int64_t>(getpid());
  head.arena_ptr = reinterpret_cast<uint64_t>(t->arena.p);
  head.arena_bytes = t->arena_bytes;
  head.ipc_ok = cudaIpcGetMemHandle(&head.handle, t->arena.p) == cudaSuccess ? 1 : 0;
  (void)cudaGetLastError();
  auto ps = remote_plans(h);
  head.n_plans = static_cast<int32_t>(ps.size());
  head.n_sites = static_cast<int32_t>(t->sites.size());
  head.fused = h->fused ? 1 : 0;
  std::memcpy(blob.data(), &head, sizeof head);
  auto put = [&](const void* p, size_t n) {
    const char* c = static_cast<const char*>(p);
    blob.insert(blob.end(), c, c + n);
  };
  for (size_t i = 0; i < ps.size(); ++i) {
    const int32_t n = static_cast<int32_t>(ps[i]->recv_segs.size());
    const int32_t pad = 0;
    put(&n, 4);
    put(&pad, 4);
    for (const auto& s : ps[i]->recv_segs) {
      BlobSeg b{s.peer, 0, t->plans[i].stage_off + 8 * s.off, s.len};
      put(&b, sizeof b);
    }
  }
  for (const auto& o : t->sites) {
    BlobSite b{o.stage_off, o.count};
    put(&b, sizeof b);
  }
  const int64_t n = static_cast<int64_t>(blob.size());
  if (buf && cap >= n) std::memcpy(buf, blob.data(), blob.size());
  return n;
}

void peer_import(pf_hierarchy* h, const void* blobs, int64_t stride) {
  auto* t = dynamic_cast<PeerTransport*>(h->xport.get());
  if (!t) throw Error(PF_ERR_STATE, "pf_hierarchy_peer_export must run before pf_hierarchy_init_peer");
  if (t->ready) throw Error(PF_ERR_STATE, "peer transport already initialized");
  const int W = t->world, me = t->rank;
  auto ps = remote_plans(h);
  std::vector<bool> is_acc;
  remote_plans(h, &is_acc);
  struct Parsed {
    BlobHead head;
    std::vector<std::vector<BlobSeg>> recv;  // per plan
    std::vector<BlobSite> sites;
  };
  std::vector<Parsed> P(static_cast<size_t>(W));
  for (int r = 0; r < W; ++r) {
    const char* b = static_cast<const char*>(blobs) + static_cast<int64_t>(r) * stride;
    const char* end = b + stride;
    Parsed& q = P[static_cast<size_t>(r)];
    std::memcpy(&q.head, b, sizeof(BlobHead));
    if (q.head.magic != kMagic || q.head.version != 1)
      throw Error(PF_ERR_INVALID_ARGUMENT, "peer blob " + std::to_string(r) + " is not a pf peer export");
    if (q.head.rank != r || q.head.world != W)
      throw Error(PF_ERR_INVALID_ARGUMENT, "peer blob " + std::to_string(r) + " belongs to rank " +
                                               std::to_string(q.head.rank) + " of " + std::to_string(q.head.world));
    if (q.head.n_plans != static_cast<int32_t>(ps.size()) || q.head.n_sites != static_cast<int32_t>(t->sites.size()) ||
        q.head.fused != (h->fused ? 1 : 0))
      throw Error(PF_ERR_INVALID_ARGUMENT, "rank " + std::to_string(r) + " has a different hierarchy shape");
    const char* c = b + sizeof(BlobHead);
    auto take = [&](void* dst, size_t n) {
      if (c + n > end) throw Error(PF_ERR_INVALID_ARGUMENT, "peer blob truncated");
      std::memcpy(dst, c, n);
      c += n;
    };
    q.recv.resize(ps.size());
    for (size_t i = 0; i < ps.size(); ++i) {
      int32_t n = 0, pad = 0;
      take(&n, 4);
      take(&pad, 4);
      q.recv[i].resize(static_cast<size_t>(n));
      for (auto& s : q.recv[i]) take(&s, sizeof s);
    }
    q.sites.resize(t->sites.size());
    for (auto& s : q.sites) take(&s, sizeof s);
  }
  // map every peer's arena
  std::vector<char*> base(static_cast<size_t>(W), nullptr);
  const int64_t pid = static_cast<int64_t>(getpid());
  int same_process = 0;
  for (int r = 0; r < W; ++r) same_process += P[static_cast<size_t>(r)].head.pid == pid;
  t->in_process = same_process > 1;
  if (same_process > 1) {
    // Ranks of one process share its context: a kernel waiting for a peer's kernel must
    // not sit ahead of that kernel in a hardware work queue (streams beyond
    // CUDA_DEVICE_MAX_CONNECTIONS share queues) or race a lazy module load of it.
    const char* ml = std::getenv("CUDA_MODULE_LOADING");
    const char* mc = std::getenv("CUDA_DEVICE_MAX_CONNECTIONS");
    if (!ml || std::string(ml) != "EAGER" || !mc || std::atoi(mc) < 2 * same_process)
      throw Error(PF_ERR_STATE, "in-process peer ranks need CUDA_MODULE_LOADING=EAGER and CUDA_DEVICE_MAX_CONNECTIONS >= " +
                                    std::to_string(2 * same_process) +
                                    " set before CUDA initialises (or one process per rank)");
  }
  for (int r = 0; r < W; ++r) {
    const BlobHead& hd = P[static_cast<size_t>(r)].head;
    if (r == me) {
      base[static_cast<size_t>(r)] = t->arena.p;
    } else if (hd.pid == pid) {  // another hierarchy of this process
      if (hd.device != h->device) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(hd.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cuda_check(e, "cudaDeviceEnablePeerAccess");
        (void)cudaGetLastError();
      }
      base[static_cast<size_t>(r)] = reinterpret_cast<char*>(hd.arena_ptr);
    } else {
      if (!hd.ipc_ok) throw Error(PF_ERR_TRANSPORT, "rank " + std::to_string(r) + " could not export its arena");
      void* p = nullptr;
      cuda_check(cudaIpcOpenMemHandle(&p, hd.handle, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      t->opened.push_back(p);
      base[static_cast<size_t>(r)] = static_cast<char*>(p);
    }
  }
  std::vector<PeerCtl*> rc(static_cast<size_t>(W));
  for (int r = 0; r < W; ++r) rc[static_cast<size_t>(r)] = reinterpret_cast<PeerCtl*>(base[static_cast<size_t>(r)]);
  upload_on(t->remote_ctl, rc, h->stream);
  // plans: my sends pair with the peer's receives from me (k-th with k-th, NCCL order)
  for (size_t i = 0; i < ps.size(); ++i) {
    const ExchangePlan& X = *ps[i];
    PeerTransport::Op& o = t->plans[i];
    std::vector<PeerGroup> sg, rg;
    std::vector<PeerPiece> pieces;
    std::vector<int> peers;
    for (const auto& s : X.send_segs) peers.push_back(s.peer);
    std::sort(peers.begin(), peers.end());
    peers.erase(std::unique(peers.begin(), peers.end()), peers.end());
    for (int p : peers) {
      const auto& theirs = P[static_cast<size_t>(p)].recv[i];
      std::vector<const BlobSeg*> from_me;
      for (const auto& b : theirs)
        if (b.peer == me) from_me.push_back(&b);
      PeerGroup g{p, static_cast<int32_t>(pieces.size()), 0, 0};
      size_t k = 0;
      for (const auto& s : X.send_segs) {
        if (s.peer != p) continue;
        if (k >= from_me.size() || from_me[k]->len != s.len)
          throw Error(PF_ERR_TRANSPORT, "channel lists of ranks " + std::to_string(me) + " and " + std::to_string(p) +
                                            " do not pair up (plan " + std::to_string(i) + ")");
        pieces.push_back(PeerPiece{s.len, X.pack_idx.p + s.off, nullptr,
                                   reinterpret_cast<double*>(base[static_cast<size_t>(p)] + from_me[k]->stage_off)});
        ++k;
      }
      if (k != from_me.size())
        throw Error(PF_ERR_TRANSPORT, "rank " + std::to_string(p) + " expects more messages from rank " +
                                          std::to_string(me) + " (plan " + std::to_string(i) + ")");
      g.seg1 = static_cast<int32_t>(pieces.size());
      sg.push_back(g);
    }
    peers.clear();
    for (const auto& s : X.recv_segs) peers.push_back(s.peer);
    std::sort(peers.begin(), peers.end());
    peers.erase(std::unique(peers.begin(), peers.end()), peers.end());
    for (int p : peers) {
      PeerGroup g{p, static_cast<int32_t>(pieces.size()), 0, 0};
      for (const auto& s : X.recv_segs) {
        if (s.peer != p) continue;
        const int32_t* idx = is_acc[i] ? nullptr : X.unpack_idx.p + s.off;
        pieces.push_back(PeerPiece{s.len, idx, reinterpret_cast<const double*>(t->arena.p + o.stage_off) + s.off,
                                   nullptr});
      }
      g.seg1 = static_cast<int32_t>(pieces.size());
      rg.push_back(g);
    }
    o.n_sends = static_cast<int32_t>(sg.size());
    o.n_recvs = static_cast<int32_t>(rg.size());
    upload_on(o.sends, sg, h->stream);
    upload_on(o.recvs, rg, h->stream);
    upload_on(o.segs, pieces, h->stream);
  }
  // allgather sites
  for (size_t j = 0; j < t->sites.size(); ++j) {
    PeerTransport::Op& o = t->sites[j];
    const int64_t c = o.count;
    std::vector<PeerGroup> sg, rg;
    std::vector<PeerPiece> pieces;
    for (int q = 0; q < W; ++q) {
      if (q == me) continue;
      const BlobSite& bs = P[static_cast<size_t>(q)].sites[j];
      if (bs.count != c) throw Error(PF_ERR_TRANSPORT, "allgather sizes differ across ranks");
      sg.push_back(PeerGroup{q, static_cast<int32_t>(pieces.size()), static_cast<int32_t>(pieces.size()) + 1, 0});
      pieces.push_back(PeerPiece{c, nullptr, o.send,
                                 reinterpret_cast<double*>(base[static_cast<size_t>(q)] + bs.stage_off) + me * c});
    }
    for (int q = 0; q < W; ++q) {
      rg.push_back(PeerGroup{q, static_cast<int32_t>(pieces.size()), static_cast<int32_t>(pieces.size()) + 1, 0});
      const double* src = q == me ? o.send : reinterpret_cast<const double*>(t->arena.p + o.stage_off) + q * c;
      pieces.push_back(PeerPiece{c, nullptr, src, o.recv + q * c});
    }
    o.n_sends = static_cast<int32_t>(sg.size());
    o.n_recvs = static_cast<int32_t>(rg.size());
    upload_on(o.sends, sg, h->stream);
    upload_on(o.recvs, rg, h->stream);
    upload_on(o.segs, pieces, h->stream);
  }
  t->ready = true;
}

}  // namespace pf
