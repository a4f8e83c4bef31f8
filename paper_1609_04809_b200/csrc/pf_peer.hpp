// pf_peer.hpp — the peer-memory transport (internal; kernels in pf_peer.cuh).
//
// Ranks in separate processes (one per GPU over NVLink/NVSwitch, or several on one GPU)
// map each other's exchange arenas with CUDA IPC; ranks that are hierarchies of one
// process use the arena pointers directly.  Setup is two collective steps driven by the
// host framework (like the NCCL unique id): every rank exports a blob describing its
// arena (pf_hierarchy_peer_export), the blobs are allgathered by the caller (files,
// torch.distributed, the reference's own fabric ...), and every rank imports all of them
// (pf_hierarchy_init_peer).  From then on every exchange of the V-cycle is one kernel
// launch, capturable into the solve's CUDA graph.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <vector>

#include "pf_nccl.hpp"
#include "pf_peer.cuh"
#include "pf_runtime.hpp"

namespace pf {

struct PeerTransport final : Transport {
  pf_hierarchy* h = nullptr;
  int rank = 0, world = 1;
  bool ready = false;
  bool in_process = false;           // some peers are hierarchies of this process
  DevBuf<char> arena;                // PeerCtl, then every plan's and site's staging
  int64_t arena_bytes = 0;
  std::vector<void*> opened;         // IPC-mapped peer arenas (closed at destruction)
  DevBuf<PeerCtl*> remote_ctl;       // [world]: every rank's control block, mapped here
  unsigned long long timeout_ns = 0;
  struct Op {                        // one plan or allgather site, ready to launch
    DevBuf<PeerGroup> sends, recvs;
    DevBuf<PeerPiece> segs;
    int32_t n_sends = 0, n_recvs = 0;
    int64_t stage_off = 0;           // this rank's staging of the op inside the arena
    const double* send = nullptr;    // allgather site: registered send / recv / count
    double* recv = nullptr;
    int64_t count = 0;
  };
  std::vector<Op> plans, sites;
  std::map<const double*, int> site_of;  // allgather recv pointer -> site

  PeerCtl* ctl() const { return reinterpret_cast<PeerCtl*>(arena.p); }
  PeerArgs args(const Op& o, bool wait_only) const;
  void launch_exchange(const Op& o, double* v, bool wait_only, cudaStream_t s);

  void group_start() override;
  void group_end(cudaStream_t s) override;
  void send(const double* buf, int64_t count, int peer, cudaStream_t s) override;
  void recv(double* buf, int64_t count, int peer, cudaStream_t s) override;
  void allgather(const double* send, double* recv, int64_t count, cudaStream_t s) override;
  void check_async() override;
  bool direct() const override { return true; }
  // in-process peers: no side-stream overlap (a forked graph's branches may share a
  // hardware queue with another rank's waiting exchange)
  bool overlap_ok() const override { return !in_process; }
  void run_plan(const ExchangePlan& P, double* v, bool wait_only, cudaStream_t s) override;
  const double* staging(const ExchangePlan& P) const override;
  void ack_plan(const ExchangePlan& P, cudaStream_t s) override;
  ~PeerTransport() override;
};

// Bytes of this rank's export blob (allocating the arena on the first call); copies the
// blob into buf when cap is large enough.
int64_t peer_export(pf_hierarchy* h, void* buf, int64_t cap);
// Import every rank's blob (world blobs, each at blobs + r * stride) and activate.
void peer_import(pf_hierarchy* h, const void* blobs, int64_t stride);

}  // namespace pf
