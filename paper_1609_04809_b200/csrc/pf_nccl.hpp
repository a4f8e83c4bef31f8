// pf_nccl.hpp — transports between processes (internal).
//
// Replaces Transport::send/recv and the allgather-based collectives of the reference
// (transport.cpp:92-189) for the hot-path exchanges.  Two implementations:
//   Nccl      one process per GPU; NCCL is opened with dlopen at pf_hierarchy_init_nccl
//             time, so single-GPU use and the CPU-only tests never need it, and the
//             process shares whichever libnccl.so.2 the host framework already loaded.
//   Loopback  several single-subdomain hierarchies driven by their own host threads on
//             one device (a single-GPU test bench for the multi-process code path):
//             exchanges become device-to-device copies ordered by CUDA events, with the
//             reference's watchdog semantics (a rank that never arrives raises
//             TransportError instead of hanging).
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

namespace pf {

struct ExchangePlan;  // pf_runtime.hpp

struct Transport {
  virtual ~Transport() = default;
  virtual void group_start() = 0;
  virtual void group_end(cudaStream_t s) = 0;
  virtual void send(const double* buf, int64_t count, int peer, cudaStream_t s) = 0;
  virtual void recv(double* buf, int64_t count, int peer, cudaStream_t s) = 0;
  virtual void allgather(const double* send, double* recv, int64_t count, cudaStream_t s) = 0;
  virtual void check_async() {}
  virtual bool capturable() const { return true; }  // may be recorded into CUDA graphs
  // the reference fabric's watchdog (transport.cpp:54-60): host waits on a stream that
  // carries this transport's operations give up after this many seconds (0: never)
  virtual double watchdog_seconds() const { return 0.0; }
  virtual void abort() {}
  // Direct transports (PeerTransport, pf_peer.hpp) execute a whole exchange plan as one
  // kernel that stores straight into the peers' memory, instead of pack + send/recv +
  // unpack.  run_plan: receivers scatter into v, or with wait_only only wait for their
  // messages; the caller then consumes staging(P) (the master accumulate) and ack_plan()s.
  virtual bool direct() const { return false; }
  // may an exchange run on the side stream, overlapped with the interior sweep
  virtual bool overlap_ok() const { return true; }
  virtual void run_plan(const ExchangePlan&, double*, bool, cudaStream_t) {}
  virtual const double* staging(const ExchangePlan&) const { return nullptr; }
  virtual void ack_plan(const ExchangePlan&, cudaStream_t) {}
};

struct Nccl final : Transport {
  void* lib = nullptr;
  void* comm = nullptr;
  int rank = 0, world = 1;
  void group_start() override;
  void group_end(cudaStream_t s) override;
  void send(const double* buf, int64_t count, int peer, cudaStream_t s) override;
  void recv(double* buf, int64_t count, int peer, cudaStream_t s) override;
  void allgather(const double* send, double* recv, int64_t count, cudaStream_t s) override;
  void check_async() override;
  double watchdog = 300.0;  // PF_WATCHDOG_S
  double watchdog_seconds() const override { return watchdog; }
  void abort() override;
  ~Nccl() override;
};

void nccl_unique_id(void* out, int nbytes);
std::unique_ptr<Nccl> nccl_init(int rank, int world, const void* id, int nbytes);

// Shared rendezvous of the loopback ranks.
struct LoopbackHub {
  struct Msg {
    int peer = 0;
    const double* src = nullptr;
    double* dst = nullptr;
    int64_t n = 0;
  };
  struct Post {
    std::vector<Msg> sends, recvs;
    const double* gather_src = nullptr;
    cudaEvent_t ready = nullptr, done = nullptr;
  };
  int world = 1;
  double watchdog_s = 60.0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t generation = 0;
  bool aborted = false;
  std::vector<Post> posts;
  explicit LoopbackHub(int w);
  ~LoopbackHub();
  void barrier();
  void abort();
};

struct Loopback final : Transport {
  LoopbackHub* hub = nullptr;
  int rank = 0;
  void group_start() override;
  void group_end(cudaStream_t s) override;
  void send(const double* buf, int64_t count, int peer, cudaStream_t s) override;
  void recv(double* buf, int64_t count, int peer, cudaStream_t s) override;
  void allgather(const double* send, double* recv, int64_t count, cudaStream_t s) override;
  bool capturable() const override { return false; }
};

}  // namespace pf
