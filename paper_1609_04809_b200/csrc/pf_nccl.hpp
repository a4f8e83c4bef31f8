// pf_nccl.hpp — NCCL transport for one-process-per-GPU runs (internal).
//
// NCCL is opened with dlopen at pf_hierarchy_init_nccl time, so single-GPU use and
// the CPU-only tests never need it, and the process shares whichever libnccl.so.2
// the host framework (torch) already loaded.  Replaces Transport::send/recv and the
// allgather-based allreduce of the reference (transport.cpp:92-165).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>

namespace pf {

struct Nccl {
  void* lib = nullptr;
  void* comm = nullptr;
  int rank = 0, world = 1;
  void group_start();
  void group_end();
  void send(const double* buf, int64_t count, int peer, cudaStream_t s);
  void recv(double* buf, int64_t count, int peer, cudaStream_t s);
  void allgather(const double* send, double* recv, int64_t count, cudaStream_t s);
  void check_async();
  ~Nccl();
};

void nccl_unique_id(void* out, int nbytes);
std::unique_ptr<Nccl> nccl_init(int rank, int world, const void* id, int nbytes);

}  // namespace pf
