// pf_nccl.cpp — dlopen'd NCCL point-to-point and allgather for the halo exchange.
#include "pf_nccl.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstring>
#include <string>

#include "pf_runtime.hpp"

namespace pf {

namespace {

struct Api {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Api& api() {
  static Api a;
  if (a.lib) return a;
  for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
    a.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    if (a.lib) break;
  }
  if (!a.lib) throw Error(PF_ERR_TRANSPORT, std::string("cannot dlopen libnccl.so.2: ") + dlerror());
  auto sym = [&](const char* n) {
    void* p = dlsym(a.lib, n);
    if (!p) throw Error(PF_ERR_TRANSPORT, std::string("libnccl lacks ") + n);
    return p;
  };
  a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
  a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
  a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
  a.CommAbort = reinterpret_cast<decltype(a.CommAbort)>(sym("ncclCommAbort"));
  a.CommGetAsyncError = reinterpret_cast<decltype(a.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
  a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
  a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
  a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
  a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
  a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
  a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
  return a;
}

void ck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(PF_ERR_TRANSPORT, std::string(what) + ": " + api().GetErrorString(r));
}

}  // namespace

void nccl_unique_id(void* out, int nbytes) {
  if (nbytes < static_cast<int>(sizeof(ncclUniqueId)))
    throw Error(PF_ERR_INVALID_ARGUMENT, "unique id buffer smaller than 128 bytes");
  ncclUniqueId id;
  ck(api().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof id);
}

std::unique_ptr<Nccl> nccl_init(int rank, int world, const void* id, int nbytes) {
  if (nbytes < static_cast<int>(sizeof(ncclUniqueId)))
    throw Error(PF_ERR_INVALID_ARGUMENT, "unique id buffer smaller than 128 bytes");
  auto n = std::make_unique<Nccl>();
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  ncclComm_t comm = nullptr;
  ck(api().CommInitRank(&comm, world, uid, rank), "ncclCommInitRank");
  n->comm = comm;
  n->lib = api().lib;
  n->rank = rank;
  n->world = world;
  return n;
}

void Nccl::group_start() { ck(api().GroupStart(), "ncclGroupStart"); }
void Nccl::group_end(cudaStream_t) { ck(api().GroupEnd(), "ncclGroupEnd"); }
void Nccl::send(const double* buf, int64_t count, int peer, cudaStream_t s) {
  ck(api().Send(buf, static_cast<size_t>(count), ncclFloat64, peer, static_cast<ncclComm_t>(comm), s),
     "ncclSend");
}
void Nccl::recv(double* buf, int64_t count, int peer, cudaStream_t s) {
  ck(api().Recv(buf, static_cast<size_t>(count), ncclFloat64, peer, static_cast<ncclComm_t>(comm), s),
     "ncclRecv");
}
void Nccl::allgather(const double* send, double* recv, int64_t count, cudaStream_t s) {
  ck(api().AllGather(send, recv, static_cast<size_t>(count), ncclFloat64,
                     static_cast<ncclComm_t>(comm), s),
     "ncclAllGather");
}
void Nccl::check_async() {
  ncclResult_t r = ncclSuccess;
  ck(api().CommGetAsyncError(static_cast<ncclComm_t>(comm), &r), "ncclCommGetAsyncError");
  ck(r, "NCCL async error");
}
void Nccl::abort() {
  if (comm) api().CommAbort(static_cast<ncclComm_t>(comm));
  comm = nullptr;
}
Nccl::~Nccl() {
  if (comm) api().CommDestroy(static_cast<ncclComm_t>(comm));
}

// ---------------------------------------------------------------- loopback --

LoopbackHub::LoopbackHub(int w) : world(w), posts(static_cast<size_t>(w)) {
  for (Post& p : posts) {
    cuda_check(cudaEventCreateWithFlags(&p.ready, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventCreateWithFlags(&p.done, cudaEventDisableTiming), "cudaEventCreate");
  }
}

LoopbackHub::~LoopbackHub() {
  for (Post& p : posts) {
    if (p.ready) cudaEventDestroy(p.ready);
    if (p.done) cudaEventDestroy(p.done);
  }
}

// Host barrier of all loopback ranks with the reference fabric's watchdog
// (transport.cpp:44-65): a missing rank surfaces as TransportError.
void LoopbackHub::barrier() {
  std::unique_lock<std::mutex> lock(mu);
  if (aborted) throw Error(PF_ERR_TRANSPORT, "loopback fabric aborted");
  const int64_t gen = generation;
  if (++arrived == world) {
    arrived = 0;
    ++generation;
    cv.notify_all();
    return;
  }
  if (!cv.wait_for(lock, std::chrono::duration<double>(watchdog_s),
                   [&] { return generation != gen || aborted; })) {
    aborted = true;
    cv.notify_all();
    throw Error(PF_ERR_TRANSPORT, "loopback watchdog: a rank did not reach the exchange");
  }
  if (aborted) throw Error(PF_ERR_TRANSPORT, "loopback fabric aborted");
}

void LoopbackHub::abort() {
  std::lock_guard<std::mutex> lock(mu);
  aborted = true;
  cv.notify_all();
}

void Loopback::group_start() {
  auto& p = hub->posts[static_cast<size_t>(rank)];
  p.sends.clear();
  p.recvs.clear();
}

void Loopback::send(const double* buf, int64_t count, int peer, cudaStream_t) {
  hub->posts[static_cast<size_t>(rank)].sends.push_back({peer, buf, nullptr, count});
}

void Loopback::recv(double* buf, int64_t count, int peer, cudaStream_t) {
  hub->posts[static_cast<size_t>(rank)].recvs.push_back({peer, nullptr, buf, count});
}

// B1: every rank's sends are posted and their data ready-event recorded; each rank pulls
// its receives behind the senders' events; B2: done-events recorded; every sender waits
// for its receivers before it may overwrite its send buffers; B3: posts may be reused.
void Loopback::group_end(cudaStream_t s) {
  auto& mine = hub->posts[static_cast<size_t>(rank)];
  cuda_check(cudaEventRecord(mine.ready, s), "cudaEventRecord");
  hub->barrier();
  // NCCL semantics: the k-th receive from a peer in a group matches that peer's k-th
  // send to this rank in the same group
  std::vector<int> nth(static_cast<size_t>(hub->world), 0);
  for (const auto& r : mine.recvs) {
    const auto& src = hub->posts[static_cast<size_t>(r.peer)];
    const LoopbackHub::Msg* m = nullptr;
    int k = nth[static_cast<size_t>(r.peer)]++;
    for (const auto& snd : src.sends)
      if (snd.peer == rank && k-- == 0) {
        m = &snd;
        break;
      }
    if (!m || m->n != r.n) {
      hub->abort();
      throw Error(PF_ERR_TRANSPORT, "loopback: unmatched receive from rank " + std::to_string(r.peer));
    }
    cuda_check(cudaStreamWaitEvent(s, src.ready, 0), "cudaStreamWaitEvent");
    cuda_check(cudaMemcpyAsync(r.dst, m->src, sizeof(double) * static_cast<size_t>(r.n),
                               cudaMemcpyDeviceToDevice, s), "cudaMemcpyAsync");
  }
  cuda_check(cudaEventRecord(mine.done, s), "cudaEventRecord");
  hub->barrier();
  for (const auto& snd : mine.sends)
    cuda_check(cudaStreamWaitEvent(s, hub->posts[static_cast<size_t>(snd.peer)].done, 0), "cudaStreamWaitEvent");
  hub->barrier();
}

void Loopback::allgather(const double* send, double* recv, int64_t count, cudaStream_t s) {
  auto& mine = hub->posts[static_cast<size_t>(rank)];
  mine.gather_src = send;
  cuda_check(cudaEventRecord(mine.ready, s), "cudaEventRecord");
  hub->barrier();
  for (int q = 0; q < hub->world; ++q) {
    const auto& src = hub->posts[static_cast<size_t>(q)];
    cuda_check(cudaStreamWaitEvent(s, src.ready, 0), "cudaStreamWaitEvent");
    cuda_check(cudaMemcpyAsync(recv + static_cast<int64_t>(q) * count, src.gather_src,
                               sizeof(double) * static_cast<size_t>(count), cudaMemcpyDeviceToDevice, s),
               "cudaMemcpyAsync");
  }
  cuda_check(cudaEventRecord(mine.done, s), "cudaEventRecord");
  hub->barrier();
  for (int q = 0; q < hub->world; ++q)
    cuda_check(cudaStreamWaitEvent(s, hub->posts[static_cast<size_t>(q)].done, 0), "cudaStreamWaitEvent");
  hub->barrier();
}

}  // namespace pf
