// pf_nccl.cpp — dlopen'd NCCL point-to-point and allgather for the halo exchange.
#include "pf_nccl.hpp"

#include <dlfcn.h>
#include <nccl.h>

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
void Nccl::group_end() { ck(api().GroupEnd(), "ncclGroupEnd"); }
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
Nccl::~Nccl() {
  if (comm) api().CommDestroy(static_cast<ncclComm_t>(comm));
}

}  // namespace pf
