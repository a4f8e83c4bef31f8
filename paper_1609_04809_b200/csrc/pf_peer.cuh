// pf_peer.cuh — peer-memory exchange kernels (the PeerTransport of pf_peer.cu).
//
// Replaces ParFECommunicator::scatter / update_master_slave (fecomm.cpp:25-62) and the
// allgather behind allreduce_sum (transport.cpp:139-165) for ranks that can map each
// other's device memory: other processes on the same GPU or on NVLink/NVSwitch peers
// (CUDA IPC), or other hierarchies of the same process.  One kernel moves a whole message
// group: the sending blocks gather the values straight out of the local vector and STORE
// them into the receiving rank's staging area (no NCCL, no send buffer), then raise a
// per-(sender, receiver) sequence flag in the receiver's control block; the receiving
// blocks wait for the flags and scatter the staged values into the local vector.  Every
// operation is an ordinary kernel, so an exchange can be recorded into a CUDA graph.
//
// Protocol, per ordered pair (s -> r), with monotonically increasing counters:
//   s: wait ack_r >= sent  (r consumed everything s sent before: the staging may be reused)
//      store payload into r's staging; fence.sys; flag[s] at r := sent + 1 (release.sys)
//   r: wait flag[s] >= rcvd + 1 (acquire.sys); read the staging (L2, bypassing L1);
//      ack[r] at s := rcvd + 1 (release.sys)
// Both sides walk the same plans in the same order (the channel lists pair up), so the
// counters stay in lockstep.  A wait that exceeds the watchdog sets the control block's
// error word and returns (the reference fabric's TransportError, transport.cpp:54-60)
// instead of hanging the device.
#pragma once

#include <cstdint>

#include "pf_types.hpp"

namespace pf {

constexpr int kPeerMaxWorld = 64;
constexpr int kPeerBlock = 512;

// Control block of one rank (the first bytes of its peer-visible arena).
struct PeerCtl {
  unsigned long long flag[kPeerMaxWorld];  // flag[p]: message groups rank p delivered here
  unsigned long long ack[kPeerMaxWorld];   // ack[p]: this rank's groups rank p consumed
  unsigned long long sent[kPeerMaxWorld];  // local: groups sent to p
  unsigned long long rcvd[kPeerMaxWorld];  // local: groups received from p
  unsigned int error;                      // watchdog tripped (1), waiting on error_peer
  int error_peer;
};

// One contiguous piece of a message.
//   send: dst[i] = idx ? v[idx[i]] : src[i]   (dst in the receiver's staging)
//   recv: (idx ? v[idx[i]] : dst[i]) = src[i] (src in this rank's staging)
struct PeerPiece {
  int64_t n;
  const int32_t* idx;
  const double* src;
  double* dst;
};

// The pieces exchanged with one peer in one message group.  peer == me on the receiving
// side: a local copy (allgather's own slot), no synchronisation.
struct PeerGroup {
  int32_t peer, seg0, seg1, pad;
};

struct PeerArgs {
  const PeerGroup* sends;
  const PeerGroup* recvs;
  const PeerPiece* segs;
  int32_t n_sends, n_recvs;
  int32_t me;
  int32_t wait_only;  // receivers only wait (the master accumulate reads the staging next)
  PeerCtl* mine;
  PeerCtl* const* remote;  // remote[p]: rank p's control block, mapped here
  unsigned long long timeout_ns;
};

__device__ __forceinline__ unsigned long long peer_ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void peer_st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long peer_clock_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Thread 0 spins until *p >= want; false (and the error word set) after the watchdog.
__device__ __forceinline__ bool peer_wait(const PeerArgs& a, const unsigned long long* p, unsigned long long want,
                                          int peer) {
  if (peer_ld_acquire(p) >= want) return true;
  const unsigned long long t0 = peer_clock_ns();
  unsigned int ns = 32;
  for (;;) {
    if (peer_ld_acquire(p) >= want) return true;
    if (*reinterpret_cast<volatile unsigned int*>(&a.mine->error)) return false;
    if (a.timeout_ns && peer_clock_ns() - t0 > a.timeout_ns) {
      a.mine->error_peer = peer;
      atomicExch(&a.mine->error, 1u);
      return false;
    }
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
  }
}

// One block per peer group: blocks [0, n_sends) send, the rest receive.  The kernel waits
// for its predecessor (PDL) but never releases its dependents early: a dependent grid
// parked on griddepcontrol.wait would hold SM slots that a peer sharing this GPU needs to
// deliver the message this kernel waits for.
static __global__ void __launch_bounds__(kPeerBlock) k_peer_exchange(PeerArgs a, double* __restrict__ v) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ int s_ok;
  __shared__ unsigned long long s_seq;
  const bool sending = static_cast<int>(blockIdx.x) < a.n_sends;
  const PeerGroup g = sending ? a.sends[blockIdx.x] : a.recvs[blockIdx.x - a.n_sends];
  const int p = g.peer;
  const bool local = !sending && p == a.me;
  if (threadIdx.x == 0) {
    s_ok = 1;
    if (!local) {
      volatile unsigned long long* ctr = sending ? a.mine->sent : a.mine->rcvd;
      const unsigned long long seq = ctr[p];
      s_seq = seq;
      s_ok = sending ? peer_wait(a, &a.mine->ack[p], seq, p) : peer_wait(a, &a.mine->flag[p], seq + 1, p);
    }
  }
  __syncthreads();
  if (!s_ok) return;
  if (sending) {
    for (int k = g.seg0; k < g.seg1; ++k) {
      const PeerPiece s = a.segs[k];
      if (s.idx) {
        for (int64_t i = threadIdx.x; i < s.n; i += kPeerBlock) s.dst[i] = v[s.idx[i]];
      } else {
        for (int64_t i = threadIdx.x; i < s.n; i += kPeerBlock) s.dst[i] = s.src[i];
      }
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      peer_st_release(&a.remote[p]->flag[a.me], s_seq + 1);
      a.mine->sent[p] = s_seq + 1;
    }
    return;
  }
  if (a.wait_only && !local) return;  // k_peer_ack acknowledges after the consumer ran
  for (int k = g.seg0; k < g.seg1; ++k) {
    const PeerPiece s = a.segs[k];
    if (s.idx) {
      for (int64_t i = threadIdx.x; i < s.n; i += kPeerBlock) v[s.idx[i]] = __ldcg(s.src + i);
    } else {
      for (int64_t i = threadIdx.x; i < s.n; i += kPeerBlock) s.dst[i] = __ldcg(s.src + i);
    }
  }
  if (local) return;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    peer_st_release(&a.remote[p]->ack[a.me], s_seq + 1);
    a.mine->rcvd[p] = s_seq + 1;
  }
}

// After a wait_only exchange and the kernel that consumed the staging: acknowledge every
// receiving group (one thread per group).
static __global__ void k_peer_ack(PeerArgs a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n_recvs) return;
  const int p = a.recvs[i].peer;
  if (p == a.me || a.mine->error) return;
  const unsigned long long seq = a.mine->rcvd[p] + 1;
  __threadfence_system();
  peer_st_release(&a.remote[p]->ack[a.me], seq);
  a.mine->rcvd[p] = seq;
}

}  // namespace pf
