// parfem_gpu_bridge.hpp — the reference-side binding of the B200 hot path.
//
// This file belongs in the reference tree (proj/src or proj/integration): it is the code
// a parfem maintainer adds to switch solve_outer to the GPU.  It includes the reference's
// own headers and calls only the C ABI of libpf_gpu.so (include/pf_gpu.h) through the
// header-only shim include/parfem_b200.hpp.
#pragma once

#include "parfem/multigrid.hpp"

namespace parfem::gpu {

// Drop-in for parfem::solve_outer (multigrid.cpp:210-246): same arguments, same
// SolveStats, NoConvergenceError on a stall.  Collective like the original: every rank
// thread of run_on_ranks calls it together.  The first call for a hierarchy uploads its
// levels (system CSR, owns_row, classes, channels, prolong_map) to the GPU of this rank
// (rank % device count); later calls only move x and b.  With several ranks the
// hierarchies exchange through the library's loopback transport, and every rank holds
// the replicated coarse level, gathered once over the reference's own Transport.
SolveStats solve_outer(MultigridHierarchy& h, DistributedVector& x, const DistributedVector& b,
                       const MultigridConfig& cfg);

// Forget the device mirror of h (call before h is destroyed).  Collective.
void release(const MultigridHierarchy& h);

}  // namespace parfem::gpu
