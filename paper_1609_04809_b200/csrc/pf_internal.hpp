// pf_internal.hpp — declarations shared by the runtime's translation units (not a public
// interface):
//   pf_runtime.cu  launches, CUDA graphs and the core C ABI (pf_gpu.h): the enqueue side
//   pf_build.cu    host level data -> device layout: SELL-32x4 operators, transfers,
//                  exchange plans, coarse packs, replicas, the bottom kernel's descriptor
//   pf_ops.cu      the heat / operator / assembly / load C ABI (pf_gpu.h, pf_fe.h)
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

#include "pf_bottom_types.hpp"
#include "pf_runtime.hpp"

namespace pf {

void set_error(const char* m);  // the thread's pf_last_error text

namespace rt {

inline unsigned grid_for(int64_t n) { return static_cast<unsigned>((n + kBlock - 1) / kBlock); }
double wall_now();
int sm_count(int device);
[[noreturn]] void invalid(const std::string& m);
[[noreturn]] void state(const std::string& m);
void trace(const char* what, int rank = -1);  // PF_TRACE=1: one stderr line per major host step

// Every kernel launch of the library: programmatic dependent launch (PF_PDL) on the
// hierarchy's stream (or `stream`), counted into the hierarchy (or, while a graph is being
// captured, into the graph entry: g_capture_counter).
struct Launcher {
  pf_hierarchy* h;
  int64_t* counter;
  cudaStream_t stream = nullptr;  // default: the hierarchy's stream
  size_t smem = 0;                // dynamic shared memory of the next launch (with_smem)
  Launcher& with_smem(size_t bytes) {
    smem = bytes;
    return *this;
  }
  template <typename... KArgs, typename... Args>
  void operator()(unsigned grid, unsigned block, void (*kern)(KArgs...), Args... args) {
    if (grid == 0) return;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(block);
    lc.dynamicSmemBytes = smem;
    smem = 0;
    lc.stream = stream ? stream : h->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = h->opt.pdl ? 1 : 0;
    PF_CUDA(cudaLaunchKernelEx(&lc, kern, static_cast<KArgs>(args)...));
    ++*counter;
  }
};

extern thread_local int64_t* g_capture_counter;
inline Launcher launcher(pf_hierarchy* h, cudaStream_t stream = nullptr) {
  return Launcher{h, g_capture_counter ? g_capture_counter : &h->launches, stream};
}

// ---- per-hierarchy options (pf_runtime.hpp Options; pf_hierarchy_set_option)
Options options_from_env();

// ---- operator views and the kernels' value-kind dispatch
inline SellView view_of(const DevVals& v, const DevSell& s) {
  const void* idx = v.vkind == 1 ? static_cast<const void*>(v.vi8.p)
                  : v.vkind == 2 ? static_cast<const void*>(v.vi16.p) : nullptr;
  return SellView{v.vals.p, s.cols.p, s.slice_ptr.p, s.row_len.p, idx, v.table.p, v.vkind,
                  static_cast<int32_t>(v.table.n)};
}
inline SellView view(const DevSell& s) { return view_of(s.vals, s); }

// Kernel instantiation for a view's value kind: f(std::integral_constant<int, kind>).
template <typename F>
void vk_dispatch(int vkind, F&& f) {
  switch (vkind) {
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    default: f(std::integral_constant<int, 0>{}); break;
  }
}

// vk_dispatch for the operator row kernels (they stage the value table, vtab_stage, and
// pick the load policy from the kVKCached bit).
template <typename F>
void vk_dispatch_rows(const DevSell& S, F&& f) {
  const bool cached = S.keep_l2;
  const int kind = S.vals.vkind == 1 && S.smem_table ? kVKSmem : S.vals.vkind;
  switch (kind | (cached ? kVKCached : 0)) {
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    case kVKSmem: f(std::integral_constant<int, kVKSmem>{}); break;
    case kVKCached: f(std::integral_constant<int, kVKCached>{}); break;
    case 1 | kVKCached: f(std::integral_constant<int, 1 | kVKCached>{}); break;
    case 2 | kVKCached: f(std::integral_constant<int, 2 | kVKCached>{}); break;
    case kVKSmem | kVKCached: f(std::integral_constant<int, kVKSmem | kVKCached>{}); break;
    default: f(std::integral_constant<int, 0>{}); break;
  }
}

// PF_TIMING=1: host-side phase times of pf_hierarchy_finalize on stderr (large grids)
struct PhaseTimer {
  bool on = std::getenv("PF_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void operator()(const char* what, int level) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[pf_timing] level %d %-22s %8.3f s\n", level, what,
                 std::chrono::duration<double>(now - t).count());
    t = now;
  }
};

// ---- pf_build.cu
constexpr size_t kCoarseSmemMax = 160 * 1024;  // opt-in shared memory for the coarse pack
void encode_values(const std::vector<double>& sv, DevVals& out, const Options& o);
void check_level(const pf_hierarchy* h, int level);
void check_vec(const pf_hierarchy* h, const pf_vector* v, int level, const char* what);
HostLevel parse_desc(const pf_level_desc& dd, int me, int world, bool need_p);
void build_dev_level(const HostLevel& H, DevLevel& D, int level, const Options& o);
void build_transfer(const HostLevel& F, DevLevel& DF, const HostLevel& Cc, const DevLevel& DC,
                    const Options& o);
void build_plans(pf_hierarchy* h, int l);
CoarsePack make_coarse_pack(const std::vector<HostLevel>& H, const std::vector<DevLevel>& D,
                            const std::array<ExchangePlan, PF_NUM_CHANNEL_KINDS>& plans,
                            DevBuf<int32_t>& sub_rows, DevBuf<int32_t>& rowptr, DevBuf<int32_t>& rowdev,
                            DevBuf<int32_t>& cols, DevBuf<double>& vals);
void build_replica(pf_hierarchy* h);
void build_bottom(pf_hierarchy* h);
void build_rep_bottom(pf_hierarchy* h);
bool bottom_for(const pf_hierarchy* h, const pf_multigrid_config& cfg);

// ---- pf_runtime.cu
size_t bottom_kernel_static_smem();
void bottom_kernel_caps(int device);          // dynamic shared memory caps of the bottom kernels
int bottom_kernel_occupancy(size_t smem);     // resident k_bottom blocks per SM
void sync(pf_hierarchy* h);
void enq_update_ms(pf_hierarchy* h, int l, double* v, int mode);
pf_vector* new_vector(pf_hierarchy* h, int level);
void solve_outer_dev(pf_hierarchy* h, pf_vector* x, const pf_vector* b, const pf_multigrid_config& cfg,
                     pf_solve_stats* st, double* residuals, int max_res);

}  // namespace rt
}  // namespace pf

// Clear any runtime error left on this thread by unrelated code, so the launch checks
// below report only this call's failures.
#define PF_API_BEGIN \
  (void)cudaGetLastError(); \
  try {
#define PF_API_END                                   \
  }                                                  \
  catch (const pf::Error& e) {                       \
    pf::set_error(e.what());                         \
    return e.code;                                   \
  }                                                  \
  catch (const std::bad_alloc&) {                    \
    pf::set_error("host out of memory");             \
    return PF_ERR_STATE;                             \
  }                                                  \
  catch (const std::exception& e) {                  \
    pf::set_error(e.what());                         \
    return PF_ERR_STATE;                             \
  }                                                  \
  return PF_OK;

