// api_host.h -- host-side helpers shared by the C ABI translation units
// (api.cu: retrieval, planning, workspace; api_apps.cu: sort, joins, lookups).
// Internal to libdpg.so; not part of include/dpg.h.
#pragma once
#include <cstdint>
#include <mutex>

#include "dpg.h"
#include "dpg_internal.cuh"

namespace dpg {

extern thread_local uint32_t t_launches;   // kernel launches of the last call (dpg_last_launch_count)

int current_sm_count();
uint64_t current_l2_bytes();
unsigned long long* device_status();       // the per-device status word (dpg_sync_status)
uint64_t align_up(uint64_t x, uint64_t a);
uint32_t pow2_divisor(uint64_t x);         // largest power of two <= 16 dividing x
bool overlaps(const void* a, uint64_t na, const void* b, uint64_t nb);
uint64_t l2_run_budget(uint64_t l2_bytes);
// Library-owned workspace, persistent per (device, stream): grid-barrier and
// counter words (zero-restored by the kernels) and `bytes` of scratch.
// *hold keeps the (device, stream) entry locked until the caller's launches
// are enqueued (declare it before the call, in the entry point's scope).
using WsHold = std::unique_lock<std::recursive_mutex>;
dpg_status_t persist_ws(cudaStream_t st, uint64_t K, uint64_t bytes, uint32_t** gbar,
                        uint32_t** total, void** scratch, WsHold* hold);
// Stream-ordered scratch from the library's private pool (cudaFreeAsync frees it).
cudaError_t ws_malloc(void** p, size_t bytes, cudaStream_t st);
template <typename T>
inline cudaError_t ws_malloc(T** p, size_t bytes, cudaStream_t st) {
  return ws_malloc(reinterpret_cast<void**>(p), bytes, st);
}
dpg_status_t cuda_status(cudaError_t e);
dpg_status_t make_plan(uint64_t rec, uint64_t n_src, uint64_t n_out, uint64_t pay,
                       const dpg_options_t* opt, int sm, dpg_plan_t* p);
// Boundary-mode runs (section 2.3): the device layout of the current call on
// this thread (set around run_dpg / dpg_distribute by the bounds entry points).
struct BoundsLayout {
  const uint32_t* bmap;   // [K+1] run starts: the caller's bounds merged with the multiples of L
  const uint32_t* btab;   // [ceil(n_src/L)+1] index in bmap of the run starting at h*L
  uint64_t K;
};
extern thread_local const BoundsLayout* t_bounds;
dpg_status_t run_dpg(const void* src, uint64_t rec, uint64_t n_src, const uint32_t* rids,
                     uint64_t n_out, const void* pay_src, uint64_t pay, void* dst, cudaStream_t st,
                     const dpg_options_t* opt);

}  // namespace dpg
