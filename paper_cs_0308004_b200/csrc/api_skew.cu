// api_skew.cu -- the C ABI of DPG under data skew (section 2.3):
// run boundaries chosen from a sorted sample of the rids (dpg_skew_partition)
// and retrieval / Phase I over runs given by boundaries (dpg_retrieve_bounds,
// dpg_distribute_bounds).  The multi-kernel plan (path 2) runs them: the
// caller's boundaries are merged with the multiples of L = 2^s, so that no run
// is wider than a shared-memory stage (constraint (1)), and each
// rid finds its run by a search between the two multiples of L around it
// (bounds_run, dpg_internal.cuh).
#include <cstring>
#include <vector>

#include "api_host.h"

using namespace dpg;

namespace {

// Host bounds: bounds[0] = 0, bounds[n_runs] = n_src < 2^32, non-decreasing.
bool valid_bounds(const uint32_t* b, uint64_t n_runs, uint64_t n_src) {
  if (!b || n_runs == 0 || n_runs >= (1ull << 31) || n_src == 0 || n_src > 0xFFFFFFFFull)
    return false;
  if (b[0] != 0 || b[n_runs] != n_src) return false;
  for (uint64_t k = 0; k < n_runs; ++k)
    if (b[k] > b[k + 1]) return false;
  return true;
}

// The caller's boundaries merged with the multiples of L (ties: the caller's
// first, leaving an empty run), and the index of each multiple of L in it.
void merge_layout(const uint32_t* b, uint64_t n_runs, uint64_t n_src, uint32_t s,
                  std::vector<uint32_t>* M, std::vector<uint32_t>* tab) {
  const uint64_t L = 1ull << s, J = (n_src + L - 1) >> s;
  M->clear();
  M->reserve(n_runs + J);
  tab->assign(J + 1, 0);
  uint64_t k = 0;
  for (uint64_t j = 1; j < J; ++j) {
    const uint64_t g = j * L;
    while (k <= n_runs && b[k] <= g) M->push_back(b[k++]);
    (*tab)[j] = (uint32_t)M->size();
    M->push_back((uint32_t)g);
  }
  while (k <= n_runs) M->push_back(b[k++]);
  (*tab)[J] = (uint32_t)(M->size() - 1);
}

// Upload the merged layout (stream-ordered scratch, freed by the caller with
// cudaFreeAsync on the same stream).
dpg_status_t upload_layout(const uint32_t* bounds, uint64_t n_runs, uint64_t n_src, uint32_t s,
                           cudaStream_t st, BoundsLayout* bl, void** mem) {
  std::vector<uint32_t> M, tab;
  merge_layout(bounds, n_runs, n_src, s, &M, &tab);
  if (M.size() - 1 >= (1ull << 31)) return DPG_ERR_UNSUPPORTED;
  const uint64_t off_tab = align_up(M.size() * 4, 256);
  if (ws_malloc(mem, off_tab + tab.size() * 4, st) != cudaSuccess) {
    cudaGetLastError();
    return DPG_ERR_OOM;
  }
  uint8_t* base = (uint8_t*)*mem;
  // (pageable sources: the copies are staged before the calls return)
  cudaError_t e = cudaMemcpyAsync(base, M.data(), M.size() * 4, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(base + off_tab, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) {
    cudaFreeAsync(*mem, st);
    return cuda_status(e);
  }
  bl->bmap = (const uint32_t*)base;
  bl->btab = (const uint32_t*)(base + off_tab);
  bl->K = M.size() - 1;
  return DPG_OK;
}

}  // namespace

extern "C" {

dpg_status_t dpg_skew_partition(const uint32_t* rids, uint64_t n_out, uint64_t n_src,
                                uint32_t num_runs, uint32_t sample_size, uint64_t seed,
                                uint32_t* bounds_out, uint32_t* n_runs_out, dpg_stream_t stream) {
  t_launches = 0;
  if (n_out == 0 || !rids || !bounds_out || !n_runs_out || num_runs == 0 ||
      sample_size < num_runs || n_src == 0)
    return DPG_ERR_INVALID_ARG;
  if (sample_size > kSkewMaxSample || n_src > 0xFFFFFFFFull) return DPG_ERR_UNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream;
  void* mem = nullptr;
  if (ws_malloc(&mem, ((uint64_t)num_runs + 2) * 4, st) != cudaSuccess) {
    cudaGetLastError();
    return DPG_ERR_OOM;
  }
  uint32_t* dev = (uint32_t*)mem;
  uint32_t nl = 0;
  std::vector<uint32_t> h((uint64_t)num_runs + 2);
  cudaError_t e = launch_skew_partition(rids, n_out, (uint32_t)n_src, num_runs, sample_size, seed,
                                        dev + 1, dev, st, &nl);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), dev, h.size() * 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(mem, st);
  if (e == cudaSuccess) {
    *n_runs_out = h[0];
    std::memcpy(bounds_out, h.data() + 1, ((uint64_t)h[0] + 1) * 4);
  }
  t_launches = nl;
  return cuda_status(e);
}

dpg_status_t dpg_retrieve_bounds(const void* src, size_t rec_bytes, uint64_t n_src,
                                 const uint32_t* rids, uint64_t n_out, const uint32_t* bounds,
                                 uint64_t n_runs, void* dst, dpg_stream_t stream) {
  t_launches = 0;
  if (rec_bytes == 0 || !valid_bounds(bounds, n_runs, n_src)) return DPG_ERR_INVALID_ARG;
  if (n_out == 0) return DPG_OK;
  if (!src || !rids || !dst) return DPG_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  dpg_options_t o;
  std::memset(&o, 0, sizeof(o));
  o.path = 2;
  dpg_plan_t p;
  dpg_status_t ps = make_plan(rec_bytes, n_src, n_out, 0, &o, current_sm_count(), &p);
  if (ps != DPG_OK) return ps;
  BoundsLayout bl;
  void* mem = nullptr;
  ps = upload_layout(bounds, n_runs, n_src, p.log2_run, st, &bl, &mem);
  if (ps != DPG_OK) return ps;
  o.log2_run = p.log2_run;
  t_bounds = &bl;
  ps = run_dpg(src, rec_bytes, n_src, rids, n_out, nullptr, 0, dst, st, &o);
  t_bounds = nullptr;
  const uint32_t nl = t_launches;
  cudaFreeAsync(mem, st);
  t_launches = nl;
  return ps;
}

dpg_status_t dpg_distribute_bounds(const uint32_t* rids, uint64_t n_out, uint64_t n_src,
                                   const uint32_t* bounds, uint64_t n_runs, uint32_t log2_run,
                                   uint64_t* pairs_out, uint64_t* run_start_out,
                                   uint64_t* num_runs_out, dpg_stream_t stream) {
  t_launches = 0;
  if (!valid_bounds(bounds, n_runs, n_src) || log2_run > 31 || !num_runs_out)
    return DPG_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<uint32_t> M, tab;
  merge_layout(bounds, n_runs, n_src, log2_run, &M, &tab);
  *num_runs_out = M.size() - 1;
  if (!run_start_out) return DPG_OK;      // (a size query)
  BoundsLayout bl;
  void* mem = nullptr;
  dpg_status_t ps = upload_layout(bounds, n_runs, n_src, log2_run, st, &bl, &mem);
  if (ps != DPG_OK) return ps;
  t_bounds = &bl;
  ps = dpg_distribute(rids, n_out, n_src, log2_run, pairs_out, run_start_out, stream, nullptr);
  t_bounds = nullptr;
  const uint32_t nl = t_launches;
  cudaFreeAsync(mem, st);
  t_launches = nl;
  return ps;
}

}  // extern "C"
