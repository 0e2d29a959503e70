// api_apps.cu -- the C ABI of the paper's applications of DPG (include/dpg.h):
// the three-phase key-pointer sort (section 3), the DPG-Sort join
// (P:595-615), and the batch index lookups (section 4).  The
// retrieval path itself, planning and the shared host helpers are in api.cu.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "api_host.h"

using namespace dpg;

namespace {

dpg_status_t btree_args(const uint32_t* const* levels, const uint64_t* level_n,
                               uint32_t n_levels, const uint32_t* rids, BTreeIdx* T) {
  if (!levels || !level_n || !rids || n_levels == 0 || n_levels > (uint32_t)kBtMaxLevels)
    return DPG_ERR_INVALID_ARG;
  std::memset(T, 0, sizeof(*T));
  T->levels = n_levels;
  T->rids = rids;
  for (uint32_t t = 0; t < n_levels; ++t) {
    if (!levels[t] || level_n[t] == 0 || level_n[t] >= (1ull << 32) || (uintptr_t)levels[t] % 64)
      return DPG_ERR_INVALID_ARG;
    if (t && level_n[t] != (level_n[t - 1] + 15) / 16) return DPG_ERR_INVALID_ARG;
    T->lv[t] = levels[t];
    T->n[t] = (uint32_t)level_n[t];
  }
  if (level_n[n_levels - 1] > 16) return DPG_ERR_INVALID_ARG;
  return DPG_OK;
}

}  // namespace

extern "C" {

dpg_status_t dpg_sort_rids(const void* src, size_t rec_bytes, uint64_t n, size_t key_off,
                           size_t key_bytes, uint32_t* rids_out, dpg_stream_t stream) {
  WsHold ws_hold;   // the stream's workspace stays ours until the launches are enqueued
  // Phases 1-2 of three-phase sorting: stable rid order by key.
  t_launches = 0;
  if (rec_bytes == 0 || key_bytes == 0 || key_bytes > 12 || key_off + key_bytes > rec_bytes)
    return DPG_ERR_INVALID_ARG;
  if (n == 0) return DPG_OK;
  if (!src || !rids_out) return DPG_ERR_INVALID_ARG;
  if (n >= (1ull << 32) || rec_bytes > UINT32_MAX / 2) return DPG_ERR_UNSUPPORTED;
  uint64_t src_bytes;
  if (__builtin_mul_overflow(n, (uint64_t)rec_bytes, &src_bytes)) return DPG_ERR_INVALID_ARG;
  if (overlaps(rids_out, n * 4, src, src_bytes)) return DPG_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int sm = current_sm_count();
  uint32_t *gbar = nullptr, *total = nullptr;
  void* ws = nullptr;
  dpg_status_t w = persist_ws(st, 1, sort_ws_bytes(n, sm), &gbar, &total, &ws, &ws_hold);
  if (w != DPG_OK) return w;
  uint32_t nl = 0;
  cudaError_t e = launch_sort_rids((const uint8_t*)src, (uint32_t)rec_bytes, n, (uint32_t)key_off,
                                   (uint32_t)key_bytes, (uint8_t*)ws, rids_out, gbar + 16, sm, st,
                                   &nl);
  t_launches = nl;
  return cuda_status(e);
}

dpg_status_t dpg_sort(const void* src, size_t rec_bytes, uint64_t n, size_t key_off,
                      size_t key_bytes, void* dst, dpg_stream_t stream) {
  // The whole three-phase sort: phases 1-2 (dpg_sort_rids), then phase 3 =
  // DPG record retrieval of the records in sorted rid order.
  t_launches = 0;
  if (n == 0) return (rec_bytes && key_bytes && key_off + key_bytes <= rec_bytes) ? DPG_OK
                                                                                 : DPG_ERR_INVALID_ARG;
  if (!dst) return DPG_ERR_INVALID_ARG;
  uint64_t bytes;
  if (__builtin_mul_overflow(n, (uint64_t)rec_bytes, &bytes)) return DPG_ERR_INVALID_ARG;
  if (overlaps(dst, bytes, src, bytes)) return DPG_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  void* rids = nullptr;
  if (ws_malloc(&rids, n * 4 + 64, st) != cudaSuccess) {
    cudaGetLastError();
    return DPG_ERR_OOM;
  }
  dpg_status_t s = dpg_sort_rids(src, rec_bytes, n, key_off, key_bytes, (uint32_t*)rids, stream);
  uint32_t nl = t_launches;
  if (s == DPG_OK) {
    s = run_dpg(src, rec_bytes, n, (const uint32_t*)rids, n, nullptr, 0, dst, st, nullptr);
    nl += t_launches;
  }
  cudaFreeAsync(rids, st);
  t_launches = nl;
  return s;
}

dpg_status_t dpg_fk_join_direct(const void* fact, size_t fact_bytes, uint64_t n_fact,
                                const uint32_t* fk_col, const void* dim, size_t rec_bytes,
                                uint64_t n_dim, void* out, dpg_stream_t stream) {
  // The standard join the paper compares against: for each fact
  // row, one random access to the dimension record its key names.
  t_launches = 0;
  if (rec_bytes == 0) return DPG_ERR_INVALID_ARG;
  if (n_fact == 0) return DPG_OK;
  if ((fact_bytes && !fact) || !fk_col || !dim || !out || n_dim == 0) return DPG_ERR_INVALID_ARG;
  uint64_t row, out_bytes, fact_total, dim_total;
  if (__builtin_add_overflow((uint64_t)fact_bytes, (uint64_t)rec_bytes, &row) ||
      __builtin_mul_overflow(n_fact, row, &out_bytes) ||
      __builtin_mul_overflow(n_fact, (uint64_t)fact_bytes, &fact_total) ||
      __builtin_mul_overflow(n_dim, (uint64_t)rec_bytes, &dim_total))
    return DPG_ERR_INVALID_ARG;
  if (row > UINT32_MAX / 2) return DPG_ERR_UNSUPPORTED;
  if (overlaps(out, out_bytes, fact, fact_total) || overlaps(out, out_bytes, dim, dim_total) ||
      overlaps(out, out_bytes, fk_col, n_fact * 4))
    return DPG_ERR_INVALID_ARG;
  unsigned long long* status = device_status();
  if (!status) return DPG_ERR_CUDA;
  const uint32_t W = pow2_divisor(fact_bytes | rec_bytes | (uintptr_t)fact | (uintptr_t)dim |
                                  (uintptr_t)out);
  uint32_t nl = 0;
  cudaError_t e = launch_zip_gather((const uint8_t*)fact, (uint32_t)fact_bytes, (const uint8_t*)dim,
                                    (uint32_t)rec_bytes, n_dim, fk_col, n_fact, (uint8_t*)out, W,
                                    current_sm_count(), (cudaStream_t)stream, &nl, status);
  t_launches = nl;
  return cuda_status(e);
}

dpg_status_t dpg_fk_join_sort(const void* fact, size_t fact_bytes, uint64_t n_fact,
                              const uint32_t* fk_col, const void* dim, size_t rec_bytes,
                              uint64_t n_dim, void* out, dpg_stream_t stream) {
  WsHold ws_hold;   // the stream's workspace stays ours until the launches are enqueued
  // DPG-Sort join: sort the pairs (rid_R = i, rid_F =
  // fk[i]) by rid_F (stable radix sort, sort.cu), move the records of R (the
  // fact rows) into a temporary file in that order by DPG retrieval, then join
  // the temporary file with F read in rid_F order.  out row j = fact[rid_R_j]
  // ++ dim[rid_F_j]; rows with fk >= n_dim stay unwritten and are reported.
  t_launches = 0;
  if (rec_bytes == 0 || fact_bytes == 0) return DPG_ERR_INVALID_ARG;
  if (n_fact == 0) return DPG_OK;
  if (!fact || !fk_col || !dim || !out || n_dim == 0) return DPG_ERR_INVALID_ARG;
  if (n_fact >= (1ull << 32) || n_dim > (1ull << 32)) return DPG_ERR_UNSUPPORTED;
  uint64_t row, out_bytes, fact_total, dim_total;
  if (__builtin_add_overflow((uint64_t)fact_bytes, (uint64_t)rec_bytes, &row) ||
      __builtin_mul_overflow(n_fact, row, &out_bytes) ||
      __builtin_mul_overflow(n_fact, (uint64_t)fact_bytes, &fact_total) ||
      __builtin_mul_overflow(n_dim, (uint64_t)rec_bytes, &dim_total))
    return DPG_ERR_INVALID_ARG;
  if (row > UINT32_MAX / 2) return DPG_ERR_UNSUPPORTED;
  if (overlaps(out, out_bytes, fact, fact_total) || overlaps(out, out_bytes, dim, dim_total) ||
      overlaps(out, out_bytes, fk_col, n_fact * 4))
    return DPG_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* status = device_status();
  if (!status) return DPG_ERR_CUDA;
  const int sm = current_sm_count();
  // [rid_R | rid_F sorted | temporary file of fact rows]
  const uint64_t o_fk = align_up(n_fact * 4 + 16, 256);
  const uint64_t o_tmp = o_fk + align_up(n_fact * 4 + 16, 256);
  void* buf = nullptr;
  if (ws_malloc(&buf, o_tmp + n_fact * fact_bytes + 64, st) != cudaSuccess) {
    cudaGetLastError();
    return DPG_ERR_OOM;
  }
  uint32_t* rid_r = (uint32_t*)buf;
  uint32_t* fks = (uint32_t*)((uint8_t*)buf + o_fk);
  uint8_t* tmp = (uint8_t*)buf + o_tmp;
  uint32_t *gbar = nullptr, *total = nullptr;
  void* ws = nullptr;
  uint32_t nl = 0;
  dpg_status_t s = persist_ws(st, 1, sort_ws_bytes(n_fact, sm), &gbar, &total, &ws, &ws_hold);
  cudaError_t e = cudaSuccess;
  if (s == DPG_OK)
    e = launch_sort_rids(nullptr, 4, n_fact, 0, 4, (uint8_t*)ws, rid_r, gbar + 16, sm, st, &nl,
                         fk_col, fks, n_dim, status);
  if (s == DPG_OK && e == cudaSuccess) {
    // the fact rows in rid_F order: DPG retrieval (all rid_R are valid)
    s = run_dpg(fact, fact_bytes, n_fact, rid_r, n_fact, nullptr, 0, tmp, st, nullptr);
    nl += t_launches;
  }
  if (s == DPG_OK && e == cudaSuccess) {
    const uint32_t W = pow2_divisor(fact_bytes | rec_bytes | (uintptr_t)tmp | (uintptr_t)dim |
                                    (uintptr_t)out);
    e = launch_zip_gather(tmp, (uint32_t)fact_bytes, (const uint8_t*)dim, (uint32_t)rec_bytes, n_dim,
                          fks, n_fact, (uint8_t*)out, W, sm, st, &nl);
  }
  cudaFreeAsync(buf, st);
  t_launches = nl;
  return s != DPG_OK ? s : cuda_status(e);
}

dpg_status_t dpg_hash_lookup_direct(const void* table, uint32_t m_log2, const void* pool,
                                    const uint32_t* keys, uint64_t n, uint32_t* out,
                                    dpg_stream_t stream) {
  t_launches = 0;
  if (m_log2 == 0 || m_log2 > 31) return DPG_ERR_INVALID_ARG;
  if (n == 0) return DPG_OK;
  if (!table || !keys || !out) return DPG_ERR_INVALID_ARG;
  uint32_t nl = 0;
  const cudaError_t e = launch_hash_direct(table, m_log2, pool, keys, n, out, current_sm_count(),
                                           (cudaStream_t)stream, &nl);
  t_launches = nl;
  return cuda_status(e);
}

dpg_status_t dpg_hash_lookup(const void* table, uint32_t m_log2, const void* pool,
                             const uint32_t* keys, uint64_t n, uint32_t* out, dpg_stream_t stream,
                             uint32_t log2_run) {
  WsHold ws_hold;   // the stream's workspace stays ours until the launches are enqueued
  // DPG batch lookup: Phase I distributes the keys by partition
  // of the hash array, Phase II probes partition by partition with the
  // partition L2-resident, Phase III gathers the rids back into query order.
  t_launches = 0;
  if (m_log2 == 0 || m_log2 > 31) return DPG_ERR_INVALID_ARG;
  if (n == 0) return DPG_OK;
  if (!table || !keys || !out) return DPG_ERR_INVALID_ARG;
  if (n >= (1ull << 32) - 1) return DPG_ERR_UNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream;
  const int sm = current_sm_count();
  // partitions of at most one L2 run budget of slots (16 bytes each), <= 512 runs
  uint32_t s = m_log2;
  if (log2_run) {
    s = std::min<uint32_t>(log2_run, m_log2);
  } else {
    const uint64_t B1 = l2_run_budget(current_l2_bytes());
    while (s > 0 && (1ull << s) * 16 > B1) --s;
  }
  const uint32_t K = 1u << (m_log2 - s);
  if (K > 512) return DPG_ERR_UNSUPPORTED;
  // fixed run capacity: the hash spreads keys evenly (expectation + 6 sigma);
  // the keys beyond it (duplicates of hot keys) are looked up directly
  const double mean = (double)n / K;
  const uint64_t cap64 = (uint64_t)(mean + 6.0 * std::sqrt(mean) + 64);
  const uint32_t cap = (uint32_t)std::min<uint64_t>(cap64, UINT32_MAX / K);
  uint32_t *gbar = nullptr, *total = nullptr;
  void* ws = nullptr;
  const uint64_t slots = (uint64_t)K * cap;
  const uint64_t off_cur = 0;                                   // [K] cursors + overflow count
  const uint64_t off_q = align_up((K + 1) * 4, 256);
  const uint64_t off_inv = align_up(off_q + slots * 4 + 16, 256);
  const uint64_t off_tmp = align_up(off_inv + n * 4 + 16, 256);
  const uint64_t off_ovf = align_up(off_tmp + slots * 4 + 16, 256);
  const uint64_t bytes = off_ovf + n * 8 + 64;
  dpg_status_t w = persist_ws(st, 1, bytes, &gbar, &total, &ws, &ws_hold);
  if (w != DPG_OK) return w;
  uint8_t* wb = (uint8_t*)ws;
  uint32_t* cursor = (uint32_t*)(wb + off_cur);
  uint32_t* qk = (uint32_t*)(wb + off_q);
  uint32_t* inv = (uint32_t*)(wb + off_inv);
  uint32_t* tmp = (uint32_t*)(wb + off_tmp);
  uint64_t* ovf = (uint64_t*)(wb + off_ovf);
  uint32_t nl = 0;
  cudaError_t e = cudaMemsetAsync(cursor, 0, (K + 1) * 4, st);
  if (e == cudaSuccess)
    e = launch_hash_distribute(keys, n, m_log2, s, K, cap, cursor, qk, inv, ovf, cursor + K, sm, st, &nl);
  if (e == cudaSuccess)
    e = launch_hash_probe(table, m_log2, s, K, pool, qk, nullptr, tmp, gbar, sm, st, &nl, cursor, cap);
  if (e == cudaSuccess) e = launch_gather_u32(tmp, inv, n, out, sm, st, &nl);
  if (e == cudaSuccess) e = launch_hash_overflow(table, m_log2, pool, ovf, cursor + K, out, sm, st, &nl);
  t_launches = nl;
  return cuda_status(e);
}

dpg_status_t dpg_btree_lookup_direct(const uint32_t* const* levels, const uint64_t* level_n,
                                     uint32_t n_levels, const uint32_t* rids, const uint32_t* keys,
                                     uint64_t n, uint32_t* out, dpg_stream_t stream) {
  t_launches = 0;
  BTreeIdx T;
  const dpg_status_t a = btree_args(levels, level_n, n_levels, rids, &T);
  if (a != DPG_OK) return a;
  if (n == 0) return DPG_OK;
  if (!keys || !out) return DPG_ERR_INVALID_ARG;
  uint32_t nl = 0;
  const cudaError_t e = launch_bt_direct(T, keys, n, out, current_sm_count(), (cudaStream_t)stream, &nl);
  t_launches = nl;
  return cuda_status(e);
}

dpg_status_t dpg_btree_lookup(const uint32_t* const* levels, const uint64_t* level_n,
                              uint32_t n_levels, const uint32_t* rids, const uint32_t* keys,
                              uint64_t n, uint32_t* out, dpg_stream_t stream, uint32_t log2_run) {
  WsHold ws_hold;   // the stream's workspace stays ours until the launches are enqueued
  // the two-pass DPG lookup
  t_launches = 0;
  BTreeIdx T;
  const dpg_status_t a = btree_args(levels, level_n, n_levels, rids, &T);
  if (a != DPG_OK) return a;
  if (n == 0) return DPG_OK;
  if (!keys || !out) return DPG_ERR_INVALID_ARG;
  if (n >= (1ull << 32) - 1) return DPG_ERR_UNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream;
  const int sm = current_sm_count();
  const uint64_t N = level_n[0];
  // run = 2^s consecutive level-0 entries (keys + rids, 8 bytes each) within
  // one L2 run budget, rooted at a level whose entries span 16^stop <= 2^s
  uint32_t s = 0;
  while ((1ull << s) < N) ++s;
  if (log2_run) {
    s = std::min<uint32_t>(s, log2_run);
  } else {
    const uint64_t B1 = l2_run_budget(current_l2_bytes());
    while (s > 4 && (1ull << s) * 8 > B1) --s;
  }
  uint32_t stop = std::min<uint32_t>(s / 4, n_levels - 1);
  const uint32_t shift = s - 4 * stop;
  const uint64_t K64 = (N + (1ull << s) - 1) >> s;
  if (K64 > 512) return DPG_ERR_UNSUPPORTED;
  const uint32_t K = (uint32_t)std::max<uint64_t>(1, K64);
  uint32_t *gbar = nullptr, *total = nullptr;
  void* ws = nullptr;
  const uint64_t off_counts = 0;
  const uint64_t off_rs = align_up((uint64_t)K * sm * 4, 256);
  const uint64_t off_run = align_up(off_rs + (K + 1) * 4, 256);
  const uint64_t off_q = align_up(off_run + n * 4 + 16, 256);
  const uint64_t off_inv = align_up(off_q + n * 4 + 16, 256);
  const uint64_t off_tmp = align_up(off_inv + n * 4 + 16, 256);
  const uint64_t bytes = off_tmp + n * 4 + 64;
  dpg_status_t w = persist_ws(st, 1, bytes, &gbar, &total, &ws, &ws_hold);
  if (w != DPG_OK) return w;
  unsigned long long* status = device_status();
  if (!status) return DPG_ERR_CUDA;
  uint8_t* wb = (uint8_t*)ws;
  uint32_t* run = (uint32_t*)(wb + off_run);
  uint32_t* tmp = (uint32_t*)(wb + off_tmp);
  uint32_t nl = 0;
  cudaError_t e = launch_bt_top(T, stop, shift, keys, n, run, sm, st, &nl);
  L2KArgs d;
  std::memset(&d, 0, sizeof(d));
  d.rids = run;
  d.rid_bytes = 4;
  d.n_out = n;
  d.n_src = K;
  d.s = 0;
  d.K = K;
  d.chunk = align_up((n + sm - 1) / sm, 32);
  d.counts = (uint32_t*)(wb + off_counts);
  d.run_start = (uint32_t*)(wb + off_rs);
  d.local = (uint32_t*)(wb + off_q);
  d.inv = (uint32_t*)(wb + off_inv);
  d.gbar = gbar + 16;
  d.status = status;
  d.payload = keys;
  if (e == cudaSuccess) e = launch_l2k_distribute(d, (uint32_t)sm, st, &nl);
  if (e == cudaSuccess)
    e = launch_bt_probe(T, K, s, stop, d.local, d.run_start, tmp, gbar, sm, st, &nl);
  if (e == cudaSuccess) e = launch_gather_u32(tmp, d.inv, n, out, sm, st, &nl);
  t_launches = nl;
  return cuda_status(e);
}

}  // extern "C"
