// comm.cu -- the multi-GPU retrieval behind the C ABI (SURVEY.md 8(b) "L3":
// dpg_get_unique_id / dpg_comm_create / dpg_retrieve_dist / dpg_comm_destroy;
// DESIGN.md section 8).  One process per GPU; NCCL (loaded at run time from
// the NCCL library the process already uses) carries the counts, the requests
// and the barriers; the records themselves go owner -> requester through
// receive windows mapped into every peer (CUDA IPC over NVLink), written by
// the owner's local DPG (dpg_retrieve_segments).  The same exchange as
// paper_cs_0308004_b200/dist.py (retrieve_dist, fused=True), native.
//
//   Phase I    dpg_partition_inv: rids (uint64) grouped by owner = rid >> log2 S
//              (S = 2^ceil(log2(ceil(n_src_total / P))) records per owner),
//              owner-local offsets and every row's request position (inv);
//   exchange 1 one all-gather of the P x P count matrix (plus every rank's
//              row count, which sizes the windows), grouped send/recv of the
//              uint32 requests;
//   Phase II   the owner's DPG over all requests it received, one output
//              segment per requester: requester q's rows land in q's window
//              at the rows q requests from owners before this one;
//   barrier    a one-word all-reduce on the stream (every owner's window
//              writes precede every requester's reads);
//   Phase III  dst[i] = window[inv[i]] (dpg_gather_rows).
#include "dpg_internal.cuh"

#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <vector>

#ifndef DPG_NO_NCCL
#include <nccl.h>
#endif

#include "dpg.h"

namespace dpg {
namespace {

#ifndef DPG_NO_NCCL
struct NcclApi {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  bool ok = false;
};

// NCCL is resolved at run time: the process's own copy if one is loaded (e.g.
// by torch), else the library the build found (DPG_NCCL_LIB).
const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
#ifdef DPG_NCCL_LIB
    if (!h) h = dlopen(DPG_NCCL_LIB, RTLD_NOW | RTLD_GLOBAL);
#endif
    if (!h) return a;
    a.getUniqueId = (decltype(a.getUniqueId))dlsym(h, "ncclGetUniqueId");
    a.commInitRank = (decltype(a.commInitRank))dlsym(h, "ncclCommInitRank");
    a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
    a.allGather = (decltype(a.allGather))dlsym(h, "ncclAllGather");
    a.allReduce = (decltype(a.allReduce))dlsym(h, "ncclAllReduce");
    a.send = (decltype(a.send))dlsym(h, "ncclSend");
    a.recv = (decltype(a.recv))dlsym(h, "ncclRecv");
    a.groupStart = (decltype(a.groupStart))dlsym(h, "ncclGroupStart");
    a.groupEnd = (decltype(a.groupEnd))dlsym(h, "ncclGroupEnd");
    a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.allGather && a.allReduce &&
           a.send && a.recv && a.groupStart && a.groupEnd;
    return a;
  }();
  return api;
}

struct Comm {
  ncclComm_t nc = nullptr;
  int nranks = 0, rank = 0, dev = 0;
  uint8_t* win = nullptr;              // this rank's receive window (IPC-exportable)
  uint64_t win_bytes = 0;
  std::vector<uint8_t*> peer;          // every rank's window as mapped here
  uint64_t* scratch = nullptr;         // device words for the small collectives
  std::mutex mu;
};

dpg_status_t nccl_status(ncclResult_t r) { return r == ncclSuccess ? DPG_OK : DPG_ERR_NCCL; }

// Close the peers' windows and free this rank's.
void drop_windows(Comm* c) {
  for (int q = 0; q < (int)c->peer.size(); ++q)
    if (q != c->rank && c->peer[q]) cudaIpcCloseMemHandle(c->peer[q]);
  c->peer.clear();
  if (c->win) cudaFree(c->win);
  c->win = nullptr;
  c->win_bytes = 0;
}

// Every rank's window of at least `bytes`, mapped here (collective: all ranks
// call it with the same bytes).
dpg_status_t ensure_windows(Comm* c, uint64_t bytes, cudaStream_t st) {
  if (c->win && c->win_bytes >= bytes) return DPG_OK;
  const NcclApi& N = nccl();
  if (cudaStreamSynchronize(st) != cudaSuccess) return DPG_ERR_CUDA;
  drop_windows(c);
  if (cudaMalloc(&c->win, bytes) != cudaSuccess) {
    cudaGetLastError();
    c->win = nullptr;
    return DPG_ERR_OOM;
  }
  c->win_bytes = bytes;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, c->win) != cudaSuccess) return DPG_ERR_CUDA;
  uint8_t* dh = nullptr;
  if (cudaMallocAsync(&dh, 64ull * (c->nranks + 1), st) != cudaSuccess) return DPG_ERR_OOM;
  cudaMemcpyAsync(dh, &h, 64, cudaMemcpyHostToDevice, st);
  dpg_status_t s = nccl_status(N.allGather(dh, dh + 64, 64, ncclUint8, c->nc, st));
  std::vector<uint8_t> all(64ull * c->nranks);
  if (s == DPG_OK && cudaMemcpyAsync(all.data(), dh + 64, all.size(), cudaMemcpyDeviceToHost, st) !=
                         cudaSuccess)
    s = DPG_ERR_CUDA;
  if (s == DPG_OK && cudaStreamSynchronize(st) != cudaSuccess) s = DPG_ERR_CUDA;
  cudaFreeAsync(dh, st);
  if (s != DPG_OK) return s;
  c->peer.assign(c->nranks, nullptr);
  for (int q = 0; q < c->nranks; ++q) {
    if (q == c->rank) {
      c->peer[q] = c->win;
      continue;
    }
    cudaIpcMemHandle_t hq;
    std::memcpy(&hq, all.data() + 64ull * q, 64);
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, hq, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      return DPG_ERR_CUDA;
    }
    c->peer[q] = (uint8_t*)p;
  }
  return DPG_OK;
}
#endif  // DPG_NO_NCCL

}  // namespace
}  // namespace dpg

using namespace dpg;

extern "C" {

dpg_status_t dpg_get_unique_id(uint8_t id[128]) {
#ifdef DPG_NO_NCCL
  (void)id;
  return DPG_ERR_NCCL;
#else
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
  if (!id) return DPG_ERR_INVALID_ARG;
  const NcclApi& N = nccl();
  if (!N.ok) return DPG_ERR_NCCL;
  ncclUniqueId u;
  dpg_status_t s = nccl_status(N.getUniqueId(&u));
  if (s == DPG_OK) std::memcpy(id, &u, 128);
  return s;
#endif
}

dpg_status_t dpg_comm_create(const uint8_t id[128], int nranks, int rank, void** comm) {
#ifdef DPG_NO_NCCL
  (void)id; (void)nranks; (void)rank; (void)comm;
  return DPG_ERR_NCCL;
#else
  if (!id || !comm || nranks <= 0 || rank < 0 || rank >= nranks || nranks > kMaxSegs)
    return DPG_ERR_INVALID_ARG;
  const NcclApi& N = nccl();
  if (!N.ok) return DPG_ERR_NCCL;
  Comm* c = new Comm();
  c->nranks = nranks;
  c->rank = rank;
  cudaGetDevice(&c->dev);
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  if (N.commInitRank(&c->nc, nranks, u, rank) != ncclSuccess) {
    delete c;
    return DPG_ERR_NCCL;
  }
  if (cudaMalloc(&c->scratch, 8ull * (nranks * nranks + 2 * nranks + 8)) != cudaSuccess) {
    cudaGetLastError();
    N.commDestroy(c->nc);
    delete c;
    return DPG_ERR_OOM;
  }
  *comm = c;
  return DPG_OK;
#endif
}

dpg_status_t dpg_comm_destroy(void* comm) {
#ifdef DPG_NO_NCCL
  (void)comm;
  return DPG_ERR_NCCL;
#else
  if (!comm) return DPG_ERR_INVALID_ARG;
  Comm* c = (Comm*)comm;
  cudaDeviceSynchronize();
  drop_windows(c);
  if (c->scratch) cudaFree(c->scratch);
  const dpg_status_t s = nccl_status(nccl().commDestroy(c->nc));
  delete c;
  return s;
#endif
}

dpg_status_t dpg_retrieve_dist(void* comm, const void* src_shard, size_t rec_bytes,
                               uint64_t n_src_total, const uint64_t* rids, uint64_t n_out_local,
                               void* dst, dpg_stream_t stream) {
#ifdef DPG_NO_NCCL
  (void)comm; (void)src_shard; (void)rec_bytes; (void)n_src_total; (void)rids;
  (void)n_out_local; (void)dst; (void)stream;
  return DPG_ERR_NCCL;
#else
  if (!comm || rec_bytes == 0 || n_src_total == 0) return DPG_ERR_INVALID_ARG;
  if (n_out_local && (!rids || !dst)) return DPG_ERR_INVALID_ARG;
  if (n_out_local >= (1ull << 32) - 1) return DPG_ERR_UNSUPPORTED;
  Comm* c = (Comm*)comm;
  std::lock_guard<std::mutex> lk(c->mu);
  const NcclApi& N = nccl();
  cudaStream_t st = (cudaStream_t)stream;
  const int P = c->nranks, me = c->rank;
  // owner spans: S = 2^ceil(log2(ceil(n_src_total / P))) records per rank
  const uint64_t per = std::max<uint64_t>(1, (n_src_total + P - 1) / P);
  uint32_t log2_span = 0;
  while ((1ull << log2_span) < per) ++log2_span;
  const uint64_t lo = std::min<uint64_t>(n_src_total, (uint64_t)me << log2_span);
  const uint64_t n_own = std::min<uint64_t>(n_src_total, lo + (1ull << log2_span)) - lo;
  if (n_own && !src_shard) return DPG_ERR_INVALID_ARG;

  // Phase I by owner
  uint32_t *local = nullptr, *inv = nullptr;
  const uint64_t nb = std::max<uint64_t>(n_out_local, 1) * 4 + 64;
  if (cudaMallocAsync(&local, nb, st) != cudaSuccess || cudaMallocAsync(&inv, nb, st) != cudaSuccess) {
    cudaGetLastError();
    return DPG_ERR_OOM;
  }
  uint64_t* counts = c->scratch;                  // [P+1]: my requests per owner, my row count
  uint64_t* cmat = c->scratch + (P + 1);          // [P][P+1] all ranks' rows of the above
  uint64_t* flag = cmat + (uint64_t)P * (P + 1);  // barrier word
  dpg_status_t s = dpg_partition_inv(rids, 8, n_out_local, n_src_total, log2_span, (uint32_t)P,
                                     local, inv, counts, stream);
  uint32_t nl = t_launches_get();
  if (s == DPG_OK) {
    const uint64_t rows = n_out_local;
    cudaMemcpyAsync(counts + P, &rows, 8, cudaMemcpyHostToDevice, st);
    s = nccl_status(N.allGather(counts, cmat, P + 1, ncclUint64, c->nc, st));
  }
  std::vector<uint64_t> C((uint64_t)P * (P + 1));
  if (s == DPG_OK && (cudaMemcpyAsync(C.data(), cmat, C.size() * 8, cudaMemcpyDeviceToHost, st) !=
                          cudaSuccess ||
                      cudaStreamSynchronize(st) != cudaSuccess))
    s = DPG_ERR_CUDA;
  auto cm = [&](int q, int o) { return C[(uint64_t)q * (P + 1) + o]; };
  // exchange 1: requests (uint32), grouped send/recv
  uint64_t n_req = 0, cap = 1;
  std::vector<uint64_t> roff(P + 1, 0), soff(P + 1, 0);
  for (int q = 0; q < P; ++q) {
    roff[q + 1] = roff[q] + cm(q, me);
    soff[q + 1] = soff[q] + cm(me, q);
    cap = std::max<uint64_t>(cap, cm(q, P));
  }
  n_req = roff[P];
  uint32_t* req = nullptr;
  if (s == DPG_OK && cudaMallocAsync(&req, std::max<uint64_t>(n_req, 1) * 4 + 64, st) != cudaSuccess) {
    cudaGetLastError();
    s = DPG_ERR_OOM;
  }
  if (s == DPG_OK) {
    N.groupStart();
    for (int q = 0; q < P; ++q) {
      if (cm(me, q)) N.send(local + soff[q], cm(me, q), ncclUint32, q, c->nc, st);
      if (cm(q, me)) N.recv(req + roff[q], cm(q, me), ncclUint32, q, c->nc, st);
    }
    s = nccl_status(N.groupEnd());
  }
  // windows of the largest rank's rows (collective; grows only)
  if (s == DPG_OK) s = ensure_windows(c, cap * rec_bytes, st);
  // Phase II: the owner's DPG, requester q's rows into q's window after the
  // rows q requests from owners before this one
  if (s == DPG_OK && n_req) {
    std::vector<uint64_t> seg_rows(P);
    std::vector<void*> seg_dst(P);
    for (int q = 0; q < P; ++q) {
      uint64_t before = 0;
      for (int o = 0; o < me; ++o) before += cm(q, o);
      seg_rows[q] = cm(q, me);
      seg_dst[q] = c->peer[q] + before * rec_bytes;
    }
    s = dpg_retrieve_segments(src_shard, rec_bytes, n_own, req, n_req, (uint32_t)P,
                              seg_rows.data(), seg_dst.data(), stream);
    nl += t_launches_get();
  }
  // every owner's writes before any requester's reads (stream-ordered)
  if (s == DPG_OK) s = nccl_status(N.allReduce(flag, flag, 1, ncclUint64, ncclSum, c->nc, st));
  // Phase III from the window
  if (s == DPG_OK && n_out_local) {
    s = dpg_gather_rows(c->win, rec_bytes, soff[P], inv, n_out_local, dst, stream);
    nl += t_launches_get();
  }
  cudaFreeAsync(local, st);
  cudaFreeAsync(inv, st);
  if (req) cudaFreeAsync(req, st);
  t_launches_set(nl);
  return s;
#endif
}

}  // extern "C"
