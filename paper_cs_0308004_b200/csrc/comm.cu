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
#include "api_host.h"
#include "dpg_internal.cuh"

#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#ifndef DPG_NO_NCCL
#include <nccl.h>
#endif

#include "dpg.h"

namespace dpg {
namespace {

// ---- the exchange's arithmetic, shared by the NCCL path and the loopback ----
// Owner spans: rank r owns records [r S, (r+1) S), S = 2^log2_span the
// smallest power of two with P S >= n_src_total (reading A14).
uint32_t owner_log2_span(uint64_t n_src_total, int P) {
  const uint64_t per = std::max<uint64_t>(1, (n_src_total + P - 1) / P);
  uint32_t l = 0;
  while ((1ull << l) < per) ++l;
  return l;
}

// From the P x (P+1) count matrix C (row q: q's requests per owner, then q's
// row count), for rank `me`: roff[o..] = where owner `me` receives requester
// q's requests (requester-major), soff = where me's requests to owner o start
// in its owner-grouped request array, cap = the largest rank's row count (the
// window size in rows), and for every requester q the row of q's window at
// which owner `me`'s replies start (the rows q asks from owners before me).
struct ExchangePlan {
  std::vector<uint64_t> roff, soff, win_row;
  uint64_t n_req = 0, cap = 1;
};
ExchangePlan exchange_plan(const std::vector<uint64_t>& C, int P, int me) {
  auto cm = [&](int q, int o) { return C[(uint64_t)q * (P + 1) + o]; };
  ExchangePlan x;
  x.roff.assign(P + 1, 0);
  x.soff.assign(P + 1, 0);
  x.win_row.assign(P, 0);
  for (int q = 0; q < P; ++q) {
    x.roff[q + 1] = x.roff[q] + cm(q, me);
    x.soff[q + 1] = x.soff[q] + cm(me, q);
    x.cap = std::max<uint64_t>(x.cap, cm(q, P));
    uint64_t before = 0;
    for (int o = 0; o < me; ++o) before += cm(q, o);
    x.win_row[q] = before;
  }
  x.n_req = x.roff[P];
  return x;
}

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
  decltype(&ncclCommAbort) commAbort = nullptr;
  decltype(&ncclCommGetAsyncError) getAsyncError = nullptr;
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
    a.commAbort = (decltype(a.commAbort))dlsym(h, "ncclCommAbort");
    a.getAsyncError = (decltype(a.getAsyncError))dlsym(h, "ncclCommGetAsyncError");
    a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.allGather && a.allReduce &&
           a.send && a.recv && a.groupStart && a.groupEnd && a.commAbort && a.getAsyncError;
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
  bool aborted = false;                // after an NCCL failure or timeout: unusable
  std::mutex mu;
};

dpg_status_t nccl_status(ncclResult_t r) { return r == ncclSuccess ? DPG_OK : DPG_ERR_NCCL; }

// Seconds a rank waits for the stream (its collectives) before it aborts the
// communicator (DPG_NCCL_TIMEOUT_S, default 600).
double nccl_timeout_s() {
  static double t = [] {
    const char* e = getenv("DPG_NCCL_TIMEOUT_S");
    return e ? atof(e) : 600.0;
  }();
  return t;
}

// Wait for the stream while polling the communicator's asynchronous error
// state: a peer that failed or vanished surfaces as an NCCL error (or the
// timeout) instead of a hang.  On either, the communicator is aborted.
dpg_status_t wait_stream(Comm* c, cudaStream_t st) {
  const NcclApi& N = nccl();
  const auto t0 = std::chrono::steady_clock::now();
  for (uint32_t spin = 0;; ++spin) {
    const cudaError_t q = cudaStreamQuery(st);
    if (q == cudaSuccess) return DPG_OK;
    if (q != cudaErrorNotReady) {
      cudaGetLastError();
      return DPG_ERR_CUDA;
    }
    ncclResult_t ae = ncclSuccess;
    if (N.getAsyncError(c->nc, &ae) != ncclSuccess || (ae != ncclSuccess && ae != ncclInProgress)) {
      N.commAbort(c->nc);
      c->aborted = true;
      return DPG_ERR_NCCL;
    }
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > nccl_timeout_s()) {
      N.commAbort(c->nc);
      c->aborted = true;
      return DPG_ERR_NCCL;
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

// Every rank's local status, agreed on before the next collective: an
// all-reduce (min) of 1 = ok / 0 = failed, so that a rank that failed locally
// (allocation, IPC mapping, a launch) makes every rank return together
// instead of leaving its peers blocked in the next collective.
dpg_status_t agree(Comm* c, cudaStream_t st, dpg_status_t mine) {
  const NcclApi& N = nccl();
  uint64_t* w = c->scratch + 2ull * c->nranks * (c->nranks + 2);
  const uint64_t v = mine == DPG_OK ? 1 : 0;
  if (cudaMemcpyAsync(w, &v, 8, cudaMemcpyHostToDevice, st) != cudaSuccess) {
    cudaGetLastError();
  }
  if (N.allReduce(w, w, 1, ncclUint64, ncclMin, c->nc, st) != ncclSuccess) return DPG_ERR_NCCL;
  uint64_t all = 0;
  if (cudaMemcpyAsync(&all, w, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess) return DPG_ERR_CUDA;
  const dpg_status_t ws = wait_stream(c, st);
  if (ws != DPG_OK) return ws;
  if (mine != DPG_OK) return mine;
  return all ? DPG_OK : DPG_ERR_NCCL;   // a peer failed
}

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
// call it with the same bytes; a rank whose allocation fails still joins the
// handle all-gather, and the outcome is agreed on by all).
dpg_status_t ensure_windows(Comm* c, uint64_t bytes, cudaStream_t st) {
  if (c->win && c->win_bytes >= bytes) return DPG_OK;
  const NcclApi& N = nccl();
  if (cudaStreamSynchronize(st) != cudaSuccess) return DPG_ERR_CUDA;
  drop_windows(c);
  dpg_status_t mine = DPG_OK;
  cudaIpcMemHandle_t h;
  std::memset(&h, 0, sizeof(h));
  if (cudaMalloc(&c->win, bytes) != cudaSuccess) {
    cudaGetLastError();
    c->win = nullptr;
    mine = DPG_ERR_OOM;
  } else {
    c->win_bytes = bytes;
    if (cudaIpcGetMemHandle(&h, c->win) != cudaSuccess) {
      cudaGetLastError();
      mine = DPG_ERR_CUDA;
    }
  }
  uint8_t* dh = reinterpret_cast<uint8_t*>(c->scratch + 2ull * c->nranks * (c->nranks + 2) + 8);
  cudaMemcpyAsync(dh, &h, 64, cudaMemcpyHostToDevice, st);
  dpg_status_t s = nccl_status(N.allGather(dh, dh + 64, 64, ncclUint8, c->nc, st));
  std::vector<uint8_t> all(64ull * c->nranks);
  if (s == DPG_OK && cudaMemcpyAsync(all.data(), dh + 64, all.size(), cudaMemcpyDeviceToHost, st) !=
                         cudaSuccess)
    s = DPG_ERR_CUDA;
  if (s == DPG_OK) s = wait_stream(c, st);
  if (s != DPG_OK) return s;
  if (mine == DPG_OK) {
    c->peer.assign(c->nranks, nullptr);
    for (int q = 0; q < c->nranks && mine == DPG_OK; ++q) {
      if (q == c->rank) {
        c->peer[q] = c->win;
        continue;
      }
      cudaIpcMemHandle_t hq;
      std::memcpy(&hq, all.data() + 64ull * q, 64);
      void* p = nullptr;
      if (cudaIpcOpenMemHandle(&p, hq, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        mine = DPG_ERR_CUDA;
        break;
      }
      c->peer[q] = (uint8_t*)p;
    }
  }
  s = agree(c, st, mine);
  if (s != DPG_OK) drop_windows(c);
  return s;
}
#endif  // DPG_NO_NCCL

}  // namespace
}  // namespace dpg

using namespace dpg;

extern "C" {

dpg_status_t dpg_exchange_plan(const uint64_t* counts, int P, int me, uint64_t* roff,
                               uint64_t* soff, uint64_t* win_row, uint64_t* n_req,
                               uint64_t* cap) {
  if (!counts || !roff || !soff || !win_row || !n_req || !cap || P < 1 || P > 64 || me < 0 ||
      me >= P)
    return DPG_ERR_INVALID_ARG;
  const std::vector<uint64_t> C(counts, counts + (uint64_t)P * (P + 1));
  const ExchangePlan x = exchange_plan(C, P, me);
  for (int q = 0; q <= P; ++q) {
    roff[q] = x.roff[q];
    soff[q] = x.soff[q];
  }
  for (int q = 0; q < P; ++q) win_row[q] = x.win_row[q];
  *n_req = x.n_req;
  *cap = x.cap;
  return DPG_OK;
}

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
  // [counts P+1 | count matrix P(P+1) | flag | ... | agree word | IPC handles 64 (P+1)]
  if (cudaMalloc(&c->scratch, 8ull * (2ull * nranks * (nranks + 2) + 8) + 64ull * (nranks + 1) + 256) !=
      cudaSuccess) {
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
  if (c->aborted) return DPG_ERR_NCCL;
  const NcclApi& N = nccl();
  cudaStream_t st = (cudaStream_t)stream;
  const int P = c->nranks, me = c->rank;
  const uint32_t log2_span = owner_log2_span(n_src_total, P);
  const uint64_t lo = std::min<uint64_t>(n_src_total, (uint64_t)me << log2_span);
  const uint64_t n_own = std::min<uint64_t>(n_src_total, lo + (1ull << log2_span)) - lo;
  // (a rank that cannot take part still joins every collective below, with a
  // failed status that the next agreement spreads to all ranks)
  dpg_status_t mine = (n_own && !src_shard) ? DPG_ERR_INVALID_ARG : DPG_OK;

  // Phase I by owner
  uint32_t *local = nullptr, *inv = nullptr, *req = nullptr;
  uint32_t nl = 0;
  const uint64_t nb = std::max<uint64_t>(n_out_local, 1) * 4 + 64;
  uint64_t* counts = c->scratch;                  // [P+1]: my requests per owner, my row count
  uint64_t* cmat = c->scratch + (P + 1);          // [P][P+1] all ranks' rows of the above
  auto cleanup = [&]() {
    if (local) cudaFreeAsync(local, st);
    if (inv) cudaFreeAsync(inv, st);
    if (req) cudaFreeAsync(req, st);
  };
  if (mine == DPG_OK &&
      (ws_malloc(&local, nb, st) != cudaSuccess || ws_malloc(&inv, nb, st) != cudaSuccess)) {
    cudaGetLastError();
    mine = DPG_ERR_OOM;
  }
  if (mine == DPG_OK) {
    mine = dpg_partition_inv(rids, 8, n_out_local, n_src_total, log2_span, (uint32_t)P, local, inv,
                             counts, stream);
    nl += t_launches_get();
  }
  if (mine != DPG_OK) cudaMemsetAsync(counts, 0, 8ull * P, st);
  const uint64_t rows = n_out_local;
  cudaMemcpyAsync(counts + P, &rows, 8, cudaMemcpyHostToDevice, st);
  // exchange 1a: the count matrix (one all-gather), agreed
  dpg_status_t s = nccl_status(N.allGather(counts, cmat, P + 1, ncclUint64, c->nc, st));
  if (s == DPG_OK) s = agree(c, st, mine);
  std::vector<uint64_t> C((uint64_t)P * (P + 1));
  if (s == DPG_OK && cudaMemcpyAsync(C.data(), cmat, C.size() * 8, cudaMemcpyDeviceToHost, st) !=
                         cudaSuccess)
    s = DPG_ERR_CUDA;
  if (s == DPG_OK) s = wait_stream(c, st);
  if (s != DPG_OK) {
    cleanup();
    return s;
  }
  const ExchangePlan x = exchange_plan(C, P, me);
  auto cm = [&](int q, int o) { return C[(uint64_t)q * (P + 1) + o]; };
  // exchange 1b: the requests (uint32), grouped send/recv
  if (ws_malloc(&req, std::max<uint64_t>(x.n_req, 1) * 4 + 64, st) != cudaSuccess) {
    cudaGetLastError();
    mine = DPG_ERR_OOM;
  }
  s = agree(c, st, mine);
  if (s == DPG_OK) {
    N.groupStart();
    for (int q = 0; q < P; ++q) {
      if (cm(me, q)) N.send(local + x.soff[q], cm(me, q), ncclUint32, q, c->nc, st);
      if (cm(q, me)) N.recv(req + x.roff[q], cm(q, me), ncclUint32, q, c->nc, st);
    }
    s = nccl_status(N.groupEnd());
  }
  // windows of the largest rank's rows (collective; grows only)
  if (s == DPG_OK) s = ensure_windows(c, x.cap * rec_bytes, st);
  // Phase II: the owner's DPG, requester q's rows into q's window after the
  // rows q requests from owners before this one
  if (s == DPG_OK && x.n_req) {
    std::vector<uint64_t> seg_rows(P);
    std::vector<void*> seg_dst(P);
    for (int q = 0; q < P; ++q) {
      seg_rows[q] = cm(q, me);
      seg_dst[q] = c->peer[q] + x.win_row[q] * rec_bytes;
    }
    mine = dpg_retrieve_segments(src_shard, rec_bytes, n_own, req, x.n_req, (uint32_t)P,
                                 seg_rows.data(), seg_dst.data(), stream);
    nl += t_launches_get();
  }
  // every owner's writes before any requester's reads (stream-ordered), and
  // every owner's outcome agreed
  if (s == DPG_OK) s = agree(c, st, mine);
  // Phase III from the window
  if (s == DPG_OK && n_out_local) {
    s = dpg_gather_rows(c->win, rec_bytes, x.soff[P], inv, n_out_local, dst, stream);
    nl += t_launches_get();
  }
  cleanup();
  t_launches_set(nl);
  return s;
#endif
}

// Virtual ranks on one GPU: the same exchange for P logical ranks in this
// process, the NCCL steps replaced by host reads of the counts and one
// device-to-device copy per (requester, owner) pair; the plan (owner spans,
// exchange_plan offsets, window rows) and every kernel are the ones above.
dpg_status_t dpg_retrieve_dist_loopback(int P, const void* const* src_shards, size_t rec_bytes,
                                        uint64_t n_src_total, const uint64_t* const* rids,
                                        const uint64_t* n_out, void* const* dst,
                                        dpg_stream_t stream) {
  if (P <= 0 || P > kMaxSegs || !src_shards || !rids || !n_out || !dst || rec_bytes == 0 ||
      n_src_total == 0)
    return DPG_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t log2_span = owner_log2_span(n_src_total, P);
  std::vector<uint64_t> n_own(P);
  for (int r = 0; r < P; ++r) {
    const uint64_t lo = std::min<uint64_t>(n_src_total, (uint64_t)r << log2_span);
    n_own[r] = std::min<uint64_t>(n_src_total, lo + (1ull << log2_span)) - lo;
    if ((n_own[r] && !src_shards[r]) || (n_out[r] && (!rids[r] || !dst[r])))
      return DPG_ERR_INVALID_ARG;
    if (n_out[r] >= (1ull << 32) - 1) return DPG_ERR_UNSUPPORTED;
  }
  std::vector<void*> bufs;
  auto alloc = [&](uint64_t bytes) -> void* {
    void* p = nullptr;
    if (ws_malloc(&p, bytes, st) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    bufs.push_back(p);
    return p;
  };
  auto done = [&](dpg_status_t s) {
    for (void* p : bufs) cudaFreeAsync(p, st);
    return s;
  };
  uint32_t nl = 0;
  std::vector<uint32_t*> local(P), inv(P), req(P);
  std::vector<uint8_t*> win(P);
  uint64_t* counts = (uint64_t*)alloc(8ull * P * P + 64);
  if (!counts) return done(DPG_ERR_OOM);
  // Phase I by owner, every rank
  for (int r = 0; r < P; ++r) {
    const uint64_t nb = std::max<uint64_t>(n_out[r], 1) * 4 + 64;
    local[r] = (uint32_t*)alloc(nb);
    inv[r] = (uint32_t*)alloc(nb);
    if (!local[r] || !inv[r]) return done(DPG_ERR_OOM);
    dpg_status_t s = dpg_partition_inv(rids[r], 8, n_out[r], n_src_total, log2_span, (uint32_t)P,
                                       local[r], inv[r], counts + (uint64_t)r * P, stream);
    nl += t_launches_get();
    if (s != DPG_OK) return done(s);
  }
  // the count matrix (the all-gather)
  std::vector<uint64_t> cnt((uint64_t)P * P);
  if (cudaMemcpyAsync(cnt.data(), counts, cnt.size() * 8, cudaMemcpyDeviceToHost, st) !=
          cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return done(DPG_ERR_CUDA);
  std::vector<uint64_t> C((uint64_t)P * (P + 1));
  for (int q = 0; q < P; ++q) {
    for (int o = 0; o < P; ++o) C[(uint64_t)q * (P + 1) + o] = cnt[(uint64_t)q * P + o];
    C[(uint64_t)q * (P + 1) + P] = n_out[q];
  }
  auto cm = [&](int q, int o) { return C[(uint64_t)q * (P + 1) + o]; };
  std::vector<ExchangePlan> x(P);
  for (int r = 0; r < P; ++r) x[r] = exchange_plan(C, P, r);
  // the requests (the grouped send/recv): requester q's block for owner o
  for (int o = 0; o < P; ++o) {
    req[o] = (uint32_t*)alloc(std::max<uint64_t>(x[o].n_req, 1) * 4 + 64);
    if (!req[o]) return done(DPG_ERR_OOM);
  }
  for (int q = 0; q < P; ++q)
    for (int o = 0; o < P; ++o)
      if (cm(q, o) && cudaMemcpyAsync(req[o] + x[o].roff[q], local[q] + x[q].soff[o], cm(q, o) * 4,
                                      cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return done(DPG_ERR_CUDA);
  // windows
  for (int r = 0; r < P; ++r) {
    win[r] = (uint8_t*)alloc(x[r].cap * rec_bytes + 64);
    if (!win[r]) return done(DPG_ERR_OOM);
  }
  // Phase II: every owner's DPG into the requesters' windows
  for (int o = 0; o < P; ++o) {
    if (!x[o].n_req) continue;
    std::vector<uint64_t> seg_rows(P);
    std::vector<void*> seg_dst(P);
    for (int q = 0; q < P; ++q) {
      seg_rows[q] = cm(q, o);
      seg_dst[q] = win[q] + x[o].win_row[q] * rec_bytes;
    }
    dpg_status_t s = dpg_retrieve_segments(src_shards[o], rec_bytes, n_own[o], req[o], x[o].n_req,
                                           (uint32_t)P, seg_rows.data(), seg_dst.data(), stream);
    nl += t_launches_get();
    if (s != DPG_OK) return done(s);
  }
  // Phase III, every rank
  for (int r = 0; r < P; ++r) {
    if (!n_out[r]) continue;
    dpg_status_t s = dpg_gather_rows(win[r], rec_bytes, x[r].soff[P], inv[r], n_out[r], dst[r],
                                     stream);
    nl += t_launches_get();
    if (s != DPG_OK) return done(s);
  }
  t_launches_set(nl);
  return done(DPG_OK);
}

}  // extern "C"
