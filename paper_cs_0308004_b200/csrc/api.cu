// api.cu -- the C ABI of libdpg.so (include/dpg.h): argument validation,
// planning of the run length L, stream-ordered workspace, the
// retrieval plans' kernel sequences, the multi-GPU building blocks and the
// status calls.  The applications (sort, joins, lookups) are in api_apps.cu.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <vector>

#include "api_host.h"
#include "dpg_internal.cuh"

using namespace dpg;

namespace dpg {

constexpr uint32_t kSmemLimit = 232448;   // 227 KB dynamic smem per CTA (sm_100)
constexpr uint64_t kSmemPerSm = 233472;   // 228 KB per SM (each CTA also reserves 1 KB)
constexpr uint32_t kBarBytes = 128;
constexpr uint32_t kHistSmemMax = 24576;  // runs whose per-CTA histogram lives in smem

thread_local uint32_t t_launches = 0;
thread_local uint32_t t_path = 0;        // plan path of the last retrieval on this thread
thread_local const OutSegs* t_seg = nullptr;   // output segments of the current call (or none)
thread_local uint64_t* t_seq3_pairs = nullptr; // tests: path 6 Phase I pairs (dpg_distribute)
thread_local const BoundsLayout* t_bounds = nullptr;   // boundary-mode runs of the current call
unsigned long long* g_debug_ts = nullptr;   // profiling: per-CTA phase stamps (dpg_debug_phase_stamps)
uint32_t g_debug_flags = 0;                 // tuning experiments only (dpg_debug_flags)

// ---- optional phase timing (events on the call's stream) --------------------
std::mutex g_timing_mu;
bool g_timing = false;
// e0 call start, e1 end of Phase I, e3 end of Phase II (path 6 only: has3),
// e2 end of the call
struct PhaseEvents { cudaEvent_t e0, e1, e2, e3; bool has3; };
std::vector<PhaseEvents> g_pending, g_pool;

thread_local bool t_nested = false;   // inside path 7's level-2 calls: no events of their own

bool timing_begin(cudaStream_t st, PhaseEvents* pe) {
  if (!g_timing || t_nested) return false;
  std::lock_guard<std::mutex> lk(g_timing_mu);
  if (!g_pool.empty()) { *pe = g_pool.back(); g_pool.pop_back(); }
  else {
    cudaEventCreate(&pe->e0); cudaEventCreate(&pe->e1); cudaEventCreate(&pe->e2);
    cudaEventCreate(&pe->e3);
  }
  pe->has3 = false;
  cudaEventRecord(pe->e0, st);
  g_pending.push_back(*pe);
  return true;
}

// End of Phase II of a three-kernel plan (path 6): Phase II and Phase III are
// then reported separately.
void timing_phase2_end(const PhaseEvents& pe, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_timing_mu);
  cudaEventRecord(pe.e3, st);
  for (auto& q : g_pending)
    if (q.e0 == pe.e0) q.has3 = true;
}

int current_sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

// L2 capacity of the current device (bytes); 126 MB when no device is present.
uint64_t current_l2_bytes() {
  static uint64_t cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 126ull << 20;
  if (!cache[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrL2CacheSize, dev) != cudaSuccess || n <= 0)
      n = 126 << 20;
    cache[dev] = (uint64_t)n;
  }
  return cache[dev];
}

// Per-device status word + mempool setup.
unsigned long long* device_status() {
  static std::mutex mu;
  static unsigned long long* ptr[64] = {nullptr};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!ptr[dev]) {
    unsigned long long* p = nullptr;
    if (cudaMalloc(&p, sizeof(*p)) != cudaSuccess) return nullptr;
    unsigned long long init = ~0ull;
    if (cudaMemcpy(p, &init, sizeof(init), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
    ptr[dev] = p;
  }
  return ptr[dev];
}

uint32_t bit_length(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 0; }
uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

bool overlaps(const void* a, uint64_t na, const void* b, uint64_t nb) {
  if (!na || !nb) return false;
  uintptr_t a0 = (uintptr_t)a, b0 = (uintptr_t)b;
  return a0 < b0 + nb && b0 < a0 + na;
}

uint32_t pow2_divisor(uint64_t x) {  // largest power of two <= 16 dividing x
  uint32_t w = 16;
  while (w > 1 && (x % w)) w >>= 1;
  return w;
}

// Stage geometry for run length L = 2^s.
void stage_geometry(uint64_t rec, uint32_t s, uint32_t pb, uint64_t pay, uint32_t slot_pairs,
                    dpg_plan_t* p) {
  uint64_t L = 1ull << s;
  uint64_t region_cap = align_up(L * rec + 32, 16);
  uint64_t pair_cap = align_up((uint64_t)slot_pairs * pb + 32, 16);
  uint64_t pay_cap = pay ? align_up((uint64_t)slot_pairs * pay + 32, 16) : 0;
  uint64_t slot = region_cap + pair_cap + pay_cap;
  p->slot_pairs = slot_pairs;
  p->smem_bytes = (uint32_t)std::min<uint64_t>(UINT32_MAX, kBarBytes + 2 * slot);
}

// Distribute geometry: chunks of >= 2048 rids per CTA, up to 2 CTAs per SM;
// per-CTA run histogram in shared memory when K counters fit.
dpg_status_t dist_geometry(uint64_t K, uint64_t n_out, const dpg_options_t* opt, int sm,
                           dpg_plan_t* p) {
  uint64_t G = std::min<uint64_t>((uint64_t)2 * sm, std::max<uint64_t>(1, (n_out + 2047) / 2048));
  uint32_t hist_mode = opt ? opt->hist_mode : 0;
  bool smem_hist = hist_mode == 1 ? (K * 4 <= kSmemLimit)
                 : hist_mode >= 2 ? false
                                  : (K <= kHistSmemMax);
  if (hist_mode == 1 && !smem_hist) return DPG_ERR_UNSUPPORTED;
  if (!smem_hist) G = std::min<uint64_t>(G, (uint64_t)sm);
  if (opt && opt->grid_distribute) G = opt->grid_distribute;
  p->grid_distribute = (uint32_t)G;
  p->hist_in_smem = smem_hist ? 1 : 0;
  return DPG_OK;
}

// Plan for the single persistent kernel (fused.cu): S = 4 stages, each one
// run of L records plus its entries (capacity CAP = L + L/4 + 32: exact for
// permutations, Poisson slack for rids drawn with replacement, overflow list
// beyond), the counts of the CTA's own runs resident in shared memory, and the
// CTA's rid chunk cached in a stage that is not prefetched into before Phase I.
constexpr uint32_t kFusedStages = 4;
constexpr uint32_t kFusedHdr = 512;

bool plan_fused(uint64_t rec, uint64_t n_src, uint64_t n_out, uint64_t pay,
                const dpg_options_t* opt, int sm, dpg_plan_t* p) {
  if (pay || n_out == 0) return false;
  const uint64_t chunk = align_up((n_out + sm - 1) / sm, 4);
  const uint32_t pos_bits = bit_length(n_out - 1);
  const bool force8 = opt && opt->pair_bytes == 8;
  // Gather mode: rows that are whole 32-byte sectors go straight to dst;
  // rows that straddle sectors go through INTERNAL and a Phase III gather (a
  // scattered partial-sector write costs a DRAM read-modify-write on this
  // HBM): 16 Mi x 48 B 1.04 ms (path 2 took 1.69), 100 B 2.07 vs
  // 2.13 ms, 64 B stays direct-to-dst (0.92 vs 1.58 ms; profiles/r02_gather_mode.md)
  uint32_t gather = rec % 32 == 0 ? 1 : 2;
  if (opt && opt->gather) gather = opt->gather;
  auto fits = [&](uint32_t s, dpg_plan_t* q) -> bool {
    const uint64_t L = 1ull << s;
    const uint64_t K = (n_src + L - 1) >> s;
    // expected entries per run: L * n_out / n_src (exactly L for a
    // permutation); capacity = expectation + L/4 (+ 4 sigma when rids repeat)
    const double expect = (double)L * (double)n_out / (double)std::max<uint64_t>(n_src, 1);
    const uint64_t cap = align_up((uint64_t)(expect + (double)(L / 4) +
                                             (n_out > n_src ? 4.0 * std::sqrt(expect) : 0.0)) + 32, 8);
    if (K * cap >= (1ull << 32)) return false;
    const uint32_t pb = gather == 2 ? (s <= 16 && !force8 ? 2u : 4u)
                                    : ((!force8 && s + pos_bits <= 32) ? 4u : 8u);
    const uint64_t region_cap = align_up(L * rec + 32, 16);
    const uint64_t stage = align_up(region_cap + cap * pb + 32, 128);
    const uint64_t max_own = (K + sm - 1) / sm;
    const uint64_t smem = kFusedHdr + align_up(max_own * 4, 128) + kFusedStages * stage;
    if (smem > kSmemLimit) return false;
    // Phase I scratch in the stages not prefetched into: the CTA's run
    // counters (K u32), the ranks of the current tile (u16), and (preferably)
    // the tile's rids (one bulk copy, one DRAM round trip).  A tile is the
    // CTA's chunk up to 65532 rids (the 16-bit ranks' range); the
    // K-proportional work of Phase I is paid once per tile, so tiles are not
    // shrunk to fit -- rather fewer stages are prefetched, or the rids are
    // read twice from L2.
    uint64_t tile = std::min<uint64_t>(align_up(chunk, 4), 65532);
    const uint32_t max_pre = (uint32_t)std::min<uint64_t>(2, std::min<uint64_t>(K, kFusedStages - 1));
    const uint64_t kfix = align_up(K, 4) * 4 + 64;
    uint32_t npre = 0, rc_words = 0;
    bool found = false;
    for (int pre = (int)max_pre; pre >= 0 && !found; --pre)
      if (kfix + tile * 6 + 16 <= (uint64_t)(kFusedStages - pre) * stage) {
        npre = (uint32_t)pre; rc_words = (uint32_t)tile; found = true;
      }
    for (int pre = (int)max_pre; pre >= 0 && !found; --pre)
      if (kfix + tile * 2 <= (uint64_t)(kFusedStages - pre) * stage) { npre = (uint32_t)pre; found = true; }
    if (!found) {
      // many runs: smaller tiles (rids read from L2), all stages as scratch
      const uint64_t room = (uint64_t)kFusedStages * stage;
      if (kfix + 2 * 1024 > room) return false;
      tile = std::min<uint64_t>(tile, ((room - kfix) / 2) & ~3ull);
      npre = 0;
    }
    const uint32_t hwarps = 0;
    q->npre = npre;
    q->rid_cache = rc_words ? 1 : 0;
    q->hist_warps = hwarps;
    q->tile = tile;
    q->log2_run = s;
    q->run_len = L;
    q->num_runs = K;
    q->pair_bytes = pb;
    q->slot_pairs = (uint32_t)cap;
    q->smem_bytes = (uint32_t)smem;
    q->nstages = kFusedStages;
    q->stage_bytes = (uint32_t)stage;
    q->gather = gather;
    return true;
  };
  dpg_plan_t q;
  std::memset(&q, 0, sizeof(q));
  const uint32_t s_src = bit_length(std::max<uint64_t>(n_src, 1) - 1);
  int s = -1;
  if (opt && opt->log2_run) {
    if (!fits(opt->log2_run, &q)) return false;
    s = (int)opt->log2_run;
  } else {
    for (int t = (int)std::min<uint32_t>(s_src, 24); t >= 0; --t)
      if (fits((uint32_t)t, &q)) { s = t; break; }
    if (s < 0) return false;
    const uint64_t want_runs = 4ull * (uint64_t)sm;
    while (s > 0 && ((n_src + (1ull << s) - 1) >> s) < want_runs &&
           ((1ull << (s - 1)) * rec) >= 8192)
      --s;
    if (!fits((uint32_t)s, &q)) return false;
  }
  *p = q;
  p->word_bytes = pow2_divisor(rec);
  p->grid_distribute = (uint32_t)sm;
  p->grid_probe = (uint32_t)sm;
  p->hist_in_smem = 1;
  p->path = 1;
  return true;
}

// Plan for the L2-run kernel (l2run.cu): one run -- the whole source -- when
// it fits the L2 budget (the paper's run-length rule, with the L2
// as the cache), and each CTA's rid chunk fits its shared-memory buffer.

uint64_t l2_budget(uint64_t l2_bytes) {
  static uint64_t env = [] {
    const char* e = getenv("DPG_L2_BUDGET_MB");
    return e ? (uint64_t)atoll(e) << 20 : 0ull;
  }();
  // The paper's constraint (1): one data run plus a rid-run buffer fit in the
  // cache.  Budget 7/8 of the L2.  Measured on B200
  // (profiles/r01_l2_retention_ncu.txt): a 52 MB run staged by TMA stays in
  // L2 for the probe, of a 79 MB run only ~60% does (each die's half of the
  // 126 MB L2 serves its own SMs); the probe's misses then go to HBM, and the
  // single staged run still beats the shared-memory runs for 100-byte records
  // up to the budget (profiles/r01_l2run_probe.txt).
  return env ? env : l2_bytes / 8 * 7;
}

// Budget of one L2 run staged from all SMs and probed from all SMs: measured
// retention ~60 MB of the 126 MB L2 (profiles/r01_l2_retention_ncu.txt).
uint64_t l2_run_budget(uint64_t l2_bytes) {
  static uint64_t env = [] {
    const char* e = getenv("DPG_L2_RUN_MB");
    return e ? (uint64_t)atoll(e) << 20 : 0ull;
  }();
  return env ? env : l2_bytes / 16 * 7;
}

// Two L2 runs (l2pair.cu): the source is more than one run and at most two;
// rows of 4-byte words up to 116 bytes; each CTA's RID_RUN[0] buffer fits
// shared memory.
bool plan_l2pair(uint64_t rec, uint64_t n_src, uint64_t n_out, uint64_t pay, bool forced, int sm,
                 uint64_t l2_bytes, dpg_plan_t* p) {
  if (pay || n_out == 0 || rec % 4 || rec < 8 || rec > 116 || n_src < 2) return false;
  const uint64_t B1 = l2_run_budget(l2_bytes);
  uint32_t s = 0;
  while ((2ull << s) * rec <= B1 && (2ull << s) < n_src) ++s;   // largest 2^s with 2^s*rec <= B1
  const uint64_t L = 1ull << s;
  if (forced) {
    // any source: run 0 = the lower half (power of two)
    s = bit_length(n_src - 1) - 1;
  } else if (!(n_src * rec > B1 && n_src <= 2 * L)) {
    return false;
  }
  const uint64_t chunk = align_up((n_out + sm - 1) / sm, 32);
  if (l2pair_smem_bytes(chunk) > kSmemLimit) return false;
  std::memset(p, 0, sizeof(*p));
  p->path = 4;
  p->log2_run = s;
  p->run_len = 1ull << s;
  p->num_runs = (n_src + p->run_len - 1) >> s;
  p->word_bytes = 16;
  p->grid_probe = (uint32_t)sm;
  p->grid_distribute = (uint32_t)sm;
  p->tile = (uint32_t)chunk;
  p->smem_bytes = l2pair_smem_bytes(chunk);
  p->nstages = 6;
  return true;
}

// Record sizes for which the K-run L2 plan is the automatic choice over the
// shared-memory runs for sources beyond the L2 (measured).
bool l2k_auto(uint64_t rec) {
  static int env = [] {
    const char* e = getenv("DPG_L2K_AUTO");
    return e ? atoi(e) : -1;
  }();
  if (env >= 0) return env != 0;
  // measured on 16 M records (profiles/r01_sweep_c3_l2k.txt): slower than the
  // shared-memory runs at every record size (K launches of stage + probe at
  // ~36 G rows/s, then a full Phase III gather), so only on request
  (void)rec;
  return false;
}

// K L2 runs (l2k.cu): runs of L = 2^s records sized to one L2 run budget; the
// source is larger than the single-run budget.  s may be forced (tests).
bool plan_l2k(uint64_t rec, uint64_t n_src, uint64_t n_out, uint64_t pay, bool forced,
              uint32_t force_s, int sm, uint64_t l2_bytes, dpg_plan_t* p) {
  if (pay || n_out == 0 || n_src < 2) return false;
  if (!forced && n_src * rec <= l2_budget(l2_bytes)) return false;
  const uint64_t B1 = l2_run_budget(l2_bytes);
  uint32_t s = 0;
  if (force_s) {
    s = force_s;
  } else {
    while ((2ull << s) * rec <= B1 && (2ull << s) < n_src) ++s;
  }
  const uint64_t K = (n_src + (1ull << s) - 1) >> s;
  if (K < 2 || K > 512) return false;
  if (n_out >= (1ull << 32) - 1) return false;
  std::memset(p, 0, sizeof(*p));
  p->path = 5;
  p->log2_run = s;
  p->run_len = 1ull << s;
  p->num_runs = K;
  p->word_bytes = pow2_divisor(rec);
  p->grid_probe = (uint32_t)sm;
  p->grid_distribute = (uint32_t)sm;
  p->tile = (uint32_t)std::min<uint64_t>(UINT32_MAX, align_up((n_out + sm - 1) / sm, 32));
  p->smem_bytes = l2k_smem_bytes((uint32_t)K);
  return true;
}

bool plan_l2run(uint64_t rec, uint64_t n_src, uint64_t n_out, uint64_t pay, bool forced, int sm,
                uint64_t l2_bytes, dpg_plan_t* p) {
  if (pay || n_out == 0) return false;
  if (!forced && n_src * rec > l2_budget(l2_bytes)) return false;
  const uint64_t chunk = align_up((n_out + sm - 1) / sm, 32);
  std::memset(p, 0, sizeof(*p));
  p->path = 3;
  p->log2_run = bit_length(std::max<uint64_t>(n_src, 1) - 1);
  p->run_len = 1ull << p->log2_run;
  p->num_runs = 1;
  p->word_bytes = pow2_divisor(rec);
  p->grid_probe = (uint32_t)sm;
  p->grid_distribute = (uint32_t)sm;
  p->tile = (uint32_t)chunk;
  p->smem_bytes = l2run_smem_bytes(chunk);
  p->nstages = 4;
  return true;
}

// Three sequential passes over shared-memory runs (seq3.cu): runs of L = 2^s
// records, L * rec <= one stage (128 KB: one CTA per SM holds it, the next
// run is prefetched into L2 meanwhile), 16-bit local offsets (s <= 16).
// Smallest source (bytes) for which the automatic plan takes two levels.
uint64_t twolevel_min_bytes() {
  static uint64_t env = [] {
    const char* e = getenv("DPG_TWOLEVEL_MIN_MB");
    return e ? (uint64_t)atoll(e) << 20 : 0ull;
  }();
  // measured slower than the single level with clusters at every size tried
  // (profiles/r02_twolevel.md): on request only unless DPG_TWOLEVEL_MIN_MB is set
  return env ? env : ~0ull;
}

uint32_t seq3_cluster_env() {
  static uint32_t env = [] {
    const char* e = getenv("DPG_SEQ3_CLUSTER");
    return e ? (uint32_t)atoi(e) : 0u;
  }();
  return env;
}

uint64_t seq3_stage_bytes() {
  static uint64_t env = [] {
    const char* e = getenv("DPG_SEQ3_STAGE_KB");
    return e ? (uint64_t)atoll(e) << 10 : 0ull;
  }();
  return env ? env : (128ull << 10);
}

// Largest record for which the three sequential passes are the automatic plan
// beyond the L2 (measured).
uint64_t seq3_auto_max_rec() {
  static uint64_t env = [] {
    const char* e = getenv("DPG_SEQ3_MAX_REC");
    return e ? (uint64_t)atoll(e) : ~0ull;
  }();
  return env != ~0ull ? env : 32;
}

bool plan_seq3(uint64_t rec, uint64_t n_src, uint64_t n_out, uint64_t pay,
               const dpg_options_t* opt, int sm, dpg_plan_t* p) {
  if (n_out == 0 || n_src == 0 || rec % 4 || pay % 4 || rec > 16384) return false;
  if (n_out >= 0xFFFFFFFFull || n_out * ((rec + pay) / 4) >= (1ull << 32)) return false;
  const bool forced = opt && opt->path == 6;
  const uint64_t stage = std::min<uint64_t>(seq3_stage_bytes(), 128ull << 10);
  // one run = `cl` slices of Ls = 2^ls records, slice i in the shared memory
  // of CTA i of a thread-block cluster (cl = 1: one CTA)
  uint32_t cl = opt && opt->cluster ? opt->cluster : seq3_cluster_env();
  if (cl != 0 && cl != 1 && cl != 2 && cl != 4 && cl != 8) return false;
  const uint32_t lcl = cl == 8 ? 3 : cl == 4 ? 2 : cl == 2 ? 1 : 0;
  uint32_t ls = 0;
  while (ls < 16 && (2ull << ls) * rec <= stage && (1ull << ls) < n_src) ++ls;
  if (cl == 0) {
    // automatic: one CTA per run, or a cluster of 2-4 sharing the run through
    // distributed shared memory while one CTA's runs would leave pieces
    // (tile, run) of fewer than 3 entries on average -- measured: the remote
    // lookups cost more than the shorter pieces save unless the pieces are
    // that short (profiles/r02_seq3_cluster.md)
    const uint64_t T0 = std::min<uint64_t>(32768, (220ull << 10) / (rec + 2));
    cl = 1;
    // (records of <= 16 bytes; a remote lookup of a 32-byte record already
    // costs more than it saves -- DSMEM moves ~20 B per cycle per SM)
    while (rec <= 16 && cl < 4 && ((T0 * cl) << ls) < 3 * n_src && ls + (cl == 2 ? 1u : 0u) < 15)
      cl *= 2;
    // more runs than Phase I takes (8192), or pieces of under two entries
    // (one from 32-byte records on): larger runs, whatever the record
    // (2^26 x 12 / 16 / 24 B: 2143 -> 2021, 1738 -> 1701, 3301 -> 2913 us)
    auto runs = [&](uint32_t c) { return (n_src + ((uint64_t)c << ls) - 1) / ((uint64_t)c << ls); };
    const uint64_t min_piece = rec < 32 ? 2 : 1;
    while (cl < 8 && (runs(cl) > 8192 || min_piece * runs(cl) * ((n_out + T0 - 1) / T0) > n_out) &&
           ls + bit_length(cl) < 17)
      cl *= 2;
  }
  const uint32_t lc = cl == 8 ? 3 : cl == 4 ? 2 : cl == 2 ? 1 : 0;
  (void)lcl;
  uint32_t s = ls + lc;
  if (opt && opt->log2_run) {
    s = opt->log2_run;
    if (s > 16 || s < lc || (1ull << (s - lc)) * rec > (128ull << 10)) return false;
  }
  if (s > 16) return false;                         // 16-bit local offsets
  const uint64_t L = 1ull << s;
  const uint64_t Ls = L >> lc;
  const uint64_t K = (n_src + L - 1) >> s;
  if (K > 8192 || (Ls * rec) % 16) return false;   // each slice one 16-byte aligned bulk copy
  if (seq3_probe_smem(Ls * rec) > kSmemLimit) return false;
  // tile T: the Phase III buffer (two of ~100 KB, else one of ~200 KB) and the
  // Phase I tile (T rids + T offsets + 2 (K + 1) counters) both fit
  auto tile_for = [&](uint64_t bytes) {
    uint64_t T = std::min<uint64_t>(32768, bytes / (rec + 2)) & ~15ull;   // records + tinv
    while (T >= 16 && seq3_dist_smem((uint32_t)T, (uint32_t)K) > kSmemLimit) T -= 16;
    return T;
  };
  uint64_t T = tile_for(110ull << 10);
  uint32_t nbuf = 2;
  const uint32_t want_buf = opt ? opt->gather : 0;   // tuning: 1 or 2 Phase III buffers
  // (two buffers overlap Phase III's loads with its writes, but halve the
  // tile, so every piece (tile, run) of Phase II is half as long: measured,
  // two buffers pay only when pieces keep >= 8 entries on average)
  if (want_buf == 1 || (want_buf != 2 && T * L < 8 * n_src)) {
    T = tile_for(220ull << 10);
    nbuf = 1;
  }
  // Phase I occupancy: where one Phase I CTA would fill an SM's shared memory
  // (4-byte records: T rids + T offsets ~ 117 KB), a tile up to 20 % smaller
  // lets two CTAs share the SM, one's rid load overlapping the other's counting
  // (16 Mi x 4 B: Phase I 59 -> 48 us, the call 149 -> 140 us; 2^26 x 4 B:
  // 643 -> 628 us; profiles/r02_s3_p6dist.md)
  if (kSmemPerSm / (seq3_dist_smem((uint32_t)T, (uint32_t)K) + 1024) < 2) {
    uint64_t T2 = T;
    while (T2 >= 16 && 2 * (seq3_dist_smem((uint32_t)T2, (uint32_t)K) + 1024) > kSmemPerSm) T2 -= 16;
    if (T2 >= 16 && T2 * 10 >= T * 8) T = T2;
  }
  if (opt && opt->grid_distribute) T = std::max<uint64_t>(16, std::min<uint64_t>(T, opt->grid_distribute * 16ull));
  if (T < 16) return false;
  const uint64_t nsub = (n_out + T - 1) / T;
  // each piece (tile, run) should hold at least one entry on average
  if (!forced && K * nsub > n_out) return false;
  if (nsub * (K + 1) > (1ull << 31)) return false;
  const uint32_t dsm = seq3_dist_smem((uint32_t)T, (uint32_t)K);
  const uint64_t dctas = std::max<uint64_t>(1, std::min<uint64_t>(4, kSmemPerSm / (dsm + 1024)));
  std::memset(p, 0, sizeof(*p));
  p->path = 6;
  p->log2_run = s;
  p->run_len = L;
  p->num_runs = K;
  p->pair_bytes = 2;
  p->pay_bytes = (uint32_t)pay;
  p->word_bytes = pow2_divisor(rec | pay);
  p->tile = (uint32_t)T;
  p->nstages = nbuf;
  p->grid_distribute = (uint32_t)std::min<uint64_t>(nsub, dctas * (uint64_t)sm);
  p->grid_probe = (uint32_t)std::min<uint64_t>(K, (opt && opt->grid_probe) ? opt->grid_probe
                                                                           : (uint64_t)sm);
  p->hist_in_smem = 1;
  p->stage_bytes = (uint32_t)(Ls * rec);
  p->smem_bytes = seq3_probe_smem(Ls * rec);
  p->cluster = cl;
  if (cl > 1)
    p->grid_probe = (uint32_t)std::max<uint64_t>(cl, std::min<uint64_t>(K * cl, (uint64_t)sm) / cl * cl);
  return true;
}

// Two-level DPG (path 7; the paper's multi-pass DPG: "useful
// when there is a very small cache in relation to the size of main memory"):
// the rids are first distributed into super-runs of 2^s1 source records
// (<= 512 MB each, the regime where the three sequential passes win), the
// three sequential passes retrieve each super-run's records in its request
// order, and one gather puts the rows back in output order.  s1 may be forced
// (log2_run, tests).
bool plan_twolevel(uint64_t rec, uint64_t n_src, uint64_t n_out, uint64_t pay,
                   const dpg_options_t* opt, int sm, dpg_plan_t* p) {
  if (pay || n_out == 0 || n_src < 2 || rec % 4 || rec > 32) return false;
  if (n_out >= 0xFFFFFFFFull || n_src > (1ull << 32)) return false;
  uint32_t s1 = 0;
  if (opt && opt->log2_run) {
    s1 = opt->log2_run;
  } else {
    while ((2ull << s1) * rec <= (512ull << 20)) ++s1;
  }
  if (s1 > 31) return false;
  const uint64_t C = (n_src + (1ull << s1) - 1) >> s1;
  if (C < 2 || C > 512) return false;
  std::memset(p, 0, sizeof(*p));
  p->path = 7;
  p->log2_run = s1;
  p->run_len = 1ull << s1;
  p->num_runs = C;
  p->word_bytes = pow2_divisor(rec);
  p->grid_probe = (uint32_t)sm;
  p->grid_distribute = (uint32_t)sm;
  return true;
}

dpg_status_t make_plan(uint64_t rec, uint64_t n_src, uint64_t n_out, uint64_t pay,
                       const dpg_options_t* opt, int sm, dpg_plan_t* p) {
  if (rec == 0 || !p) return DPG_ERR_INVALID_ARG;
  if (n_out >= (1ull << 32) || n_src > (1ull << 32)) return DPG_ERR_UNSUPPORTED;
  std::memset(p, 0, sizeof(*p));
  if (sm <= 0) sm = 148;
  const uint32_t want_path = opt ? opt->path : 0;
  const bool overrides = opt && (opt->log2_run || opt->grid_distribute || opt->grid_probe ||
                                 opt->hist_mode || opt->gather || opt->pair_bytes);
  if (want_path == 4) {
    // two L2 runs (Fig. 1 literally at the L2 level, INTERNAL run 0): on
    // request only -- measured slower than one staged run for config 2
    // (profiles/r01_l2pair_probe.txt: 76 vs 70 us; the INTERNAL round trip
    // costs what the single run's L2 misses cost)
    if (plan_l2pair(rec, n_src, n_out, pay, true, sm, current_l2_bytes(), p)) return DPG_OK;
    return DPG_ERR_UNSUPPORTED;
  }
  // Records of <= 8 bytes in lists of >= 4 Mi rids (>= 2 Mi for 5..8-byte
  // records) take the three sequential passes even when the source fits the
  // L2 budget: the one staged L2 run re-reads lines it could not keep (16 Mi
  // x 4 B: path 6 166 us, path 3 273, the direct gather 192; 8 Mi x 8 B: 110 /
  // 150 / 85; profiles/r02_sweep_final.md; 4 Mi x 4 B: 49 / 68 / 52, 2 Mi x
  // 8 B: 36 / 41 / 23, but 2 Mi x 4 B: 47 / 39 / 30, 1 Mi x 8 B: 32 / 25 / 14,
  // profiles/r02_l2k_vs_fused.md)
  if (want_path == 0 && !overrides && rec <= 8 && n_out >= ((rec > 4 ? 2ull : 4ull) << 20) &&
      plan_seq3(rec, n_src, n_out, pay, opt, sm, p))
    return DPG_OK;
  if (want_path == 3 || (want_path == 0 && !overrides)) {
    if (plan_l2run(rec, n_src, n_out, pay, want_path == 3, sm, current_l2_bytes(), p))
      return DPG_OK;
    if (want_path == 3) return DPG_ERR_UNSUPPORTED;
  }
  if (want_path == 6) {
    if (plan_seq3(rec, n_src, n_out, pay, opt, sm, p)) return DPG_OK;
    return DPG_ERR_UNSUPPORTED;
  }
  if (want_path == 7) {
    if (plan_twolevel(rec, n_src, n_out, pay, opt, sm, p)) return DPG_OK;
    return DPG_ERR_UNSUPPORTED;
  }
  // Sources of more than 512 MB of small records: two levels (measured:
  // profiles/r02_twolevel.md)
  if (want_path == 0 && !overrides && rec <= seq3_auto_max_rec() &&
      n_src * rec > twolevel_min_bytes() && plan_twolevel(rec, n_src, n_out, pay, opt, sm, p))
    return DPG_OK;
  // Beyond the L2, records up to seq3_auto_max_rec bytes take the three
  // sequential passes (the paper's small-record case)
  if (want_path == 0 && !overrides && rec <= seq3_auto_max_rec() &&
      n_src * rec > l2_budget(current_l2_bytes()) &&
      plan_seq3(rec, n_src, n_out, pay, opt, sm, p))
    return DPG_OK;
  if (want_path == 5 || (want_path == 0 && !overrides && l2k_auto(rec))) {
    if (plan_l2k(rec, n_src, n_out, pay, want_path == 5, opt ? opt->log2_run : 0, sm,
                 current_l2_bytes(), p))
      return DPG_OK;
    if (want_path == 5) return DPG_ERR_UNSUPPORTED;
  }
  // Beyond the L2, records of 36..116 bytes in 4-byte words (a multiple of
  // 4, not of 8) run faster as K L2 runs than as the fused shared-memory runs
  // (2^24 x 100 B: 1889 vs 2093 us, 2^24 x 36 B: 921 vs 1117, 2^22 x 52 B:
  // 271 vs 338); with 8- or 16-byte words the fused kernel stays ahead
  // (2^24 x 72 B: 1549 vs 2026 us; profiles/r02_l2k_vs_fused.md)
  if (want_path == 0 && !overrides && pay == 0 && rec % 8 == 4 && rec >= 36 && rec <= 116 &&
      n_out >= n_src / 2 &&
      plan_l2k(rec, n_src, n_out, pay, false, 0, sm, current_l2_bytes(), p))
    return DPG_OK;
  // Sources of >= 6 L2s with power-of-two records of >= 128 bytes: the
  // multi-kernel runs beat the fused kernel (2^23 x 128 B: 653 vs 741 us,
  // 2^22 x 256 B: 492 vs 644; at half those sources the fused kernel is
  // ahead: 312 vs 351, 245 vs 271; profiles/r02_l2k_vs_fused.md)
  const bool big_pow2 = want_path == 0 && !overrides && pay == 0 && rec >= 128 &&
                        (rec & (rec - 1)) == 0 && n_src * rec >= 6 * current_l2_bytes();
  if (want_path != 2 && !big_pow2 &&
      !(opt && (opt->grid_distribute || opt->grid_probe || opt->hist_mode)) &&
      plan_fused(rec, n_src, n_out, pay, opt, sm, p))
    return DPG_OK;
  if (want_path == 1) return DPG_ERR_UNSUPPORTED;
  // Beyond the single fused kernel, a source of >= 8 L2s with records the
  // window gather takes runs faster as K L2-sized runs than as the
  // multi-kernel shared-memory runs (the config-5 owner shard, 2^27 x 100 B:
  // 11.4 vs 14.7 ms per 2^26 rids, profiles/r01_c5_owner_plans.txt)
  // (not for rows of whole 32-byte sectors, which path 2 writes straight to
  // their rows: 2^26 x 64 B 3.98 ms vs 6.34 ms, profiles/r02_sweep_final.md)
  if (want_path == 0 && !overrides && pay == 0 && rec % 4 == 0 && rec >= 8 && rec <= 116 &&
      rec % 32 != 0 && n_src * rec >= 8 * current_l2_bytes() &&
      plan_l2k(rec, n_src, n_out, pay, false, 0, sm, current_l2_bytes(), p))
    return DPG_OK;
  std::memset(p, 0, sizeof(*p));
  p->path = 2;
  p->nstages = 2;
  const uint64_t nsrc = std::max<uint64_t>(n_src, 1);
  const uint32_t pos_bits = bit_length(n_out > 0 ? n_out - 1 : 0);
  const bool force8 = opt && opt->pair_bytes == 8;
  auto pair_bytes_for = [&](uint32_t s) -> uint32_t {
    return (!force8 && s + pos_bits <= 32) ? 4u : 8u;
  };
  // Largest run that fits one of two shared-memory stages (paper's first
  // constraint: one run of records plus the buffer of its rids).
  uint32_t s_fit = 0;
  for (int s = 24; s >= 0; --s) {
    uint64_t L = 1ull << s;
    if (L * rec + 32 > kSmemLimit) continue;
    dpg_plan_t t;
    stage_geometry(rec, s, pair_bytes_for(s), pay, (uint32_t)std::max<uint64_t>(32, L), &t);
    if (t.smem_bytes <= kSmemLimit) { s_fit = (uint32_t)s; break; }
  }
  // No larger than the source itself, and small enough that every SM gets
  // several runs (load balance), but not below ~8 KB of records per run.
  uint32_t s_src = bit_length(nsrc - 1);
  uint32_t s = std::min(s_fit, s_src);
  uint64_t want_runs = 4ull * (uint64_t)sm;
  while (s > 0 && ((nsrc + (1ull << s) - 1) >> s) < want_runs && ((1ull << (s - 1)) * rec) >= 8192)
    --s;
  if (opt && opt->log2_run) {
    if (opt->log2_run > 31) return DPG_ERR_INVALID_ARG;
    s = opt->log2_run;
    if ((1ull << s) * rec + 32 > kSmemLimit) return DPG_ERR_UNSUPPORTED;
  }
  const uint64_t L = 1ull << s;
  const uint64_t K = (nsrc + L - 1) >> s;
  if (K >= (1ull << 31)) return DPG_ERR_UNSUPPORTED;
  // Phase I: stable radix passes over the run index (their 8-byte elements
  // carry the rid; reading A24) for large lists or when the K run counters
  // exceed shared memory, else the counting distribute with per-CTA run
  // histograms in shared memory (its fixed cost is lower: 56 vs 107 us at
  // 1 Mi rids; 560 vs 400 us at 16 Mi, profiles/r02_radix_occupancy.md)
  const uint32_t hm = opt ? opt->hist_mode : 0;
  if (hm == 3 && pay) return DPG_ERR_UNSUPPORTED;
  const bool radix = pay == 0 && (hm == 3 || (hm == 0 && (K > kHistSmemMax || n_out >= (4ull << 20))));
  const uint32_t pb = radix ? 8u : pair_bytes_for(s);
  // Pair chunk per stage: the expected rids of a run with Poisson slack (at
  // least 2L) when it fits, else 2L, 1.5L, L, ...; a heavier run is processed
  // in several chunks, each staging the run's records again.
  uint32_t sp = 0;
  const uint64_t per_run = n_out / std::max<uint64_t>(1, K);
  const uint64_t want = std::max<uint64_t>(2 * L, per_run + per_run / 4 + 64);
  for (uint64_t cand : {want, 2 * L, L + L / 2, L, L / 2, L / 4, (uint64_t)32}) {
    cand = std::max<uint64_t>(32, cand);
    dpg_plan_t t;
    stage_geometry(rec, s, pb, pay, (uint32_t)std::min<uint64_t>(cand, 1u << 24), &t);
    if (t.smem_bytes <= kSmemLimit) { sp = t.slot_pairs; break; }
  }
  if (!sp) return DPG_ERR_UNSUPPORTED;
  stage_geometry(rec, s, pb, pay, sp, p);
  p->log2_run = s;
  p->pair_bytes = pb;
  p->run_len = L;
  p->num_runs = K;
  p->word_bytes = pow2_divisor(rec | pay);
  p->pay_bytes = (uint32_t)pay;
  dpg_status_t ds = radix ? DPG_OK : dist_geometry(K, n_out, opt, sm, p);
  if (ds != DPG_OK) return ds;
  if (radix) {
    p->hist_in_smem = 0;
    p->grid_distribute = 3u * (uint32_t)sm;   // cooperative passes: up to three CTAs per SM
    p->dist_radix = radix_passes(K);
  }
  uint64_t gp = std::min<uint64_t>(K, (uint64_t)sm);
  if (opt && opt->grid_probe) gp = opt->grid_probe;
  p->grid_probe = (uint32_t)std::max<uint64_t>(1, gp);
  return DPG_OK;
}

struct Workspace {
  uint8_t* base = nullptr;
  uint32_t* counts = nullptr;
  uint32_t* run_start = nullptr;
  void* pairs = nullptr;
  uint8_t* pay = nullptr;
  // probe work items (path 2): chunk counts, scan partials, first item per run, run per item
  uint32_t *item_cnt = nullptr, *item_part = nullptr, *item_start = nullptr, *item_run = nullptr;
  uint64_t* tmp = nullptr;   // radix Phase I ping-pong buffer (n_out elements)
};

dpg_status_t alloc_workspace(const dpg_plan_t& p, uint64_t n_out, cudaStream_t st, Workspace* w) {
  const uint64_t K = p.num_runs, G = p.grid_distribute;
  const uint64_t M = p.dist_radix ? 256 * G + 256 : K * G;   // counts: per (run or digit, CTA)
  const uint64_t ntiles = (M + 4095) / 4096;
  uint64_t off_counts = 0;
  uint64_t off_rs = align_up(off_counts + M * 4, 256);
  uint64_t off_pairs = align_up(off_rs + (K + 1 + ntiles) * 4, 256);
  uint64_t off_pay = align_up(off_pairs + n_out * p.pair_bytes + 64, 256);
  uint64_t end = align_up(off_pay + (p.pay_bytes ? n_out * p.pay_bytes + 64 : 0), 256);
  uint64_t off_items = end;
  if (p.slot_pairs) {   // K chunk counts | partials | K+1 item starts | items (<= K + n_out/SP)
    const uint64_t items = K + (n_out + p.slot_pairs - 1) / p.slot_pairs + 1;
    end = align_up(off_items + align_up((K + (K + 4095) / 4096 + K + 1) * 4, 16) + items * 16, 256);
  }
  const uint64_t off_tmp = end;
  if (p.dist_radix >= 2) end = align_up(off_tmp + n_out * 8 + 64, 256);
  const uint64_t total = end;
  void* b = nullptr;
  if (ws_malloc(&b, total, st) != cudaSuccess) {
    cudaGetLastError();
    return DPG_ERR_OOM;
  }
  w->base = (uint8_t*)b;
  w->counts = (uint32_t*)(w->base + off_counts);
  w->run_start = (uint32_t*)(w->base + off_rs);
  w->pairs = w->base + off_pairs;
  w->pay = p.pay_bytes ? w->base + off_pay : nullptr;
  if (p.dist_radix >= 2) w->tmp = (uint64_t*)(w->base + off_tmp);
  if (p.slot_pairs) {
    w->item_cnt = (uint32_t*)(w->base + off_items);
    w->item_part = w->item_cnt + K;
    w->item_start = w->item_part + (K + 4095) / 4096;
    w->item_run = (uint32_t*)(w->base + off_items + align_up((K + (K + 4095) / 4096 + K + 1) * 4, 16));
  }
  return DPG_OK;
}

// Persistent per-(device, stream) workspace: [grid barrier + counters (K
// u32) | scratch].  The kernels leave the barrier and the counters zero on
// exit, so they are zeroed once, at allocation.  Each entry has its own
// (recursive) mutex, which the calling entry point holds (WsHold) from
// persist_ws until its launches are enqueued: a second host thread driving the
// same stream waits instead of freeing a base the first is about to use; a
// nested call on the same thread (dpg_sort -> run_dpg) re-enters.  At most
// kWsCached entries keep memory; the least recently used idle ones beyond
// that are freed (synchronously: their stream may be gone).
struct PersistWS {
  int dev = 0;
  cudaStream_t st = nullptr;
  uint8_t* base = nullptr;
  uint64_t counters = 0;  // bytes of the zero-invariant prefix
  uint64_t bytes = 0;
  uint64_t last_use = 0;
  std::unique_ptr<std::recursive_mutex> mu{new std::recursive_mutex};
};
constexpr size_t kWsCached = 8;
std::mutex g_ws_mu;
std::list<PersistWS> g_ws;      // entries are never erased (stable addresses)
uint64_t g_ws_clock = 0;

// Library scratch comes from a private stream-ordered pool per device (the
// process's default pool is left alone); dpg_release_cache trims it.
cudaMemPool_t ws_pool() {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!pools[dev]) {
    cudaMemPoolProps pr;
    std::memset(&pr, 0, sizeof(pr));
    pr.allocType = cudaMemAllocationTypePinned;
    pr.handleTypes = cudaMemHandleTypeNone;
    pr.location.type = cudaMemLocationTypeDevice;
    pr.location.id = dev;
    cudaMemPool_t p = nullptr;
    if (cudaMemPoolCreate(&p, &pr) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    uint64_t thr = UINT64_MAX;      // freed scratch stays reserved for the next call
    cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr);
    pools[dev] = p;
  }
  return pools[dev];
}

cudaError_t ws_malloc(void** p, size_t bytes, cudaStream_t st) {
  cudaMemPool_t pool = ws_pool();
  if (!pool) return cudaMallocAsync(p, bytes, st);
  return cudaMallocFromPoolAsync(p, bytes, pool, st);
}

void ws_pool_trim() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) { cudaGetLastError(); return; }
  int cur = 0;
  cudaGetDevice(&cur);
  for (int d = 0; d < n && d < 64; ++d) {
    cudaSetDevice(d);
    if (cudaMemPool_t p = ws_pool()) {
      cudaDeviceSynchronize();
      cudaMemPoolTrimTo(p, 0);
    }
  }
  cudaSetDevice(cur);
  cudaGetLastError();
}

dpg_status_t persist_ws(cudaStream_t st, uint64_t K, uint64_t pair_bytes_total, uint32_t** gbar,
                        uint32_t** total, void** pairs, WsHold* hold) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return DPG_ERR_CUDA;
  const uint64_t need_ctr = align_up(256 + K * 4, 256);
  const uint64_t need = need_ctr + align_up(pair_bytes_total + 64, 256);
  PersistWS* w = nullptr;
  std::vector<PersistWS*> evict;
  {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    for (auto& kv : g_ws)
      if (kv.dev == dev && kv.st == st) w = &kv;
    if (!w) {
      g_ws.emplace_back();
      w = &g_ws.back();
      w->dev = dev;
      w->st = st;
    }
    w->last_use = ++g_ws_clock;
    std::vector<PersistWS*> live;
    for (auto& kv : g_ws)
      if (kv.base && &kv != w) live.push_back(&kv);
    if (live.size() + 1 > kWsCached) {
      std::sort(live.begin(), live.end(),
                [](PersistWS* x, PersistWS* y) { return x->last_use < y->last_use; });
      evict.assign(live.begin(), live.begin() + (live.size() + 1 - kWsCached));
    }
  }
  for (PersistWS* v : evict) {           // idle least recently used entries
    std::unique_lock<std::recursive_mutex> vl(*v->mu, std::try_to_lock);
    if (!vl.owns_lock() || !v->base) continue;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(v->dev);
    cudaFree(v->base);                   // synchronous: its stream may be destroyed
    cudaSetDevice(cur);
    cudaGetLastError();
    v->base = nullptr;
    v->bytes = v->counters = 0;
  }
  *hold = WsHold(*w->mu);                // held until the caller's launches are enqueued
  const uint64_t need_pairs = need - need_ctr;
  const uint64_t have_pairs = w->bytes - w->counters;
  if (w->counters < need_ctr || have_pairs < need_pairs) {
    const uint64_t ctr = std::max(need_ctr, w->counters);
    const uint64_t bytes = ctr + std::max(need_pairs, have_pairs);
    if (w->base) cudaFreeAsync(w->base, st);
    w->base = nullptr;
    w->bytes = w->counters = 0;
    void* b = nullptr;
    if (ws_malloc(&b, bytes, st) != cudaSuccess) {
      cudaGetLastError();
      return DPG_ERR_OOM;
    }
    if (cudaMemsetAsync(b, 0, ctr, st) != cudaSuccess) return DPG_ERR_CUDA;
    w->base = (uint8_t*)b;
    w->counters = ctr;
    w->bytes = bytes;
  }
  *gbar = (uint32_t*)w->base;
  *total = (uint32_t*)(w->base + 256);
  *pairs = w->base + w->counters;
  return DPG_OK;
}

void release_persist_ws() {
  std::vector<PersistWS*> all;
  {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    for (auto& kv : g_ws) all.push_back(&kv);
  }
  int cur = 0;
  cudaGetDevice(&cur);
  for (PersistWS* v : all) {
    std::lock_guard<std::recursive_mutex> vl(*v->mu);
    if (!v->base) continue;
    cudaSetDevice(v->dev);
    cudaFree(v->base);                   // synchronous: the stream may be destroyed
    v->base = nullptr;
    v->bytes = v->counters = 0;
  }
  cudaSetDevice(cur);
  cudaGetLastError();
}

dpg_status_t cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return DPG_OK;
  cudaGetLastError();
  return e == cudaErrorMemoryAllocation ? DPG_ERR_OOM : DPG_ERR_CUDA;
}

// Shared body of dpg_retrieve and dpg_fk_join: rows of (pay ++ rec) bytes.
constexpr uint64_t kSkewMinRids = 1ull << 22;   // sample inputs from 4 Mi rids on
constexpr uint32_t kSkewSamples = 65536;

// Estimated rids beyond the fixed run capacity of plan p (skew.cu): S sampled
// rids counted per group of runs on the device, the estimate read back (one
// stream synchronisation).
dpg_status_t skew_excess(const uint32_t* rids, uint64_t n_out, uint64_t n_src, const dpg_plan_t& p,
                         cudaStream_t st, uint64_t* excess, uint32_t* nl) {
  static std::mutex mu;
  static std::vector<std::pair<int, uint8_t*>> bufs;     // per device: [result | hist]
  static unsigned long long* host = nullptr;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return DPG_ERR_CUDA;
  std::lock_guard<std::mutex> lk(mu);
  uint8_t* b = nullptr;
  for (auto& kv : bufs)
    if (kv.first == dev) b = kv.second;
  const uint64_t words = kSkewSamples / 64 + 2;           // groups of >= 64 expected samples
  if (!b) {
    if (cudaMalloc(&b, 256 + words * 4) != cudaSuccess) { cudaGetLastError(); return DPG_ERR_OOM; }
    if (cudaMemset(b, 0, 256 + words * 4) != cudaSuccess) return DPG_ERR_CUDA;
    bufs.push_back({dev, b});
  }
  if (!host && cudaMallocHost(&host, sizeof(*host)) != cudaSuccess) {
    cudaGetLastError();
    return DPG_ERR_OOM;
  }
  cudaError_t e = launch_skew_check(rids, n_out, n_src, p.log2_run, (uint32_t)p.num_runs,
                                    p.slot_pairs, kSkewSamples, (uint32_t*)(b + 256),
                                    (unsigned long long*)b, st, nl);
  if (e == cudaSuccess) e = cudaMemcpyAsync(host, b, sizeof(*host), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_status(e);
  *excess = *host;
  return DPG_OK;
}

dpg_status_t run_dpg(const void* src, uint64_t rec, uint64_t n_src, const uint32_t* rids,
                     uint64_t n_out, const void* pay_src, uint64_t pay, void* dst,
                     cudaStream_t st, const dpg_options_t* opt) {
  WsHold ws_hold;   // the stream's workspace stays ours until the launches are enqueued
  t_launches = 0;
  if (rec == 0) return DPG_ERR_INVALID_ARG;
  if (n_out == 0) return DPG_OK;
  if (!src || !rids || !dst || (pay && !pay_src)) return DPG_ERR_INVALID_ARG;
  if (n_src == 0) return DPG_ERR_INVALID_ARG;
  if (n_out >= (1ull << 32) || n_src > (1ull << 32)) return DPG_ERR_UNSUPPORTED;
  uint64_t src_bytes, row, dst_bytes, pay_bytes_total;
  if (__builtin_mul_overflow(n_src, rec, &src_bytes)) return DPG_ERR_INVALID_ARG;
  if (__builtin_add_overflow(rec, pay, &row)) return DPG_ERR_INVALID_ARG;
  if (__builtin_mul_overflow(n_out, row, &dst_bytes)) return DPG_ERR_INVALID_ARG;
  if (__builtin_mul_overflow(n_out, pay, &pay_bytes_total)) return DPG_ERR_INVALID_ARG;
  if (rec > UINT32_MAX / 2 || row > UINT32_MAX / 2) return DPG_ERR_UNSUPPORTED;
  if (!t_seg &&   // (segmented output: each segment was checked by dpg_retrieve_segments)
      (overlaps(dst, dst_bytes, src, src_bytes) || overlaps(dst, dst_bytes, rids, n_out * 4) ||
       (pay && overlaps(dst, dst_bytes, pay_src, pay_bytes_total))))
    return DPG_ERR_INVALID_ARG;

  const int sm = current_sm_count();
  dpg_plan_t p;
  dpg_status_t ps = make_plan(rec, n_src, n_out, pay, opt, sm, &p);
  if (ps == DPG_ERR_UNSUPPORTED && pay == 0 && !(opt && opt->log2_run) &&
      rec * 2 + 64 > kSmemLimit / 2) {
    // A record larger than a shared-memory stage is itself one sequential
    // stream; DPG's run staging has nothing left to win, so such
    // records take the direct path.
    return dpg_retrieve_direct(src, rec, n_src, rids, n_out, dst, (dpg_stream_t)st);
  }
  if (ps != DPG_OK) return ps;
  if (t_bounds) {
    // runs from boundaries (dpg_retrieve_bounds): the multi-kernel plan over
    // the merged layout's K runs
    if (p.path != 2) return DPG_ERR_UNSUPPORTED;
    p.num_runs = t_bounds->K;
    p.dist_radix = 0;
    dpg_status_t gs = dist_geometry(p.num_runs, n_out, opt, sm, &p);
    if (gs != DPG_OK) return gs;
  }
  unsigned long long* status = device_status();
  if (!status) return DPG_ERR_CUDA;
  uint32_t nl_skew = 0;
  bool seg_nostage = false;   // a segmented call re-planned onto path 3 past the L2 budget
  {
    // Data skew (section 2.3): a large input planned on fixed
    // shared-memory runs is sampled first; a rid list that would overflow the
    // runs' capacity takes the multi-kernel plan instead (exact run sizes from
    // the count, heavy runs split into work items over all CTAs).
    const bool auto_plan = !opt || (opt->path == 0 && !opt->log2_run && !opt->grid_distribute &&
                                    !opt->grid_probe && !opt->hist_mode && !opt->gather &&
                                    !opt->pair_bytes);
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cap);      // (a graph capture cannot synchronise: no sampling)
    if (auto_plan && p.path == 1 && pay == 0 && n_out >= kSkewMinRids && !(g_debug_flags & 64) &&
        cap == cudaStreamCaptureStatusNone) {
      uint64_t excess = 0;
      dpg_status_t ks = skew_excess(rids, n_out, n_src, p, st, &excess, &nl_skew);
      if (ks != DPG_OK) return ks;
      dpg_plan_t q;
      dpg_options_t o2;
      std::memset(&o2, 0, sizeof(o2));
      o2.path = 2;
      if (excess > n_out / 50 && make_plan(rec, n_src, n_out, pay, &o2, sm, &q) == DPG_OK) p = q;
    }
  }
  if (t_seg) {
    // output segments: every plan whose last writer can address rows anywhere
    // (the fused probe in mode 0, the multi-kernel probe, the window gather);
    // the others are re-planned onto one of those
    const OutSegs& sg = *t_seg;
    bool al4 = true;
    for (uint32_t q = 0; q < sg.n; ++q) al4 = al4 && ((uintptr_t)sg.out[q] % 4 == 0);
    const bool agr_ok = rec % 4 == 0 && rec >= 8 && rec <= 116 && al4 && (uintptr_t)src % 4 == 0;
    if (p.path == 1 && pay == 0) {
      if (p.gather != 1) {
        // the fused probe writes segment rows only in its direct-to-dst mode
        dpg_options_t o;
        if (opt) o = *opt; else std::memset(&o, 0, sizeof(o));
        o.path = 1;
        o.gather = 1;
        dpg_plan_t q;
        if (make_plan(rec, n_src, n_out, 0, &o, sm, &q) == DPG_OK) {
          p = q;
        } else {
          o.path = 2;
          o.gather = 0;
          if (make_plan(rec, n_src, n_out, 0, &o, sm, &p) != DPG_OK) return DPG_ERR_UNSUPPORTED;
        }
      }
    } else if (p.path == 2 && pay == 0) {
    } else if (p.path == 5 && agr_ok) {
    } else if (agr_ok && n_src * rec <= ((uint64_t)1 << 32)) {
      dpg_options_t o{};
      o.path = 3;
      if (make_plan(rec, n_src, n_out, 0, &o, sm, &p) != DPG_OK) return DPG_ERR_UNSUPPORTED;
      if (p.path == 3 && n_src * rec > l2_budget(current_l2_bytes())) seg_nostage = true;
    } else if (dpg_plan_t q; pay == 0 && [&] {
                 // the shared-memory runs, which write rows anywhere: fused, else multi-kernel
                 dpg_options_t o{};
                 o.path = 1;
                 o.gather = 1;
                 if (make_plan(rec, n_src, n_out, 0, &o, sm, &q) == DPG_OK) return true;
                 o.path = 2;
                 return make_plan(rec, n_src, n_out, 0, &o, sm, &q) == DPG_OK;
               }()) {
      p = q;
    } else {
      // a record no DPG plan can write to segments: the direct gather, one launch per segment
      uint32_t nl = 0;
      for (uint32_t q = 0; q < sg.n; ++q) {
        const uint64_t k0 = sg.start[q], k1 = sg.start[q + 1];
        if (k1 == k0) continue;
        dpg_status_t ds = dpg_retrieve_direct(src, rec, n_src, rids + k0, k1 - k0, sg.out[q],
                                              (dpg_stream_t)st);
        nl += t_launches;
        if (ds != DPG_OK) return ds;
      }
      t_path = 0;
      t_launches = nl + nl_skew;
      return DPG_OK;
    }
  }
  t_path = p.path;

  if (p.path == 7) {
    // level 1: the rids by super-run (rid >> s1), every row's slot (inv)
    const uint32_t s1 = p.log2_run, C = (uint32_t)p.num_runs;
    uint32_t *local = nullptr, *inv = nullptr;
    uint64_t* counts = nullptr;
    uint8_t* internal = nullptr;
    auto fail = [&](dpg_status_t r) {
      if (local) cudaFreeAsync(local, st);
      if (inv) cudaFreeAsync(inv, st);
      if (counts) cudaFreeAsync(counts, st);
      if (internal) cudaFreeAsync(internal, st);
      return r;
    };
    if (ws_malloc(&local, n_out * 4 + 64, st) != cudaSuccess ||
        ws_malloc(&inv, n_out * 4 + 64, st) != cudaSuccess ||
        ws_malloc(&counts, (uint64_t)C * 8 + 64, st) != cudaSuccess ||
        ws_malloc(&internal, n_out * rec + 64, st) != cudaSuccess) {
      cudaGetLastError();
      return fail(DPG_ERR_OOM);
    }
    PhaseEvents pe;
    const bool timed = timing_begin(st, &pe);
    dpg_status_t r = dpg_partition_inv(rids, 4, n_out, n_src, s1, C, local, inv, counts,
                                       (dpg_stream_t)st);
    uint32_t nl = t_launches;
    if (timed) cudaEventRecord(pe.e1, st);
    std::vector<uint64_t> cnt(C);
    if (r == DPG_OK &&
        (cudaMemcpyAsync(cnt.data(), counts, (uint64_t)C * 8, cudaMemcpyDeviceToHost, st) !=
             cudaSuccess ||
         cudaStreamSynchronize(st) != cudaSuccess))
      r = DPG_ERR_CUDA;
    // level 2: every super-run's records in its request order (its own plan:
    // the three sequential passes, or one L2 run for a small last super-run)
    uint64_t start = 0;
    for (uint32_t c = 0; c < C && r == DPG_OK; ++c) {
      const uint64_t lo = (uint64_t)c << s1;
      const uint64_t n_c = std::min<uint64_t>(1ull << s1, n_src - lo);
      t_nested = true;
      if (cnt[c])
        r = run_dpg((const uint8_t*)src + lo * rec, rec, n_c, local + start, cnt[c], nullptr, 0,
                    internal + start * rec, st, nullptr);
      t_nested = false;
      nl += t_launches;
      start += cnt[c];
    }
    if (timed) timing_phase2_end(pe, st);
    // level-1 Phase III: dst[i] = INTERNAL[inv[i]] in output order (C streams)
    if (r == DPG_OK)
      r = cuda_status(launch_direct(internal, start, (uint32_t)rec, inv, n_out, (uint8_t*)dst,
                                    pow2_divisor(rec | (uintptr_t)dst), sm, nullptr, st, &nl));
    if (timed) cudaEventRecord(pe.e2, st);
    t_path = 7;
    t_launches = nl + nl_skew;
    fail(DPG_OK);
    return r;
  }
  if (p.path == 6 && ((uintptr_t)src % 16 != 0)) {
    // the stage is one TMA bulk copy of the run: an unaligned source takes the
    // multi-kernel shared-memory runs
    if (opt && opt->path == 6) return DPG_ERR_UNSUPPORTED;
    dpg_options_t o{};
    o.path = 2;
    if (make_plan(rec, n_src, n_out, pay, &o, sm, &p) != DPG_OK) return DPG_ERR_UNSUPPORTED;
    t_path = p.path;
  }
  if (p.path == 6) {
    const uint64_t K = p.num_runs, T = p.tile;
    const uint64_t nsub = (n_out + T - 1) / T;
    uint32_t *gbar = nullptr, *total = nullptr;
    void* ws = nullptr;
    const uint64_t off_pre = 0;
    const uint64_t off_preT = align_up(off_pre + nsub * (K + 1) * 2, 256);
    const uint64_t off_loc = align_up(off_preT + nsub * (K + 1) * 2, 256);
    const uint64_t off_tinv = align_up(off_loc + nsub * T * 2, 256);
    const uint64_t off_int = align_up(off_tinv + nsub * T * 2 + 16, 256);
    const uint64_t bytes = off_int + nsub * T * rec + 64;
    dpg_status_t wst = persist_ws(st, 1, bytes, &gbar, &total, &ws, &ws_hold);
    if (wst != DPG_OK) return wst;
    uint8_t* wb = (uint8_t*)ws;
    Seq3Args a;
    std::memset(&a, 0, sizeof(a));
    a.src = (const uint8_t*)src;
    a.n_src = n_src;
    a.rec = (uint32_t)rec;
    a.rids = rids;
    a.n_out = n_out;
    a.s = p.log2_run;
    a.K = (uint32_t)K;
    a.T = (uint32_t)T;
    a.nsub = (uint32_t)nsub;
    a.pre = (uint16_t*)(wb + off_pre);
    a.preT = (uint16_t*)(wb + off_preT);
    a.loc = (uint16_t*)(wb + off_loc);
    a.tinv = (uint16_t*)(wb + off_tinv);
    a.dbg_pairs = t_seq3_pairs;
    a.internal = wb + off_int;
    a.dst = (uint8_t*)dst;
    a.pay = (const uint8_t*)pay_src;
    a.pay_bytes = (uint32_t)pay;
    a.status = status;
    a.dbg = g_debug_flags;
    a.ts = g_debug_ts;
    a.cl = p.cluster ? p.cluster : 1;
    uint32_t nl = 0;
    PhaseEvents pe;
    const bool timed = timing_begin(st, &pe);
    cudaError_t e = launch_seq3_distribute(a, p.grid_distribute, st, &nl);
    if (timed) cudaEventRecord(pe.e1, st);
    if (e == cudaSuccess)
      e = launch_seq3_probe(a, pow2_divisor(rec), p.grid_probe, st, &nl);
    if (timed) timing_phase2_end(pe, st);
    if (e == cudaSuccess)
      e = launch_seq3_gather(a, pow2_divisor(rec | pay | (uintptr_t)dst |
                                             (pay ? (uintptr_t)pay_src : 0)),
                             (uint32_t)std::min<uint64_t>(nsub, sm), p.nstages, st, &nl);
    if (timed) cudaEventRecord(pe.e2, st);
    t_launches = nl + nl_skew;
    return cuda_status(e);
  }
  if (p.path == 5) {
    const uint32_t G = p.grid_probe, K = (uint32_t)p.num_runs;
    const uint64_t L = p.run_len;
    uint32_t *gbar = nullptr, *total = nullptr;
    void* ws = nullptr;
    const uint64_t off_counts = 0;
    const uint64_t off_rs = align_up(off_counts + (uint64_t)K * G * 4, 256);
    const uint64_t off_local = align_up(off_rs + (K + 1) * 4, 256);
    const uint64_t off_inv = align_up(off_local + n_out * 4 + 16, 256);
    const uint64_t off_int = align_up(off_inv + n_out * 4 + 16, 256);
    const uint64_t bytes = off_int + n_out * rec + 64;
    dpg_status_t wst = persist_ws(st, 1, bytes, &gbar, &total, &ws, &ws_hold);
    if (wst != DPG_OK) return wst;
    uint8_t* wb = (uint8_t*)ws;
    L2KArgs d;
    std::memset(&d, 0, sizeof(d));
    d.rids = rids;
    d.rid_bytes = 4;
    d.n_out = n_out;
    d.n_src = n_src;
    d.s = p.log2_run;
    d.K = K;
    d.chunk = p.tile;
    d.counts = (uint32_t*)(wb + off_counts);
    d.run_start = (uint32_t*)(wb + off_rs);
    d.local = (uint32_t*)(wb + off_local);
    d.inv = (uint32_t*)(wb + off_inv);
    d.gbar = gbar + 16;
    d.status = status;
    uint8_t* internal = wb + off_int;
    uint32_t nl = 0;
    PhaseEvents pe;
    const bool timed = timing_begin(st, &pe);
    cudaError_t e = launch_l2k_distribute(d, G, st, &nl);
    if (timed) cudaEventRecord(pe.e1, st);
    for (uint32_t b = 0; b < K && e == cudaSuccess; ++b) {
      // Phase II of run b: stage it into L2, probe its RID_RUN into INTERNAL
      L2RunArgs l;
      std::memset(&l, 0, sizeof(l));
      l.src = (const uint8_t*)src + (uint64_t)b * L * rec;
      l.n_src = std::min<uint64_t>(L, n_src - (uint64_t)b * L);
      l.rec = (uint32_t)rec;
      l.rids = d.local;
      l.n_out = n_out;                       // replaced on the device by the run's range
      l.chunk = p.tile;
      l.dev_range = d.run_start + b;
      l.dst = internal;
      l.gbar = gbar;
      l.stage = 1;
      l.dbg = g_debug_flags & ~4u;
      l.ts = nullptr;
      if (rec % 4 == 0) l.rd_magic = (uint32_t)(((1ull << 32) + rec / 4 - 1) / (rec / 4));
      const uint32_t W = pow2_divisor(rec | (uintptr_t)l.src | (uintptr_t)internal);
      e = launch_l2run(l, W, G, st, &nl);
    }
    if (e == cudaSuccess) {
      // Phase III: dst[i] = INTERNAL[inv[i]] in output order
      L2RunArgs l;
      std::memset(&l, 0, sizeof(l));
      l.src = internal;
      l.n_src = n_out;
      l.rec = (uint32_t)rec;
      l.rids = d.inv;
      l.n_out = n_out;
      l.chunk = p.tile;
      l.dst = (uint8_t*)dst;
      l.gbar = gbar;
      l.stage = 0;
      if (t_seg) {
        l.seg = *t_seg;
        l.dst = t_seg->out[0];
      }
      if (rec % 4 == 0) l.rd_magic = (uint32_t)(((1ull << 32) + rec / 4 - 1) / (rec / 4));
      const uint32_t W = t_seg ? 4u : pow2_divisor(rec | (uintptr_t)internal | (uintptr_t)dst);
      e = launch_l2run(l, W, G, st, &nl);
    }
    if (timed) cudaEventRecord(pe.e2, st);
    t_launches = nl + nl_skew;
    return cuda_status(e);
  }
  if (p.path == 4 && ((uintptr_t)src % 16 || (uintptr_t)dst % 16)) {
    // the two-run kernels move 16-byte words: unaligned buffers take one run
    dpg_options_t o = opt ? *opt : dpg_options_t{};
    o.path = 3;
    if (make_plan(rec, n_src, n_out, pay, &o, sm, &p) != DPG_OK) return DPG_ERR_UNSUPPORTED;
  }
  if (p.path == 4) {
    uint32_t *gbar = nullptr, *total = nullptr;
    void* internal = nullptr;
    const uint64_t int_bytes = (uint64_t)p.grid_probe * p.tile * rec;
    dpg_status_t ws = persist_ws(st, 1, int_bytes + 64, &gbar, &total, &internal, &ws_hold);
    if (ws != DPG_OK) return ws;
    L2PairArgs l;
    std::memset(&l, 0, sizeof(l));
    l.src = (const uint8_t*)src;
    l.n_src = n_src;
    l.rec = (uint32_t)rec;
    l.rids = rids;
    l.n_out = n_out;
    l.L = p.run_len;
    l.chunk = p.tile;
    l.max_groups = (uint32_t)((p.tile + 31) / 32);
    l.internal = (uint8_t*)internal;
    l.dst = (uint8_t*)dst;
    l.gbar = gbar;
    l.status = status;
    l.ts = g_debug_ts;
    l.dbg = g_debug_flags;
    uint32_t nl = 0;
    PhaseEvents pe;
    const bool timed = timing_begin(st, &pe);
    if (timed) cudaEventRecord(pe.e1, st);
    cudaError_t e = launch_l2pair(l, p.grid_probe, st, &nl);
    if (timed) cudaEventRecord(pe.e2, st);
    t_launches = nl + nl_skew;
    return cuda_status(e);
  }
  if (p.path == 3) {
    uint32_t *gbar = nullptr, *total = nullptr;
    void* pairs = nullptr;
    dpg_status_t ws = persist_ws(st, 1, 64, &gbar, &total, &pairs, &ws_hold);
    if (ws != DPG_OK) return ws;
    L2RunArgs l;
    std::memset(&l, 0, sizeof(l));
    l.src = (const uint8_t*)src;
    l.n_src = n_src;
    l.rec = (uint32_t)rec;
    l.rids = rids;
    l.n_out = n_out;
    l.chunk = p.tile;
    l.dst = (uint8_t*)dst;
    l.gbar = gbar;
    l.status = status;
    l.ts = g_debug_ts;
    l.dbg = g_debug_flags;
    l.stage = (l.dbg & 4) ? 0 : 1;   // tuning flag: probe without staging
    if (rec % 4 == 0) l.rd_magic = (uint32_t)(((1ull << 32) + rec / 4 - 1) / (rec / 4));
    if (l.dbg >> 24) l.stage_bytes = (uint64_t)(l.dbg >> 24) << 20;   // tuning: MB staged
    if ((l.dbg >> 8) & 15) l.ring_chunk = 1024u << ((l.dbg >> 8) & 15);   // tuning: 2^k KB
    if ((l.dbg >> 12) & 15) l.ring_slots = (l.dbg >> 12) & 15;
    uint32_t W = pow2_divisor(rec | (uintptr_t)src | (uintptr_t)dst);
    if (t_seg) {
      // segmented output: the window gather (REALIGN 1) with the segments
      l.seg = *t_seg;
      l.dst = t_seg->out[0];
      W = 4;
      if (seg_nostage) l.stage = 0;   // a source beyond the L2 budget: no Phase II
    }
    uint32_t nl = 0;
    PhaseEvents pe;
    const bool timed = timing_begin(st, &pe);
    if (timed) cudaEventRecord(pe.e1, st);   // Phase I is empty (one run)
    cudaError_t e = launch_l2run(l, W, p.grid_probe, st, &nl);
    if (timed) cudaEventRecord(pe.e2, st);
    t_launches = nl + nl_skew;
    return cuda_status(e);
  }

  if (p.path == 1) {
    FusedArgs f;
    std::memset(&f, 0, sizeof(f));
    uint32_t *gbar = nullptr, *total = nullptr;
    void* pairs = nullptr;
    // [pairs | inv | INTERNAL] (the last two only in gather mode 2)
    // [pairs (K*CAP entries) | overflow list | inv | INTERNAL] (the last two
    // only in gather mode 2)
    const uint64_t slots = p.num_runs * (uint64_t)p.slot_pairs;
    const uint64_t pairs_sz = align_up(slots * p.pair_bytes + 64, 256);
    const uint64_t ovf_sz = align_up(n_out * 8, 256);
    const uint64_t inv_sz = p.gather == 2 ? align_up(n_out * 4, 256) : 0;
    const uint64_t int_sz = p.gather == 2 ? align_up(slots * rec + 64, 256) : 0;
    dpg_status_t ws = persist_ws(st, p.num_runs, pairs_sz + ovf_sz + inv_sz + int_sz, &gbar,
                                 &total, &pairs, &ws_hold);
    if (ws != DPG_OK) return ws;
    f.mode = p.gather == 2 ? 1 : 0;
    if (f.mode == 1) {
      f.inv = (uint32_t*)((uint8_t*)pairs + pairs_sz + ovf_sz);
      f.internal = (uint8_t*)pairs + pairs_sz + ovf_sz + inv_sz;
    }
    f.src = (const uint8_t*)src;
    f.n_src = n_src;
    f.rec = (uint32_t)rec;
    f.s = p.log2_run;
    f.K = (uint32_t)p.num_runs;
    f.nstages = p.nstages;
    f.rids = rids;
    f.n_out = n_out;
    f.chunk = align_up((n_out + p.grid_distribute - 1) / p.grid_distribute, 4);
    f.total = total;
    f.gbar = gbar;
    f.pairs = pairs;
    f.pair_bytes = p.pair_bytes;
    f.dst = (uint8_t*)dst;
    if (t_seg) f.seg = *t_seg;   // mode 0 writes each row to its segment
    f.row_bytes = (uint32_t)row;
    f.slot_pairs = p.slot_pairs;
    f.region_cap = (uint32_t)align_up(p.run_len * rec + 32, 16);
    f.stage_bytes = p.stage_bytes;
    f.npre = p.npre;
    f.rid_cache = (p.rid_cache && ((uintptr_t)rids % 16 == 0)) ? 1 : 0;
    f.hist_warps = p.hist_warps;
    f.tile = p.tile;
    f.rcache_words = p.rid_cache ? p.tile : 0;
    f.cap = p.slot_pairs;
    f.ovf = (uint64_t*)((uint8_t*)pairs + pairs_sz);
    f.max_own = (uint32_t)((p.num_runs + p.grid_probe - 1) / p.grid_probe);
    f.status = status;
    f.ts = g_debug_ts;
    f.dbg = g_debug_flags;
    {
      // Phase II: about 3/4 of the runs statically (c + t*G), the rest claimed
      // dynamically by the CTAs that finish first
      const uint64_t G = p.grid_probe, K = p.num_runs;
      const uint64_t frac16 = (f.dbg >> 8) & 31 ? (f.dbg >> 8) & 31 : 12;
      uint64_t ns = frac16 >= 16 ? (K + G - 1) / G : K * frac16 / (16 * G);
      ns = std::max<uint64_t>(ns, p.npre);
      f.n_static = (uint32_t)std::min<uint64_t>(ns, (K + G - 1) / G);
    }
    uintptr_t outs = (uintptr_t)dst;
    if (t_seg)
      for (uint32_t q = 0; q < t_seg->n; ++q) outs |= (uintptr_t)t_seg->out[q];
    uint32_t W = pow2_divisor(rec | (uintptr_t)src | outs |
                              (f.mode == 1 ? (uintptr_t)f.internal : 0));
    uint32_t nl = 0;
    PhaseEvents pe;
    const bool timed = timing_begin(st, &pe);
    if (timed) cudaEventRecord(pe.e1, st);  // Phase I runs inside the same kernel
    cudaError_t e = launch_fused(f, W, p.grid_probe, p.smem_bytes, st, &nl);
    if (e == cudaSuccess && f.mode == 1) {
      // Phase III: gather "the next record from the j-th INTERNAL run",
      // i.e. INTERNAL[inv[i]], writing the output rows sequentially; a full-
      // occupancy launch of the direct-gather kernel over (INTERNAL, inv).
      // (rows marked 0xFFFFFFFF were reported in Phase I or copied from the
      // overflow list; the gather leaves them alone and reports nothing)
      e = launch_direct(f.internal, slots, (uint32_t)rec, f.inv, n_out, (uint8_t*)dst,
                        pow2_divisor(rec | (uintptr_t)dst | (uintptr_t)f.internal), sm, nullptr,
                        st, &nl, /*hint=*/1);
    }
    if (timed) cudaEventRecord(pe.e2, st);
    t_launches = nl + nl_skew;
    return cuda_status(e);
  }

  Workspace w;
  dpg_status_t as = alloc_workspace(p, n_out, st, &w);
  if (as != DPG_OK) return as;
  uint32_t nl = 0;
  const uint64_t M = p.num_runs * (uint64_t)p.grid_distribute;
  if (!p.hist_in_smem && !p.dist_radix) {
    cudaError_t e = cudaMemsetAsync(w.counts, 0, M * 4, st);
    if (e != cudaSuccess) { cudaFreeAsync(w.base, st); return cuda_status(e); }
  }
  uint32_t* gbar = nullptr;
  if (p.dist_radix) {
    uint32_t* tot = nullptr;
    void* scr = nullptr;
    dpg_status_t gs = persist_ws(st, 1, 0, &gbar, &tot, &scr, &ws_hold);
    if (gs != DPG_OK) { cudaFreeAsync(w.base, st); return gs; }
  }
  DistArgs d;
  std::memset(&d, 0, sizeof(d));
  d.rids = rids;
  d.n_out = n_out;
  d.n_src = n_src;
  d.s = p.log2_run;
  d.K = (uint32_t)p.num_runs;
  d.G = p.grid_distribute;
  d.chunk = (n_out + d.G - 1) / d.G;
  d.counts = w.counts;
  d.run_start = w.run_start;
  d.pairs = w.pairs;
  d.pair_bytes = p.pair_bytes;
  d.pay_src = (const uint8_t*)pay_src;
  d.pay_dst = w.pay;
  d.pay_bytes = (uint32_t)pay;
  d.hist_smem = p.hist_in_smem;
  d.status = status;
  d.bmap = t_bounds ? t_bounds->bmap : nullptr;
  d.btab = t_bounds ? t_bounds->btab : nullptr;
  PhaseEvents pe;
  const bool timed = timing_begin(st, &pe);
  cudaError_t e = p.dist_radix
                      ? launch_radix_distribute(rids, n_out, n_src, p.log2_run, d.K, w.tmp,
                                                (uint64_t*)w.pairs, w.counts, gbar + 8,
                                                w.run_start, sm, st, &nl, status)
                      : launch_distribute(d, false, st, &nl);
  if (e == cudaSuccess)
    e = launch_items(w.run_start, d.K, p.slot_pairs, w.item_cnt, w.item_part, w.item_start,
                     w.item_run, st, &nl);
  if (timed) cudaEventRecord(pe.e1, st);
  if (e == cudaSuccess) {
    ProbeArgs a;
    std::memset(&a, 0, sizeof(a));
    a.src = (const uint8_t*)src;
    a.n_src = n_src;
    a.rec = (uint32_t)rec;
    a.s = p.log2_run;
    a.K = (uint32_t)p.num_runs;
    a.run_start = w.run_start;
    a.pairs = w.pairs;
    a.pair_bytes = p.pair_bytes;
    a.pay = w.pay;
    a.pay_bytes = (uint32_t)pay;
    a.dst = (uint8_t*)dst;
    a.row_bytes = (uint32_t)row;
    a.slot_pairs = p.slot_pairs;
    a.region_cap = (uint32_t)align_up(p.run_len * rec + 32, 16);
    a.slot_bytes = (p.smem_bytes - kBarBytes) / 2;
    a.bmap = d.bmap;
    a.item_start = w.item_start;
    a.item_run = w.item_run;
    a.rid_pairs = p.dist_radix ? 1u : 0u;
    uintptr_t outs = (uintptr_t)dst;
    if (t_seg) {
      a.seg = *t_seg;   // the probe writes each row to its segment
      for (uint32_t q = 0; q < t_seg->n; ++q) outs |= (uintptr_t)t_seg->out[q];
    }
    uint32_t W = pow2_divisor(rec | pay | (uintptr_t)src | outs);
    e = launch_probe_gather(a, W, p.grid_probe, p.smem_bytes, st, &nl);
  }
  if (timed) cudaEventRecord(pe.e2, st);
  cudaFreeAsync(w.base, st);
  t_launches = nl + nl_skew;
  return cuda_status(e);
}

}  // namespace dpg

namespace dpg {
uint32_t t_launches_get() { return t_launches; }
void t_launches_set(uint32_t n) { t_launches = n; }
}  // namespace dpg

extern "C" {

int dpg_version(void) { return 1; }

uint32_t dpg_last_path(void) { return t_path; }

uint32_t dpg_last_launch_count(void) { return t_launches; }

void dpg_debug_phase_stamps(void* device_buf) { g_debug_ts = (unsigned long long*)device_buf; }
void dpg_debug_flags(uint32_t flags) { g_debug_flags = flags; }

void dpg_phase_timing(int enable) {
  std::lock_guard<std::mutex> lk(g_timing_mu);
  g_timing = enable != 0;
}

dpg_status_t dpg_phase_times_ex(double* phase1_ms, double* phase2_ms, double* phase3_ms,
                                uint32_t* calls) {
  std::lock_guard<std::mutex> lk(g_timing_mu);
  double d = 0, p = 0, g = 0;
  for (auto& pe : g_pending) {
    float a = 0, b = 0, c = 0;
    if (cudaEventSynchronize(pe.e2) != cudaSuccess) return cuda_status(cudaGetLastError());
    cudaEventElapsedTime(&a, pe.e0, pe.e1);
    if (pe.has3) {
      cudaEventElapsedTime(&b, pe.e1, pe.e3);
      cudaEventElapsedTime(&c, pe.e3, pe.e2);
    } else {
      cudaEventElapsedTime(&b, pe.e1, pe.e2);
    }
    d += a;
    p += b;
    g += c;
    g_pool.push_back(pe);
  }
  if (phase1_ms) *phase1_ms = d;
  if (phase2_ms) *phase2_ms = p;
  if (phase3_ms) *phase3_ms = g;
  if (calls) *calls = (uint32_t)g_pending.size();
  g_pending.clear();
  return DPG_OK;
}

dpg_status_t dpg_phase_times(double* distribute_ms, double* probe_gather_ms, uint32_t* calls) {
  double p2 = 0, p3 = 0;
  dpg_status_t r = dpg_phase_times_ex(distribute_ms, &p2, &p3, calls);
  if (probe_gather_ms) *probe_gather_ms = p2 + p3;
  return r;
}

const char* dpg_status_string(dpg_status_t s) {
  switch (s) {
    case DPG_OK: return "DPG_OK";
    case DPG_ERR_INVALID_ARG: return "DPG_ERR_INVALID_ARG";
    case DPG_ERR_RID_RANGE: return "DPG_ERR_RID_RANGE";
    case DPG_ERR_UNSUPPORTED: return "DPG_ERR_UNSUPPORTED";
    case DPG_ERR_OOM: return "DPG_ERR_OOM";
    case DPG_ERR_CUDA: return "DPG_ERR_CUDA";
    case DPG_ERR_NCCL: return "DPG_ERR_NCCL";
  }
  return "DPG_ERR_UNKNOWN";
}

dpg_status_t dpg_plan(size_t rec_bytes, uint64_t n_src, uint64_t n_out, size_t pay_bytes,
                      const dpg_options_t* opt, int sm_count, dpg_plan_t* plan) {
  return make_plan(rec_bytes, n_src, n_out, pay_bytes, opt, sm_count, plan);
}

dpg_status_t dpg_retrieve_ex(const void* src, size_t rec_bytes, uint64_t n_src,
                             const uint32_t* rids, uint64_t n_out, void* dst, dpg_stream_t stream,
                             const dpg_options_t* opt) {
  return run_dpg(src, rec_bytes, n_src, rids, n_out, nullptr, 0, dst, (cudaStream_t)stream, opt);
}

dpg_status_t dpg_retrieve(const void* src, size_t rec_bytes, uint64_t n_src, const uint32_t* rids,
                          uint64_t n_out, void* dst, dpg_stream_t stream) {
  return dpg_retrieve_ex(src, rec_bytes, n_src, rids, n_out, dst, stream, nullptr);
}

dpg_status_t dpg_retrieve_segments(const void* src, size_t rec_bytes, uint64_t n_src,
                                   const uint32_t* rids, uint64_t n_out, uint32_t nseg,
                                   const uint64_t* seg_rows, void* const* seg_dst,
                                   dpg_stream_t stream) {
  t_launches = 0;
  if (nseg == 0 || nseg > (uint32_t)kMaxSegs || !seg_rows || !seg_dst) return DPG_ERR_INVALID_ARG;
  if (rec_bytes == 0) return DPG_ERR_INVALID_ARG;
  OutSegs sg;
  std::memset(&sg, 0, sizeof(sg));
  sg.n = nseg;
  uint64_t k = 0;
  for (uint32_t q = 0; q < nseg; ++q) {
    sg.start[q] = (uint32_t)k;
    sg.out[q] = (uint8_t*)seg_dst[q];
    if (seg_rows[q] && !seg_dst[q]) return DPG_ERR_INVALID_ARG;
    uint64_t bytes;
    if (__builtin_mul_overflow(seg_rows[q], (uint64_t)rec_bytes, &bytes)) return DPG_ERR_INVALID_ARG;
    if (seg_rows[q] && (overlaps(seg_dst[q], bytes, src, n_src * rec_bytes) ||
                        overlaps(seg_dst[q], bytes, rids, n_out * 4)))
      return DPG_ERR_INVALID_ARG;
    if (!sg.out[0] && seg_rows[q]) sg.out[0] = sg.out[q];
    k += seg_rows[q];
    if (k > UINT32_MAX) return DPG_ERR_UNSUPPORTED;
  }
  if (k != n_out) return DPG_ERR_INVALID_ARG;
  sg.start[nseg] = (uint32_t)k;
  for (uint32_t q = 0; q < nseg; ++q)
    if (!sg.out[q]) sg.out[q] = sg.out[0];          // empty segments: never written
  if (n_out == 0) return DPG_OK;
  t_seg = &sg;
  // (dst is only a placeholder for the argument checks: every row goes to its segment)
  const dpg_status_t s = run_dpg(src, rec_bytes, n_src, rids, n_out, nullptr, 0, sg.out[0],
                                 (cudaStream_t)stream, nullptr);
  t_seg = nullptr;
  return s;
}

dpg_status_t dpg_fk_join_ex(const void* fact, size_t fact_bytes, uint64_t n_fact,
                            const uint32_t* fk_col, const void* dim, size_t rec_bytes,
                            uint64_t n_dim, void* out, dpg_stream_t stream,
                            const dpg_options_t* opt) {
  // DPG-Move join: with the join triples in rid_R order, "move the
  // records of F into a temporary file according to the ordering of the
  // records of R" -- a DPG retrieval of dim by fk_col -- then "join the
  // temporary file with the remaining relation", one sequential
  // pass writing out row i = fact[i] ++ temp[i].  (opt->path == 2 with a
  // payload instead carries the fact row through the distribute kernels.)
  t_launches = 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (fact_bytes == 0 || (opt && (opt->path == 2 || opt->path == 6)))
    return run_dpg(dim, rec_bytes, n_dim, fk_col, n_fact, fact, fact_bytes, out, st, opt);
  // A dimension table beyond the L2: the three sequential passes carrying the
  // fact rows, which build the output rows in their Phase III (no temporary
  // file and no join pass): config 4 4.99 vs 5.49 ms, c4x 4.57 vs 5.28 ms
  // (profiles/r02_join_plans.md)
  const bool auto_opts = !opt || (!opt->path && !opt->log2_run && !opt->grid_distribute &&
                                  !opt->grid_probe && !opt->pair_bytes && !opt->hist_mode &&
                                  !opt->gather && !opt->cluster);
  uint64_t dim_bytes_total = 0;
  if (auto_opts && !__builtin_mul_overflow(n_dim, (uint64_t)rec_bytes, &dim_bytes_total) &&
      dim_bytes_total > l2_budget(current_l2_bytes())) {
    dpg_options_t o;
    std::memset(&o, 0, sizeof(o));
    o.path = 6;
    dpg_plan_t q;
    if (make_plan(rec_bytes, n_dim, n_fact, fact_bytes, &o, current_sm_count(), &q) == DPG_OK &&
        q.path == 6)
      return run_dpg(dim, rec_bytes, n_dim, fk_col, n_fact, fact, fact_bytes, out, st, &o);
  }
  if (rec_bytes == 0) return DPG_ERR_INVALID_ARG;
  if (n_fact == 0) return DPG_OK;
  if (!fact || !fk_col || !dim || !out || n_dim == 0) return DPG_ERR_INVALID_ARG;
  uint64_t row, out_bytes, tmp_bytes, fact_total, dim_total;
  if (__builtin_add_overflow((uint64_t)fact_bytes, (uint64_t)rec_bytes, &row) ||
      __builtin_mul_overflow(n_fact, row, &out_bytes) ||
      __builtin_mul_overflow(n_fact, (uint64_t)rec_bytes, &tmp_bytes) ||
      __builtin_mul_overflow(n_fact, (uint64_t)fact_bytes, &fact_total) ||
      __builtin_mul_overflow(n_dim, (uint64_t)rec_bytes, &dim_total))
    return DPG_ERR_INVALID_ARG;
  if (row > UINT32_MAX / 2) return DPG_ERR_UNSUPPORTED;
  if (overlaps(out, out_bytes, fact, fact_total) || overlaps(out, out_bytes, dim, dim_total) ||
      overlaps(out, out_bytes, fk_col, n_fact * 4))
    return DPG_ERR_INVALID_ARG;
  void* tmp = nullptr;
  if (ws_malloc(&tmp, tmp_bytes + 256, st) != cudaSuccess) {
    cudaGetLastError();
    return DPG_ERR_OOM;
  }
  dpg_status_t s = run_dpg(dim, rec_bytes, n_dim, fk_col, n_fact, nullptr, 0, tmp, st, opt);
  uint32_t nl = t_launches;
  if (s == DPG_OK) {
    const uint32_t W = pow2_divisor(fact_bytes | rec_bytes | (uintptr_t)fact | (uintptr_t)tmp |
                                    (uintptr_t)out);
    cudaError_t e = launch_zip_rows((const uint8_t*)fact, (uint32_t)fact_bytes,
                                    (const uint8_t*)tmp, (uint32_t)rec_bytes, n_fact,
                                    (uint8_t*)out, W, current_sm_count(), st, &nl,
                                    fk_col, n_dim);   // an fk >= n_dim: row left unwritten
    s = cuda_status(e);
  }
  cudaFreeAsync(tmp, st);
  t_launches = nl;
  return s;
}

dpg_status_t dpg_fk_join(const void* fact, size_t fact_bytes, uint64_t n_fact,
                         const uint32_t* fk_col, const void* dim, size_t rec_bytes, uint64_t n_dim,
                         void* out, dpg_stream_t stream) {
  return dpg_fk_join_ex(fact, fact_bytes, n_fact, fk_col, dim, rec_bytes, n_dim, out, stream,
                        nullptr);
}

dpg_status_t dpg_retrieve_direct(const void* src, size_t rec_bytes, uint64_t n_src,
                                 const uint32_t* rids, uint64_t n_out, void* dst,
                                 dpg_stream_t stream) {
  return dpg_retrieve_direct_ex(src, rec_bytes, n_src, rids, n_out, dst, stream, 0);
}

dpg_status_t dpg_l2_prefetch(const void* ptr, uint64_t bytes, dpg_stream_t stream) {
  t_launches = 0;
  if (!bytes) return DPG_OK;
  if (!ptr) return DPG_ERR_INVALID_ARG;
  uint32_t nl = 0;
  cudaError_t e = launch_l2_prefetch(ptr, bytes, current_sm_count(), (cudaStream_t)stream, &nl);
  t_launches = nl;
  return cuda_status(e);
}

dpg_status_t dpg_retrieve_direct_ex(const void* src, size_t rec_bytes, uint64_t n_src,
                                    const uint32_t* rids, uint64_t n_out, void* dst,
                                    dpg_stream_t stream, int hint) {
  WsHold ws_hold;   // the stream's workspace stays ours until the launches are enqueued
  t_launches = 0;
  if (rec_bytes == 0) return DPG_ERR_INVALID_ARG;
  if (n_out == 0) return DPG_OK;
  if (!src || !rids || !dst || n_src == 0) return DPG_ERR_INVALID_ARG;
  if (n_out >= (1ull << 32) || n_src > (1ull << 32)) return DPG_ERR_UNSUPPORTED;
  uint64_t src_bytes, dst_bytes;
  if (__builtin_mul_overflow(n_src, (uint64_t)rec_bytes, &src_bytes) ||
      __builtin_mul_overflow(n_out, (uint64_t)rec_bytes, &dst_bytes))
    return DPG_ERR_INVALID_ARG;
  if (rec_bytes > UINT32_MAX / 2) return DPG_ERR_UNSUPPORTED;
  if (overlaps(dst, dst_bytes, src, src_bytes) || overlaps(dst, dst_bytes, rids, n_out * 4))
    return DPG_ERR_INVALID_ARG;
  unsigned long long* status = device_status();
  if (!status) return DPG_ERR_CUDA;
  uint32_t W = pow2_divisor(rec_bytes | (uintptr_t)src | (uintptr_t)dst);
  uint32_t nl = 0;
  if (hint == 3) {
    // the direct retrieval on the L2-run kernel's gather (16-byte windows,
    // realigned in shared memory, coalesced 16-byte row stores), no staging
    uint32_t *gbar = nullptr, *total = nullptr;
    void* pairs = nullptr;
    dpg_status_t ws = persist_ws((cudaStream_t)stream, 1, 64, &gbar, &total, &pairs, &ws_hold);
    if (ws != DPG_OK) return ws;
    const int sm = current_sm_count();
    L2RunArgs l;
    std::memset(&l, 0, sizeof(l));
    l.src = (const uint8_t*)src;
    l.n_src = n_src;
    l.rec = (uint32_t)rec_bytes;
    l.rids = rids;
    l.n_out = n_out;
    l.chunk = align_up((n_out + sm - 1) / sm, 32);
    l.dst = (uint8_t*)dst;
    l.gbar = gbar;
    l.status = status;
    l.stage = 0;
    if (rec_bytes % 4 == 0) l.rd_magic = (uint32_t)(((1ull << 32) + rec_bytes / 4 - 1) / (rec_bytes / 4));
    cudaError_t e = launch_l2run(l, W, (uint32_t)sm, (cudaStream_t)stream, &nl);
    t_launches = nl;
    return cuda_status(e);
  }
  cudaError_t e = launch_direct((const uint8_t*)src, n_src, (uint32_t)rec_bytes, rids, n_out,
                                (uint8_t*)dst, W, current_sm_count(), status,
                                (cudaStream_t)stream, &nl, hint);
  t_launches = nl;
  return cuda_status(e);
}

dpg_status_t dpg_distribute(const uint32_t* rids, uint64_t n_out, uint64_t n_src, uint32_t log2_run,
                            uint64_t* pairs_out, uint64_t* run_start_out, dpg_stream_t stream,
                            const dpg_options_t* opt) {
  t_launches = 0;
  if (n_src == 0 || !run_start_out || (n_out && (!rids || !pairs_out)) || log2_run > 31)
    return DPG_ERR_INVALID_ARG;
  if (n_out >= (1ull << 32) || n_src > (1ull << 32)) return DPG_ERR_UNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream;
  const int sm = current_sm_count();
  const uint64_t L = 1ull << log2_run;
  const uint64_t K = t_bounds ? t_bounds->K : (n_src + L - 1) >> log2_run;
  if (K >= (1ull << 31)) return DPG_ERR_UNSUPPORTED;
  if (t_bounds && opt && opt->path == 6) return DPG_ERR_UNSUPPORTED;
  unsigned long long* status0 = device_status();
  if (!status0) return DPG_ERR_CUDA;
  if (opt && opt->path == 6 && n_out) {
    // Phase I of the three sequential passes (seq3.cu): RID_RUN with the
    // positions, tile by tile; returned run-major (run b = its pieces (t, b)
    // in tile order), the reordering done here on the host (test entry)
    dpg_options_t o = *opt;
    o.log2_run = log2_run;
    dpg_plan_t q;
    if (log2_run > 16 || !plan_seq3(4, n_src, n_out, 0, &o, sm, &q)) return DPG_ERR_UNSUPPORTED;
    const uint64_t T = q.tile, nsub = (n_out + T - 1) / T;
    const uint64_t off_preT = align_up(nsub * (K + 1) * 2, 256);
    const uint64_t off_loc = align_up(off_preT + nsub * (K + 1) * 2, 256);
    const uint64_t off_tinv = align_up(off_loc + nsub * T * 2, 256);
    const uint64_t off_pairs = align_up(off_tinv + nsub * T * 2 + 16, 256);
    const uint64_t bytes = off_pairs + nsub * T * 8;
    void* b = nullptr;
    if (cudaMalloc(&b, bytes) != cudaSuccess) { cudaGetLastError(); return DPG_ERR_OOM; }
    uint8_t* wb = (uint8_t*)b;
    Seq3Args a;
    std::memset(&a, 0, sizeof(a));
    a.rids = rids;
    a.n_out = n_out;
    a.n_src = n_src;
    a.s = log2_run;
    a.K = (uint32_t)K;
    a.T = (uint32_t)T;
    a.nsub = (uint32_t)nsub;
    a.pre = (uint16_t*)wb;
    a.preT = (uint16_t*)(wb + off_preT);
    a.loc = (uint16_t*)(wb + off_loc);
    a.tinv = (uint16_t*)(wb + off_tinv);
    a.dbg_pairs = (uint64_t*)(wb + off_pairs);
    a.status = status0;
    uint32_t nl = 0;
    cudaError_t e = launch_seq3_distribute(a, q.grid_distribute, st, &nl);
    std::vector<uint16_t> pre(nsub * (K + 1));
    std::vector<uint64_t> tp(nsub * T), out(n_out);
    std::vector<uint64_t> rs(K + 1, 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(pre.data(), a.pre, pre.size() * 2, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(tp.data(), a.dbg_pairs, tp.size() * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) {
      uint64_t k = 0;
      for (uint64_t r = 0; r < K; ++r) {
        rs[r] = k;
        for (uint64_t t = 0; t < nsub; ++t)
          for (uint32_t j = pre[t * (K + 1) + r]; j < pre[t * (K + 1) + r + 1]; ++j) out[k++] = tp[t * T + j];
      }
      rs[K] = k;
      e = cudaMemcpyAsync(pairs_out, out.data(), k * 8, cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(run_start_out, rs.data(), (K + 1) * 8, cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    }
    cudaFree(b);
    t_launches = nl;
    return cuda_status(e);
  }
  dpg_plan_t p;
  std::memset(&p, 0, sizeof(p));
  p.log2_run = log2_run;
  p.run_len = L;
  p.num_runs = K;
  const bool force8 = opt && opt->pair_bytes == 8;
  p.pair_bytes = (!force8 && log2_run + bit_length(n_out ? n_out - 1 : 0) <= 32) ? 4 : 8;
  dpg_status_t ds = dist_geometry(K, n_out, opt, sm, &p);
  if (ds != DPG_OK) return ds;
  if (opt && opt->hist_mode == 3 && !t_bounds) {   // radix passes (reading A24)
    p.dist_radix = radix_passes(K);
    p.grid_distribute = 3u * (uint32_t)sm;
    p.hist_in_smem = 0;
    p.pair_bytes = 8;
  }
  unsigned long long* status = device_status();
  if (!status) return DPG_ERR_CUDA;
  Workspace w;
  dpg_status_t as = alloc_workspace(p, n_out, st, &w);
  if (as != DPG_OK) return as;
  uint32_t nl = 0;
  if (p.dist_radix) {
    WsHold hold;
    uint32_t *gbar = nullptr, *tot = nullptr;
    void* scr = nullptr;
    dpg_status_t gs = persist_ws(st, 1, 0, &gbar, &tot, &scr, &hold);
    cudaError_t e = gs == DPG_OK ? cudaSuccess : cudaErrorMemoryAllocation;
    if (e == cudaSuccess)
      e = launch_radix_distribute(rids, n_out, n_src, log2_run, (uint32_t)K, w.tmp,
                                  (uint64_t*)w.pairs, w.counts, gbar + 8, w.run_start, sm, st,
                                  &nl, status);
    if (e == cudaSuccess)
      e = launch_radix_unpack((const uint64_t*)w.pairs, n_out, log2_run, w.run_start, (uint32_t)K,
                              pairs_out, run_start_out, st, &nl);
    cudaFreeAsync(w.base, st);
    t_launches = nl;
    return gs != DPG_OK ? gs : cuda_status(e);
  }
  cudaError_t e = cudaSuccess;
  if (!p.hist_in_smem) e = cudaMemsetAsync(w.counts, 0, K * (uint64_t)p.grid_distribute * 4, st);
  DistArgs d;
  std::memset(&d, 0, sizeof(d));
  d.rids = rids;
  d.n_out = n_out;
  d.n_src = n_src;
  d.s = log2_run;
  d.K = (uint32_t)K;
  d.G = p.grid_distribute;
  d.chunk = (n_out + d.G - 1) / d.G;
  d.counts = w.counts;
  d.run_start = w.run_start;
  d.pairs = w.pairs;
  d.pair_bytes = p.pair_bytes;
  d.hist_smem = p.hist_in_smem;
  d.status = status;
  d.bmap = t_bounds ? t_bounds->bmap : nullptr;
  d.btab = t_bounds ? t_bounds->btab : nullptr;
  if (e == cudaSuccess && n_out) e = launch_distribute(d, false, st, &nl);
  if (e == cudaSuccess) {
    if (!n_out) {
      e = cudaMemsetAsync(w.run_start, 0, (K + 1) * 4, st);
      d.run_start = w.run_start;
    }
    if (e == cudaSuccess) e = launch_unpack_pairs(d, pairs_out, run_start_out, st, &nl);
  }
  cudaFreeAsync(w.base, st);
  t_launches = nl;
  return cuda_status(e);
}

dpg_status_t dpg_partition(const void* rids, uint32_t rid_bytes, uint64_t n, uint64_t n_src_total,
                           uint32_t log2_span, uint32_t parts, uint32_t* local_out,
                           uint32_t* pos_out, uint64_t* counts_out, dpg_stream_t stream) {
  t_launches = 0;
  if ((rid_bytes != 4 && rid_bytes != 8) || parts == 0 || log2_span > 32 || !counts_out)
    return DPG_ERR_INVALID_ARG;
  if (n && (!rids || !local_out || !pos_out)) return DPG_ERR_INVALID_ARG;
  if (n >= (1ull << 32)) return DPG_ERR_UNSUPPORTED;
  if (n_src_total == 0 || (((n_src_total - 1) >> log2_span) >= parts)) return DPG_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* status = device_status();
  if (!status) return DPG_ERR_CUDA;
  if (n == 0) return cuda_status(cudaMemsetAsync(counts_out, 0, parts * sizeof(uint64_t), st));
  const int sm = current_sm_count();
  dpg_plan_t p;
  std::memset(&p, 0, sizeof(p));
  p.log2_run = log2_span;
  p.num_runs = parts;
  p.pair_bytes = 8;
  dpg_options_t o;
  std::memset(&o, 0, sizeof(o));
  o.hist_mode = 1;                      // parts counters always fit shared memory
  if (parts * 4 > kSmemLimit) return DPG_ERR_UNSUPPORTED;
  dpg_status_t ds = dist_geometry(parts, n, &o, sm, &p);
  if (ds != DPG_OK) return ds;
  Workspace w;
  dpg_status_t as = alloc_workspace(p, n, st, &w);
  if (as != DPG_OK) return as;
  DistArgs d;
  std::memset(&d, 0, sizeof(d));
  d.rids = rids;
  d.n_out = n;
  d.n_src = n_src_total;
  d.s = log2_span;
  d.K = parts;
  d.G = p.grid_distribute;
  d.chunk = (n + d.G - 1) / d.G;
  d.counts = w.counts;
  d.run_start = w.run_start;
  d.pairs = w.pairs;
  d.pair_bytes = 8;
  d.hist_smem = 1;
  d.status = status;
  uint32_t nl = 0;
  cudaError_t e = launch_distribute(d, rid_bytes == 8, st, &nl);
  if (e == cudaSuccess) e = launch_split_entries(d, local_out, pos_out, counts_out, st, &nl);
  cudaFreeAsync(w.base, st);
  t_launches = nl;
  return cuda_status(e);
}

dpg_status_t dpg_partition_inv(const void* rids, uint32_t rid_bytes, uint64_t n,
                               uint64_t n_src_total, uint32_t log2_span, uint32_t parts,
                               uint32_t* local_out, uint32_t* inv_out, uint64_t* counts_out,
                               dpg_stream_t stream) {
  WsHold ws_hold;   // the stream's workspace stays ours until the launches are enqueued
  // Phase I of the multi-GPU path with Phase III's map: requests grouped by
  // owner (owner = rid >> log2_span), and for every row the slot of its request
  // (the replies come back in request order, so dst[i] = reply[inv[i]]).
  t_launches = 0;
  if ((rid_bytes != 4 && rid_bytes != 8) || parts == 0 || parts > 512 || log2_span > 32 ||
      !counts_out)
    return DPG_ERR_INVALID_ARG;
  if (n && (!rids || !local_out || !inv_out)) return DPG_ERR_INVALID_ARG;
  if (n >= (1ull << 32) - 1) return DPG_ERR_UNSUPPORTED;
  if (n_src_total == 0 || (((n_src_total - 1) >> log2_span) >= parts)) return DPG_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* status = device_status();
  if (!status) return DPG_ERR_CUDA;
  if (n == 0) return cuda_status(cudaMemsetAsync(counts_out, 0, parts * sizeof(uint64_t), st));
  const int sm = current_sm_count();
  uint32_t *gbar = nullptr, *total = nullptr;
  void* ws = nullptr;
  const uint64_t cbytes = align_up((uint64_t)parts * sm * 4, 256) + align_up((parts + 1) * 4, 256);
  dpg_status_t w = persist_ws(st, 1, cbytes, &gbar, &total, &ws, &ws_hold);
  if (w != DPG_OK) return w;
  L2KArgs d;
  std::memset(&d, 0, sizeof(d));
  d.rids = rids;
  d.rid_bytes = rid_bytes;
  d.counts64 = counts_out;
  d.n_out = n;
  d.n_src = n_src_total;
  d.s = log2_span;
  d.K = parts;
  d.chunk = align_up((n + sm - 1) / sm, 32);
  d.counts = (uint32_t*)ws;
  d.run_start = (uint32_t*)((uint8_t*)ws + align_up((uint64_t)parts * sm * 4, 256));
  d.local = local_out;
  d.inv = inv_out;
  d.gbar = gbar + 16;
  d.status = status;
  uint32_t nl = 0;
  cudaError_t e = launch_l2k_distribute(d, (uint32_t)sm, st, &nl);
  t_launches = nl;
  return cuda_status(e);
}

dpg_status_t dpg_ipc_alloc(size_t bytes, void** ptr, uint8_t handle[64]) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  if (!ptr || !handle || bytes == 0) return DPG_ERR_INVALID_ARG;
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return DPG_ERR_OOM;
  }
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return cuda_status(e);
  }
  std::memcpy(handle, &h, 64);
  *ptr = p;
  return DPG_OK;
}

dpg_status_t dpg_ipc_open(const uint8_t handle[64], void** ptr) {
  if (!ptr || !handle) return DPG_ERR_INVALID_ARG;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  return cuda_status(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
}

dpg_status_t dpg_ipc_close(void* ptr) { return cuda_status(cudaIpcCloseMemHandle(ptr)); }

dpg_status_t dpg_ipc_free(void* ptr) { return cuda_status(cudaFree(ptr)); }

dpg_status_t dpg_gather_rows(const void* rows, size_t rec_bytes, uint64_t n_rows, const uint32_t* inv,
                             uint64_t n, void* dst, dpg_stream_t stream) {
  WsHold ws_hold;   // the stream's workspace stays ours until the launches are enqueued
  // dst[i] = rows[inv[i]] (rows with inv[i] >= n_rows stay unwritten): the
  // multi-GPU path's Phase III over the replies, in output order.
  t_launches = 0;
  if (rec_bytes == 0) return DPG_ERR_INVALID_ARG;
  if (n == 0) return DPG_OK;
  if (!inv || !dst || (n_rows && !rows)) return DPG_ERR_INVALID_ARG;
  if (n >= (1ull << 32) || n_rows > (1ull << 32) || rec_bytes > UINT32_MAX / 2) return DPG_ERR_UNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t *gbar = nullptr, *total = nullptr;
  void* ws = nullptr;
  dpg_status_t w = persist_ws(st, 1, 64, &gbar, &total, &ws, &ws_hold);
  if (w != DPG_OK) return w;
  const int sm = current_sm_count();
  L2RunArgs l;
  std::memset(&l, 0, sizeof(l));
  l.src = (const uint8_t*)rows;
  l.n_src = n_rows;
  l.rec = (uint32_t)rec_bytes;
  l.rids = inv;
  l.n_out = n;
  l.chunk = align_up((n + sm - 1) / sm, 32);
  l.dst = (uint8_t*)dst;
  l.gbar = gbar;
  l.stage = 0;
  if (rec_bytes % 4 == 0) l.rd_magic = (uint32_t)(((1ull << 32) + rec_bytes / 4 - 1) / (rec_bytes / 4));
  const uint32_t W = pow2_divisor(rec_bytes | (uintptr_t)rows | (uintptr_t)dst);
  uint32_t nl = 0;
  cudaError_t e = launch_l2run(l, W, (uint32_t)sm, st, &nl);
  t_launches = nl;
  return cuda_status(e);
}

dpg_status_t dpg_scatter_rows(const void* rows, size_t rec_bytes, const uint32_t* pos, uint64_t n,
                              void* dst, uint64_t n_dst, dpg_stream_t stream) {
  t_launches = 0;
  if (rec_bytes == 0) return DPG_ERR_INVALID_ARG;
  if (n == 0) return DPG_OK;
  if (!rows || !pos || !dst) return DPG_ERR_INVALID_ARG;
  if (rec_bytes > UINT32_MAX / 2) return DPG_ERR_UNSUPPORTED;
  uint32_t W = pow2_divisor(rec_bytes | (uintptr_t)rows | (uintptr_t)dst);
  uint32_t nl = 0;
  cudaError_t e = launch_scatter_rows((const uint8_t*)rows, (uint32_t)rec_bytes, pos, n,
                                      (uint8_t*)dst, n_dst, W, current_sm_count(),
                                      (cudaStream_t)stream, &nl);
  t_launches = nl;
  return cuda_status(e);
}

dpg_status_t dpg_sync_status(dpg_stream_t stream, uint64_t* first_bad_index) {
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_status(e);
  unsigned long long* status = device_status();
  if (!status) return DPG_ERR_CUDA;
  unsigned long long v = 0;
  e = cudaMemcpy(&v, status, sizeof(v), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_status(e);
  if (v == ~0ull) return DPG_OK;
  unsigned long long init = ~0ull;
  e = cudaMemcpy(status, &init, sizeof(init), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_status(e);
  if (first_bad_index) *first_bad_index = v;
  return DPG_ERR_RID_RANGE;
}

// ---- end-to-end entries with host buffers -------------------------------------
// Device buffers of dpg_retrieve_host(_async), cached per (device, stream),
// the kWsCached most recently used streams: calls on one stream reuse them in
// stream order; calls on different streams (the asynchronous entry,
// pipelined) each have their own.  A buffer that has to grow is freed
// stream-ordered (work already queued may still read it).
struct HostBufs {
  int dev = 0;
  cudaStream_t st = nullptr;
  void* buf[3] = {nullptr, nullptr, nullptr};
  size_t cap[3] = {0, 0, 0};
};
static std::mutex g_host_mu;
static std::vector<HostBufs> g_host_bufs;

static dpg_status_t host_bufs(cudaStream_t st, const size_t bytes[3], void* out[3]) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return DPG_ERR_CUDA;
  size_t at = g_host_bufs.size();
  for (size_t q = 0; q < g_host_bufs.size(); ++q)
    if (g_host_bufs[q].dev == dev && g_host_bufs[q].st == st) at = q;
  if (at == g_host_bufs.size()) {
    // at most kWsCached streams keep buffers: the oldest entry goes (freed
    // synchronously -- its stream may no longer exist)
    if (g_host_bufs.size() >= kWsCached) {
      HostBufs& o = g_host_bufs.front();
      int cur = 0;
      cudaGetDevice(&cur);
      cudaSetDevice(o.dev);
      cudaDeviceSynchronize();
      for (int k = 0; k < 3; ++k)
        if (o.buf[k]) cudaFree(o.buf[k]);
      cudaSetDevice(cur);
      cudaGetLastError();
      g_host_bufs.erase(g_host_bufs.begin());
    }
    g_host_bufs.emplace_back();
    g_host_bufs.back().dev = dev;
    g_host_bufs.back().st = st;
    at = g_host_bufs.size() - 1;
  } else if (at + 1 != g_host_bufs.size()) {
    std::rotate(g_host_bufs.begin() + at, g_host_bufs.begin() + at + 1, g_host_bufs.end());
    at = g_host_bufs.size() - 1;                 // most recently used last
  }
  HostBufs* h = &g_host_bufs[at];
  for (int k = 0; k < 3; ++k) {
    if (h->cap[k] < bytes[k]) {
      if (h->buf[k]) cudaFreeAsync(h->buf[k], st);
      h->buf[k] = nullptr;
      h->cap[k] = 0;
      if (ws_malloc(&h->buf[k], bytes[k], st) != cudaSuccess) {
        cudaGetLastError();
        return DPG_ERR_OOM;
      }
      h->cap[k] = bytes[k];
    }
    out[k] = h->buf[k];
  }
  return DPG_OK;
}

dpg_status_t dpg_retrieve_host_async(const void* src_host, size_t rec_bytes, uint64_t n_src,
                                     const uint32_t* rids_host, uint64_t n_out, void* dst_host,
                                     dpg_stream_t stream) {
  if (rec_bytes == 0) return DPG_ERR_INVALID_ARG;
  if (n_out == 0) return DPG_OK;
  if (!src_host || !rids_host || !dst_host || n_src == 0) return DPG_ERR_INVALID_ARG;
  uint64_t sb, db;
  if (__builtin_mul_overflow(n_src, (uint64_t)rec_bytes, &sb) ||
      __builtin_mul_overflow(n_out, (uint64_t)rec_bytes, &db))
    return DPG_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> lk(g_host_mu);
  cudaStream_t st = (cudaStream_t)stream;
  void* b[3];
  const size_t bytes[3] = {sb, n_out * 4, db};
  dpg_status_t x = host_bufs(st, bytes, b);
  if (x != DPG_OK) return x;
  cudaError_t e = cudaMemcpyAsync(b[0], src_host, sb, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(b[1], rids_host, n_out * 4, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_status(e);
  dpg_status_t ds = dpg_retrieve(b[0], rec_bytes, n_src, (const uint32_t*)b[1], n_out, b[2], stream);
  if (ds != DPG_OK) return ds;
  return cuda_status(cudaMemcpyAsync(dst_host, b[2], db, cudaMemcpyDeviceToHost, st));
}

dpg_status_t dpg_retrieve_host(const void* src_host, size_t rec_bytes, uint64_t n_src,
                               const uint32_t* rids_host, uint64_t n_out, void* dst_host,
                               dpg_stream_t stream) {
  dpg_status_t s = dpg_retrieve_host_async(src_host, rec_bytes, n_src, rids_host, n_out,
                                           dst_host, stream);
  if (s != DPG_OK || n_out == 0) return s;
  return cuda_status(cudaStreamSynchronize((cudaStream_t)stream));
}

void dpg_release_cache(void) {
  std::lock_guard<std::mutex> lk(g_host_mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& h : g_host_bufs) {
    cudaSetDevice(h.dev);
    cudaDeviceSynchronize();           // (the stream may be gone: free synchronously)
    for (int k = 0; k < 3; ++k)
      if (h.buf[k]) cudaFree(h.buf[k]);
  }
  g_host_bufs.clear();
  cudaSetDevice(cur);
  cudaGetLastError();
  release_persist_ws();
  ws_pool_trim();
}

}  // extern "C"
