// dpg_internal.cuh -- device helpers and launcher declarations shared by the
// CUDA translation units of libdpg.so (product path; no oracle code here).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dpg.h"

#include <utility>

namespace dpg {

__host__ __device__ __forceinline__ uint64_t min_u64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ uint64_t max_u64(uint64_t a, uint64_t b) { return a > b ? a : b; }

// ---------------------------------------------------------------------------
// Device status word (one per device, library-owned): smallest position i
// whose rid was out of range; ~0 when clean.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void report_bad(unsigned long long* status, uint64_t i) {
  if (status) atomicMin(status, (unsigned long long)i);
}

// ---------------------------------------------------------------------------
// PTX wrappers: mbarrier + cp.async.bulk (TMA bulk copy, sm_90+ / sm_100a).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(tx)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier of a cooperative launch: gbar[0] arrival count, gbar[1]
// generation (both persistent; the count returns to zero).
__device__ __forceinline__ void grid_barrier(uint32_t* gbar, uint32_t G) {
  __syncthreads();
  if (threadIdx.x == 0) {
    // arrival with acq_rel (cumulative over the CTA's writes, ordered by the
    // bar.sync above); the last arriver resets the count and releases the
    // next generation; the others acquire it
    const uint32_t gen = ld_acquire_gpu(gbar + 1);
    uint32_t old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(gbar) : "memory");
    if (old == G - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(gbar) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gbar + 1) : "memory");
    } else {
      while (ld_acquire_gpu(gbar + 1) == gen) {
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
// Named barrier over n threads (a multiple of 32) of the CTA.
__device__ __forceinline__ void named_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Grid barrier with one poller: every CTA adds 1 to a monotonic arrival
// count (red.release, no return); CTA 0 waits for the count of this epoch and
// publishes the next epoch; the others wait for the epoch word (a different
// cache line from the count, so the waiters do not slow the arrivals).
// w[0] = count, w[32] = epoch; both only grow (zero at allocation).  All
// launches sharing w must use the same grid size G: the per-stream workspace
// (persist_ws) keeps three word pairs -- gbar + 0 and gbar + 16 for kernels
// of one CTA per SM, gbar + 8 for path 2's radix passes (sort.cu, 3 CTAs per SM).
__device__ __forceinline__ void grid_barrier_mono(uint32_t* w, uint32_t G) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t epoch = ld_acquire_gpu(w + 32);
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(w) : "memory");
    if (blockIdx.x == 0) {
      const uint32_t target = (epoch + 1) * G;
      while ((int32_t)(ld_acquire_gpu(w) - target) < 0) {
      }
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(w + 32), "r"(epoch + 1) : "memory");
    } else {
      while (ld_acquire_gpu(w + 32) == epoch) __nanosleep(64);
    }
  }
  __syncthreads();
}

// Programmatic dependent launch (PDL) between the kernels of one plan: a
// kernel launched by launch_pdl may be scheduled while its stream predecessor
// is still finishing (its CTAs take SMs as the predecessor's CTAs exit, which
// hides the launch gap, ~2-4 us per kernel boundary); it calls pdl_wait()
// before it touches anything earlier kernels wrote (griddepcontrol.wait
// returns once the predecessor grid has completed and its writes are
// visible; a no-op for an ordinary launch).  pdl_trigger() lets the
// dependent grid be scheduled before this one ends.  Dependents are only
// scheduled once every CTA of this grid has triggered or exited, so a grid's
// own CTAs are all resident first.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Bulk async copy global -> shared, completion counted on `bar` (bytes).
// dst_smem, src and bytes must be 16-byte aligned / multiples of 16.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// ---------------------------------------------------------------------------
// Vector word of W bytes.
// ---------------------------------------------------------------------------
template <int W> struct Word;
template <> struct Word<1> { using T = uint8_t; };
template <> struct Word<2> { using T = uint16_t; };
template <> struct Word<4> { using T = uint32_t; };
template <> struct Word<8> { using T = uint2; };
template <> struct Word<16> { using T = uint4; };

// ---------------------------------------------------------------------------
// Workspace layout of one distribute (host computes, kernels consume).
// ---------------------------------------------------------------------------
struct DistArgs {
  const void* rids;       // uint32 or uint64 rids
  uint64_t n_out;
  uint64_t n_src;
  uint32_t s;             // log2 run length
  uint32_t K;             // number of runs
  uint32_t G;             // number of distribute chunks (CTAs)
  uint64_t chunk;         // rids per chunk
  uint32_t* counts;       // [K*G] bucket-major counts, then exclusive offsets
  uint32_t* run_start;    // [K+1] start of each run in the pair array
  void* pairs;            // [n_out] packed pairs (4 or 8 bytes)
  uint32_t pair_bytes;
  // optional payload carried with each pair (join: the fact row)
  const uint8_t* pay_src;
  uint8_t* pay_dst;
  uint32_t pay_bytes;
  uint32_t hist_smem;     // 1: shared-memory histogram of K counters
  unsigned long long* status;
  // Boundary-mode runs (section 2.3; null: run = r >> s):
  // run b = [bmap[b], bmap[b+1]), at most L = 2^s records wide; btab[h] =
  // the run starting at h*L (a multiple of L is always a run start).
  const uint32_t* bmap;   // [K+1]
  const uint32_t* btab;   // [ceil(n_src / L) + 1], btab[last] = K
};

// Run of rid r in boundary mode: the last b in [btab[h], btab[h+1]) with
// bmap[b] <= r, h = r >> s (the multiples of L bound the search).
__device__ __forceinline__ uint32_t bounds_run(const uint32_t* __restrict__ bmap,
                                               const uint32_t* __restrict__ btab, uint32_t s,
                                               uint64_t r, uint32_t* start) {
  const uint32_t h = (uint32_t)(r >> s);
  uint32_t lo = __ldg(btab + h), hi = __ldg(btab + h + 1);
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((uint64_t)__ldg(bmap + mid) <= r) lo = mid; else hi = mid;
  }
  *start = __ldg(bmap + lo);
  return lo;
}

// Output split into segments (dpg_retrieve_segments; the multi-GPU exchange
// writes each requester's replies straight into its window over NVLink):
// output row k of segment q (start[q] <= k < start[q+1]) goes to
// out[q] + (k - start[q]) * row_bytes.  n = 0: one contiguous dst.
constexpr int kMaxSegs = 8;
struct OutSegs {
  uint32_t n;
  uint32_t start[kMaxSegs + 1];
  uint8_t* out[kMaxSegs];
};
__device__ __forceinline__ uint32_t seg_of(const OutSegs& o, uint64_t k) {
  uint32_t q = 0;
#pragma unroll
  for (int j = 1; j < kMaxSegs; ++j) q += (j < (int)o.n && k >= o.start[j]) ? 1u : 0u;
  return q;
}
__device__ __forceinline__ uint8_t* seg_row(const OutSegs& o, uint8_t* dst, uint64_t k,
                                            uint32_t row_bytes) {
  if (!o.n) return dst + k * row_bytes;
  const uint32_t q = seg_of(o, k);
  return o.out[q] + (k - o.start[q]) * row_bytes;
}

struct ProbeArgs {
  const uint8_t* src;     // staged source records
  uint64_t n_src;
  uint32_t rec;
  uint32_t s;
  uint32_t K;
  const uint32_t* run_start;   // [K+1]
  const void* pairs;
  uint32_t pair_bytes;
  const uint8_t* pay;          // [n_out * pay_bytes] or null
  uint32_t pay_bytes;
  uint8_t* dst;                // row r at dst + r*row_bytes
  uint32_t row_bytes;          // pay_bytes + rec
  uint32_t slot_pairs;         // pairs per stage
  uint32_t region_cap;         // bytes reserved for a region in a stage
  uint32_t slot_bytes;         // total bytes per stage
  OutSegs seg;                 // output segments (seg.n = 0: dst)
  const uint32_t* bmap;        // boundary-mode runs [K+1] (DistArgs), or null
  const uint32_t* item_start;  // [K+1] first item (pair chunk) of each run (launch_items)
  const uint32_t* item_run;    // [items] uint4 {run, chunk, p0, p1} of each item (16-aligned)
  uint32_t rid_pairs;          // 8-byte pairs are radix Phase I elements (rid << 32) | position
};

// One persistent cooperative kernel for the whole path (fused.cu).
struct FusedArgs {
  const uint8_t* src;
  uint64_t n_src;
  uint32_t rec;
  uint32_t s;            // log2 run length
  uint32_t K;            // runs
  uint32_t nstages;      // shared-memory stages (<= kMaxStages)
  const uint32_t* rids;
  uint64_t n_out;
  uint64_t chunk;        // rids per CTA in the distribute phases
  uint32_t* total;       // [K] run totals; zero on entry, restored to zero on exit
  uint32_t* gbar;        // [5] grid barrier (count, generation), overflow count, done
                         //     counter, dynamic run counter; persistent, zero-restored
                         //     by the kernel
  void* pairs;           // [n_out] pairs (+ slack for 16-byte bulk copies)
  uint32_t pair_bytes;
  uint8_t* dst;
  uint32_t row_bytes;
  uint32_t slot_pairs;   // pairs per stage
  uint32_t region_cap;   // bytes of a stage reserved for the run's records
  uint32_t stage_bytes;  // bytes per stage
  unsigned long long* status;
  unsigned long long* ts;  // optional [grid * 8] %globaltimer stamps (profiling), or null
  // mode 1 (three-phase, INTERNAL materialised as in Fig. 1):
  uint32_t npre;         // stages whose source run is prefetched before Phase I (0..2)
  uint32_t rid_cache;    // 1: the CTA's rid chunk is bulk-copied into shared memory
  uint32_t cap;          // fixed capacity of a run (entries); run b at [b*cap, b*cap + n_b)
  uint32_t max_own;      // runs per CTA, ceil(K / grid)
  uint32_t hist_warps;   // warps owning a private 16-bit counter per run (Phase I)
  uint32_t tile;         // rids per Phase I tile (multiple of 4, <= 65535)
  uint32_t rcache_words; // shared-memory words reserved for a cached tile (0: no cache)
  uint64_t* ovf;         // [n_out] (i | rid << 32) of entries beyond a run's capacity
  uint32_t mode;         // 0: probe writes rows straight to dst; 1: probe -> INTERNAL -> gather
  uint8_t* internal;     // [n_out * rec] INTERNAL file (mode 1)
  uint32_t* inv;         // [n_out] INTERNAL slot of output row i (mode 1)
  uint32_t n_static;     // Phase II: static runs per CTA (c + t*grid, t < n_static); the
                         // rest are claimed dynamically (gbar[4])
  uint32_t dbg;          // tuning flags (dpg_debug_flags): bit0 plain row stores (no
                         // evict_last hint), bit1 staggered run reservations,
                         // bits 8-12 static share of Phase II runs in 16ths
  OutSegs seg;           // mode 0: output segments (seg.n = 0: dst)
};

// DPG with one L2-resident run (l2run.cu).
struct L2RunArgs {
  const uint8_t* src;
  uint64_t n_src;
  uint32_t rec;
  const uint32_t* rids;
  uint64_t n_out;
  uint64_t chunk;        // output rows (and rids) per CTA
  uint8_t* dst;
  uint32_t* gbar;        // [2] grid barrier (persistent, zero-restored)
  unsigned long long* status;
  unsigned long long* ts;  // optional [grid * 16] %globaltimer stamps, or null
  uint64_t stage_bytes;  // bytes of the source staged into L2 by Phase II (0: all)
  uint32_t stage;        // 1: Phase II stages the source into L2 (then a grid barrier)
  uint32_t ring_chunk;   // Phase II bulk-copy bytes per slot (0: 32 KB)
  uint32_t ring_slots;   // Phase II ring slots (0: 6)
  const uint32_t* dev_range;  // optional [2] on the device: rows [r0, r1) (rids, dst offset by r0)
  uint32_t rd_magic;     // ceil(2^32 / (rec / 4)): dword -> row division of the gather
  uint32_t dbg;          // tuning flags (dpg_debug_flags): bit0 LSU stores of the tile,
                         // bit1 no tile store, bit2 no Phase II load, bit3 L2 prefetch first,
                         // bit16 Phase II by L2 bulk prefetches, bit17 no barrier after
                         // Phase II (only with bit16), bits 20/21 skip consume/issue
                         // (profiles/r01_l2_prefetch_staging.txt, r01_engine_probe.txt)
  OutSegs seg;           // output segments (seg.n = 0: dst); the window-gather path only
};

// DPG with two L2-resident runs (l2pair.cu).
struct L2PairArgs {
  const uint8_t* src;
  uint64_t n_src;
  uint32_t rec;
  const uint32_t* rids;
  uint64_t n_out;
  uint64_t L;            // records of run 0 (a power of two); run 1 = [L, n_src)
  uint64_t chunk;        // output rows per CTA (multiple of 32)
  uint32_t max_groups;   // ceil(chunk / 32)
  uint8_t* internal;     // INTERNAL run 0: the chunk of CTA c at internal + c*chunk*rec
  uint8_t* dst;
  uint32_t* gbar;        // [2] grid barrier (persistent, zero-restored)
  unsigned long long* status;
  unsigned long long* ts;
  uint32_t dbg;          // tuning flags: bit0 skip Phase I (timing only), bit1 no grid barrier
};

// Phase I of the K-run L2 plan (l2k.cu).
struct L2KArgs {
  const void* rids;      // uint32 or uint64 (rid_bytes)
  uint32_t rid_bytes;
  uint64_t* counts64;    // optional [K]: rows per run (CTA 0 writes)
  uint64_t n_out;
  uint64_t n_src;
  uint32_t s;            // log2 of the run length L (records)
  uint32_t K;            // runs
  uint64_t chunk;        // output rows per CTA (multiple of 32; the gather's geometry)
  uint32_t* counts;      // [K * grid] rows per (run, CTA)
  uint32_t* run_start;   // [K + 1] first slot of each run; [K] = valid rows
  uint32_t* local;       // [n_out] r - b*L, run-major
  uint32_t* inv;         // [n_out] slot of output row i (0xFFFFFFFF: bad rid)
  uint32_t* gbar;        // monotonic grid barrier words (w[0], w[32])
  unsigned long long* status;
  uint32_t hash_m;       // 0: rids; else the entries are uint32 keys, run of key k =
                         // hash slot (k * 0x9E3779B1) >> (32 - hash_m) >> s, local = k
  const uint32_t* payload;   // rids mode: local[slot] = payload[i] instead of r & (L-1)
};

// Enhanced B+-tree of the batch lookup (btree.cu): level 0 = sorted keys,
// level t = every 16th entry of level t-1, each level padded to 16 entries.
constexpr int kBtMaxLevels = 10;
struct BTreeIdx {
  const uint32_t* lv[kBtMaxLevels];
  uint32_t n[kBtMaxLevels];
  uint32_t levels;
  const uint32_t* rids;  // rid of each level-0 entry
};

// Bulk prefetch of [src, src+bytes) into L2 (no shared memory, no completion
// signal); src and bytes 16-byte aligned / multiples of 16.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes, uint64_t policy) {
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(src),
               "r"(bytes), "l"(policy)
               : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// W-byte global load / store with an L2 eviction-priority hint (W >= 4);
// narrower words fall back to plain accesses.
template <int W> struct HintIO {
  using T = typename Word<W>::T;
  static __device__ __forceinline__ T ld(const void* p, uint64_t) { return *reinterpret_cast<const T*>(p); }
  static __device__ __forceinline__ void st(void* p, T v, uint64_t) { *reinterpret_cast<T*>(p) = v; }
};
template <> struct HintIO<4> {
  static __device__ __forceinline__ uint32_t ld(const void* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
  }
  static __device__ __forceinline__ void st(void* p, uint32_t v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
  }
};
template <> struct HintIO<8> {
  static __device__ __forceinline__ uint2 ld(const void* p, uint64_t pol) {
    uint2 v;
    asm volatile("ld.global.L2::cache_hint.v2.b32 {%0, %1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
    return v;
  }
  static __device__ __forceinline__ void st(void* p, uint2 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.b32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(v.x),
                 "r"(v.y), "l"(pol) : "memory");
  }
};
template <> struct HintIO<16> {
  static __device__ __forceinline__ uint4 ld(const void* p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.L2::cache_hint.v4.b32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    return v;
  }
  static __device__ __forceinline__ void st(void* p, uint4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol) : "memory");
  }
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}

// ---------------------------------------------------------------------------
// Helpers of the L2-run kernels (l2run.cu, l2pair.cu).
// ---------------------------------------------------------------------------
// 16-byte global load under a predicate (no branch; the registers keep their
// value when off), read-only path, no L1 allocation.
__device__ __forceinline__ void ld16_pred(uint4& v, const void* p, bool on, uint64_t pol) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %4, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.L2::cache_hint.v4.b32 {%0, %1, %2, %3}, [%5], %6;\n\t}"
      : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w)
      : "r"((uint32_t)on), "l"(p), "l"(pol));
}
// 4-byte shared store under a predicate.
__device__ __forceinline__ void sts32_pred(uint32_t saddr, uint32_t v, bool on) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t"
      "@q st.shared.b32 [%0], %1;\n\t}" ::"r"(saddr), "r"(v), "r"((uint32_t)on) : "memory");
}
// Streaming 16-byte global store (evict-first).
__device__ __forceinline__ void st16_cs(void* p, uint4 v) { __stcs(reinterpret_cast<uint4*>(p), v); }

__device__ __forceinline__ uint32_t ldg_first(const uint32_t* p) {
  return __ldcs(p);   // streaming: read once
}
__device__ __forceinline__ uintptr_t al_dn(uintptr_t p) { return p & ~uintptr_t(15); }
__device__ __forceinline__ uintptr_t al_up(uintptr_t p) { return (p + 15) & ~uintptr_t(15); }

// Bulk store shared -> global (TMA), tracked by the issuing thread's bulk group.
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
               ::"l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes), "l"(pol) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// Phase II staging of [base, base + bytes) into L2 by one thread of each CTA:
// the CTA's slice (16-byte blocks) goes through a ring of NS bulk copies of CH
// bytes into shared memory with L2 evict_last; returns once every copy of the
// slice has landed (the slice is then resident in L2).  bar: NS mbarriers
// initialised with count 1.
__device__ __forceinline__ uint32_t l2_stage_slice(const uint8_t* base, uint64_t bytes, uint32_t c,
                                                   uint32_t G, uint8_t* ring, uint64_t* bar,
                                                   uint32_t CH, uint32_t NS, uint64_t pol,
                                                   uint32_t jb = 0) {
  // jb: copies issued into this ring before (the mbarrier phases continue)
  const uintptr_t s0 = al_dn(reinterpret_cast<uintptr_t>(base));
  const uintptr_t s1 = al_up(reinterpret_cast<uintptr_t>(base) + bytes);
  const uint64_t total = s1 - s0;
  const uint64_t slice = ((total + G - 1) / G + 15) & ~uint64_t(15);
  const uint64_t b0 = min_u64(total, (uint64_t)c * slice), b1 = min_u64(total, b0 + slice);
  uint32_t j = jb;
  for (uint64_t off = b0; off < b1; off += CH, ++j) {
    const uint32_t slot = j % NS;
    if (j >= NS) mbar_wait(&bar[slot], ((j / NS) - 1) & 1);
    const uint32_t nb = (uint32_t)min_u64(CH, b1 - off);
    mbar_arrive_expect_tx(&bar[slot], nb);
    bulk_g2s(ring + (size_t)slot * CH, reinterpret_cast<const void*>(s0 + off), nb, &bar[slot], pol);
  }
  for (uint32_t q = (j > jb + NS ? j - NS : jb); q < j; ++q) mbar_wait(&bar[q % NS], (q / NS) & 1);
  return j;
}

// Launchers (return cudaError_t of the launch).
cudaError_t launch_fused(const FusedArgs& a, uint32_t W, uint32_t grid, uint32_t smem,
                         cudaStream_t st, uint32_t* nlaunch);
cudaError_t launch_l2run(const L2RunArgs& a, uint32_t W, uint32_t grid, cudaStream_t st,
                         uint32_t* nlaunch);
uint32_t l2run_smem_bytes(uint64_t chunk_rids);
cudaError_t launch_l2pair(const L2PairArgs& a, uint32_t grid, cudaStream_t st, uint32_t* nlaunch);
cudaError_t launch_l2k_distribute(const L2KArgs& a, uint32_t grid, cudaStream_t st, uint32_t* nlaunch);
uint32_t l2k_smem_bytes(uint32_t K);
cudaError_t launch_sort_rids(const uint8_t* src, uint32_t rec, uint64_t n, uint32_t key_off,
                             uint32_t key_bytes, uint8_t* ws, uint32_t* rids_out, uint32_t* gbar,
                             int sm, cudaStream_t st, uint32_t* nlaunch,
                             const uint32_t* keys_u32 = nullptr, uint32_t* keys_out = nullptr,
                             uint64_t key_limit = ~0ull, unsigned long long* status = nullptr);
// Batch lookup in a hash index (hash.cu).
cudaError_t launch_hash_direct(const void* table, uint32_t m, const void* pool, const uint32_t* keys,
                               uint64_t n, uint32_t* out, int sm, cudaStream_t st, uint32_t* nl);
cudaError_t launch_gather_u32(const uint32_t* tmp, const uint32_t* inv, uint64_t n, uint32_t* out,
                              int sm, cudaStream_t st, uint32_t* nl);
cudaError_t launch_hash_probe(const void* table, uint32_t m, uint32_t s, uint32_t K, const void* pool,
                              const uint32_t* qkeys, const uint32_t* run_start, uint32_t* tmp,
                              uint32_t* gbar, int sm, cudaStream_t st, uint32_t* nl,
                              const uint32_t* counts = nullptr, uint32_t cap = 0);
cudaError_t launch_hash_distribute(const uint32_t* keys, uint64_t n, uint32_t m, uint32_t s, uint32_t K,
                                   uint32_t cap, uint32_t* cursor, uint32_t* qkeys, uint32_t* inv,
                                   uint64_t* ovf, uint32_t* n_ovf, int sm, cudaStream_t st,
                                   uint32_t* nl);
cudaError_t launch_hash_overflow(const void* table, uint32_t m, const void* pool, const uint64_t* ovf,
                                 const uint32_t* n_ovf, uint32_t* out, int sm, cudaStream_t st,
                                 uint32_t* nl);

// Batch lookup in an enhanced B+-tree (btree.cu).
cudaError_t launch_bt_direct(const BTreeIdx& T, const uint32_t* keys, uint64_t n, uint32_t* out,
                             int sm, cudaStream_t st, uint32_t* nl);
cudaError_t launch_bt_top(const BTreeIdx& T, uint32_t stop, uint32_t shift, const uint32_t* keys,
                          uint64_t n, uint32_t* run, int sm, cudaStream_t st, uint32_t* nl);
cudaError_t launch_bt_probe(const BTreeIdx& T, uint32_t K, uint32_t s, uint32_t stop,
                            const uint32_t* qkeys, const uint32_t* run_start, uint32_t* tmp,
                            uint32_t* gbar, int sm, cudaStream_t st, uint32_t* nl);

// Launch count of the last call on this host thread (api.cu).
uint32_t t_launches_get();
void t_launches_set(uint32_t n);

// Data skew check (skew.cu): estimated rids beyond the fixed run
// capacity from S evenly spaced samples; hist: ceil(K / group) zeroed words.
cudaError_t launch_skew_check(const uint32_t* rids, uint64_t n_out, uint64_t n_src, uint32_t s,
                              uint32_t K, uint32_t cap, uint32_t S, uint32_t* hist,
                              unsigned long long* out, cudaStream_t st, uint32_t* nl);
// Run boundaries from a sorted sample of S <= 32768 rids (skew.cu, reading
// A23): bounds[0..*n_runs] (room for K + 1), one CTA.
constexpr uint32_t kSkewMaxSample = 32768;
cudaError_t launch_skew_partition(const uint32_t* rids, uint64_t n_out, uint32_t n_src, uint32_t K,
                                  uint32_t S, uint64_t seed, uint32_t* bounds, uint32_t* n_runs,
                                  cudaStream_t st, uint32_t* nl);
cudaError_t launch_zip_gather(const uint8_t* a, uint32_t a_bytes, const uint8_t* b, uint32_t b_bytes,
                              uint64_t n_b, const uint32_t* idx, uint64_t n, uint8_t* out, uint32_t W,
                              int sm, cudaStream_t st, uint32_t* nlaunch,
                              unsigned long long* status = nullptr);
uint64_t sort_ws_bytes(uint64_t n, int sm);
uint32_t l2pair_smem_bytes(uint64_t chunk);
cudaError_t launch_distribute(const DistArgs& a, bool rid64, cudaStream_t st, uint32_t* nlaunch);
// Steps (1)-(2) of the distribute alone (32-bit rids): per-chunk run counts
// and their run-major exclusive scan (partials: count_scan_partials words
// past run_start[K]).
cudaError_t launch_count_scan(const DistArgs& a, cudaStream_t st, uint32_t* nlaunch);
uint32_t count_scan_partials(uint64_t K, uint64_t G);

// DPG in three sequential passes over shared-memory runs (seq3.cu, path 6),
// intermediates stored tile by tile (see seq3.cu).
struct Seq3Args {
  const uint8_t* src;      // n_src records of rec bytes (16-byte aligned)
  uint64_t n_src;
  uint32_t rec;
  const uint32_t* rids;    // n_out rids
  uint64_t n_out;
  uint32_t s;              // run length L = 2^s records (L * rec <= one stage)
  uint32_t K;              // runs
  uint32_t T;              // rids per tile (multiple of 16, <= 32768)
  uint32_t nsub;           // tiles = ceil(n_out / T)
  uint16_t* pre;           // [nsub][K+1] exclusive run prefix of each tile
  uint16_t* preT;          // [K+1][nsub] its transpose
  uint16_t* loc;           // RID_RUN, tile by tile: [nsub * T] local offsets
  uint16_t* tinv;          // [n_out] slot of row i inside its tile (0xFFFF: invalid rid)
  uint64_t* dbg_pairs;     // tests only: (local | i << 32) per RID_RUN slot
  uint8_t* internal;       // INTERNAL, tile by tile: [nsub * T * rec]
  uint8_t* dst;            // n_out rows of pay_bytes + rec
  const uint8_t* pay;      // join: n_out payload rows (pay_bytes each), or null
  uint32_t pay_bytes;
  unsigned long long* status;
  uint32_t dbg;            // tuning experiments only (dpg_debug_flags): 0 normally
  unsigned long long* ts;  // profiling only (dpg_debug_phase_stamps): per-CTA stamps
  uint32_t cl;             // Phase II: CTAs of a cluster holding one run (1, 2, 4, 8)
};
uint32_t seq3_dist_smem(uint32_t T, uint32_t K);
uint32_t seq3_probe_smem(uint64_t stage_bytes);
uint32_t seq3_gather_smem(uint32_t T, uint32_t rec, uint32_t nbuf);
cudaError_t launch_seq3_distribute(const Seq3Args& a, uint32_t grid, cudaStream_t st,
                                   uint32_t* nlaunch);
cudaError_t launch_seq3_probe(const Seq3Args& a, uint32_t W, uint32_t grid, cudaStream_t st,
                              uint32_t* nlaunch);
cudaError_t launch_seq3_gather(const Seq3Args& a, uint32_t W, uint32_t grid, uint32_t nbuf,
                               cudaStream_t st, uint32_t* nlaunch);
// Phase I of the multi-kernel plan as stable radix passes over rid >> s
// (sort.cu): out[n] = (rid << 32) | position by run, run_start[K+1].
uint32_t radix_passes(uint64_t K);
cudaError_t launch_radix_distribute(const uint32_t* rids, uint64_t n, uint64_t n_src, uint32_t s,
                                    uint32_t K, uint64_t* tmp, uint64_t* out, uint32_t* counts,
                                    uint32_t* gbar, uint32_t* run_start, int sm, cudaStream_t st,
                                    uint32_t* nl, unsigned long long* status);
cudaError_t launch_radix_unpack(const uint64_t* e, uint64_t n, uint32_t s, const uint32_t* rs,
                                uint32_t K, uint64_t* out, uint64_t* rs_out, cudaStream_t st,
                                uint32_t* nl);
// Pair chunks of the runs as work items (distribute.cu): item_cnt[K] and
// partial[count_scan_partials(K, 1)] scratch, item_start[K+1], item_run[4 x
// (up to K + n_out / sp)] (16-byte aligned: uint4 {run, chunk, p0, p1} per item).
cudaError_t launch_items(const uint32_t* run_start, uint32_t K, uint32_t sp, uint32_t* item_cnt,
                         uint32_t* partial, uint32_t* item_start, uint32_t* item_run,
                         cudaStream_t st, uint32_t* nl);
cudaError_t launch_probe_gather(const ProbeArgs& a, uint32_t W, uint32_t grid, uint32_t smem,
                                cudaStream_t st, uint32_t* nlaunch);
cudaError_t launch_direct(const uint8_t* src, uint64_t n_src, uint32_t rec, const uint32_t* rids,
                          uint64_t n_out, uint8_t* dst, uint32_t W, int sm_count,
                          unsigned long long* status, cudaStream_t st, uint32_t* nlaunch,
                          int hint = 0);
cudaError_t launch_l2_prefetch(const void* p, uint64_t bytes, int sm_count, cudaStream_t st,
                               uint32_t* nlaunch);
cudaError_t launch_zip_rows(const uint8_t* a, uint32_t a_bytes, const uint8_t* b, uint32_t b_bytes,
                            uint64_t n, uint8_t* out, uint32_t W, int sm_count, cudaStream_t st,
                            uint32_t* nlaunch, const uint32_t* key = nullptr,
                            uint64_t key_limit = 0);
cudaError_t launch_scatter_rows(const uint8_t* rows, uint32_t rec, const uint32_t* pos,
                                uint64_t n, uint8_t* dst, uint64_t n_dst, uint32_t W,
                                int sm_count, cudaStream_t st, uint32_t* nlaunch);
cudaError_t launch_split_entries(const DistArgs& a, uint32_t* local_out, uint32_t* pos_out,
                                 uint64_t* counts, cudaStream_t st, uint32_t* nlaunch);
cudaError_t launch_unpack_pairs(const DistArgs& a, uint64_t* pairs_out, uint64_t* run_start_out,
                                cudaStream_t st, uint32_t* nlaunch);

}  // namespace dpg

namespace dpg {

// ---------------------------------------------------------------------------
// Asynchronous window gather (l2pair.cu, l2run.cu): a warp moves groups of up
// to 32 rows of rec bytes (rec % 4 == 0, rec <= 116) from arbitrary 4-byte
// aligned source addresses to a contiguous output span.  Issue: each row's
// enclosing 16-byte-aligned window (<= 8 words) is copied by cp.async (16 B
// per lane, L2 only) into the group's tile in shared memory (row pitch
// 128 B); several groups are in flight per warp without holding registers.
// Consume: output dword d of the group is row d / RD, dword d % RD, read from
// the tile at the row's dword shift, and stored with coalesced 4-byte
// streaming stores (any 4-byte-aligned output).
// ---------------------------------------------------------------------------
constexpr uint32_t kAgTile = 32 * 128;   // bytes of one group's window tile

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// lane j of the warp holds row j's source address (my_addr) and whether the
// row is to be copied (my_on); rows >= cnt are off.
__device__ __forceinline__ void ag_issue(uint32_t tile_s, uint64_t my_addr, bool my_on, uint32_t rec,
                                         uint32_t lane) {
  const uint32_t FNW = (rec + 27) / 16;
  const uint32_t FRPI = 32 / FNW, flr = lane / FNW, flw = lane % FNW;
  const uint32_t lim = rec - 16 * flw;     // word flw is needed iff (addr & 15) + rec > 16 flw
  uint32_t jj = flr;
  uint32_t so = tile_s + flr * 128 + 16 * flw;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const uint32_t j = jj & 31;
    const uint32_t lo32 = __shfl_sync(0xffffffffu, (uint32_t)my_addr, j);
    const uint32_t hi32 = __shfl_sync(0xffffffffu, (uint32_t)(my_addr >> 32), j);
    const uint32_t on_j = __shfl_sync(0xffffffffu, (uint32_t)my_on, j);
    const bool on = on_j && flr < FRPI && jj < 32 && (int)(lo32 & 15) + (int)lim > 0;
    if (on)   // the window words a row needs; the consume step reads no others
      cp_async16(so, reinterpret_cast<const void*>(((((uint64_t)hi32 << 32) | lo32) & ~uint64_t(15)) +
                                                  16 * flw), 16u);
    jj += FRPI;
    so += FRPI * 128;
  }
}

// my_o4: row lane's dword shift inside its window ((addr >> 2) & 3);
// okm: rows to store; out: 4-byte aligned.
__device__ __forceinline__ void ag_consume(const uint32_t* tile, uint32_t my_o4, uint32_t okm,
                                           uint32_t cnt, uint32_t rec, uint32_t* out,
                                           uint32_t lane) {
  const uint32_t RD = rec >> 2;
  const uint32_t n = cnt * RD;
  const uint32_t q32 = 32 / RD, r32 = 32 % RD;
  uint32_t j = lane / RD, q = lane % RD;
  for (uint32_t d0 = 0; d0 < n; d0 += 32) {
    const uint32_t d = d0 + lane;
    const uint32_t jj = j < 32 ? j : 31;
    const uint32_t s = __shfl_sync(0xffffffffu, my_o4, jj);
    if (d < n && ((okm >> jj) & 1)) __stcs(out + d, tile[jj * 32 + s + q]);
    j += q32;
    q += r32;
    if (q >= RD) { q -= RD; ++j; }
  }
}

}  // namespace dpg

namespace dpg {
// ag_consume with 16-byte output words (4x fewer global store instructions):
// out 16-byte aligned and cnt * rec a multiple of 16.  The word -> (row,
// dword) map of a full group is per-lane constant: AgMap holds it for the
// lane's words m = lane + 32 i (i < 8, rec <= 116 gives <= 232 words).
struct AgMap {
  uint32_t b0[8];     // tile dword index of the word's first dword in row j0, before the shift
  uint32_t b1[8];     // same for the next row (j0 + 1), minus RD
  uint32_t jp[8];     // j0 | (j0 + 1) << 8 | split << 16 (dwords e < split are row j0's)
};
__device__ __forceinline__ void ag_map_init(AgMap& M, uint32_t rec, uint32_t lane) {
  const uint32_t RD = rec >> 2;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t d0 = 4 * (lane + 32 * i);
    const uint32_t j0 = min(d0 / RD, 31u);
    const uint32_t q0 = d0 - j0 * RD;
    const uint32_t j1 = min(j0 + 1, 31u);
    M.b0[i] = j0 * 32 + q0;
    M.b1[i] = j1 * 32 + q0 - RD;
    M.jp[i] = j0 | (j1 << 8) | (min(RD - min(q0, RD), 4u) << 16);
  }
}
__device__ __forceinline__ void ag_consume16(const uint32_t* tile, uint32_t my_o4, const AgMap& M,
                                             uint32_t cnt, uint32_t rec, uint32_t* out,
                                             uint32_t lane) {
  const uint32_t nw = cnt * (rec >> 2) / 4;         // 16-byte output words
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (32 * i >= nw) break;                        // warp-uniform
    const uint32_t m = lane + 32 * i;
    const uint32_t jp = M.jp[i];
    const uint32_t s0 = __shfl_sync(0xffffffffu, my_o4, jp & 31);
    const uint32_t s1 = __shfl_sync(0xffffffffu, my_o4, (jp >> 8) & 31);
    const uint32_t split = jp >> 16;
    const uint32_t a0 = M.b0[i] + s0, a1 = M.b1[i] + s1;
    uint4 v;
    v.x = tile[a0];                                  // split >= 1
    v.y = tile[1 < split ? a0 + 1 : a1 + 1];
    v.z = tile[2 < split ? a0 + 2 : a1 + 2];
    v.w = tile[3 < split ? a0 + 3 : a1 + 3];
    if (m < nw) __stcs(reinterpret_cast<uint4*>(out) + m, v);
  }
}
}  // namespace dpg

namespace dpg {
// One group of the asynchronous window gather: lane j's row j.
struct AgGroup {
  uint64_t addr;      // source address of the lane's row
  uint32_t cnt;       // rows in the group (<= 32)
  uint32_t okm;       // rows to store (a bad rid leaves its row unwritten)
  uint32_t o4;        // the lane's row: dword shift inside its window
  uint32_t* out;      // the group's output span (cnt * rec bytes, 4-byte aligned)
  bool on;            // the lane's row is copied
};

// Run the window gather over a warp's groups t = 0 .. nt-1 (group(t) builds
// the descriptor of group t, called in order): groups t+1 and t+2 are in
// flight (cp.async into three tiles of tile_bytes) while t is consumed; the
// descriptors rotate through registers.
template <typename F>
__device__ __forceinline__ void ag_pipeline(uint32_t nt, F group, uint8_t* wtiles, uint32_t wt_s,
                                            uint32_t tile_bytes, const AgMap& amap, uint32_t rec,
                                            uint32_t lane) {
  AgGroup q0{}, q1{}, q2{};
  if (0 < nt) { q0 = group(0); ag_issue(wt_s, q0.addr, q0.on, rec, lane); }
  cp_async_commit();
  if (1 < nt) { q1 = group(1); ag_issue(wt_s + tile_bytes, q1.addr, q1.on, rec, lane); }
  cp_async_commit();
  uint32_t slot = 0;
  for (uint32_t t = 0; t < nt; ++t) {
    const uint32_t slot2 = slot == 0 ? 2 : slot - 1;
    if (t + 2 < nt) { q2 = group(t + 2); ag_issue(wt_s + slot2 * tile_bytes, q2.addr, q2.on, rec, lane); }
    cp_async_commit();
    cp_async_wait<2>();
    __syncwarp();
    const uint32_t* wt = reinterpret_cast<const uint32_t*>(wtiles + slot * tile_bytes);
    const uint32_t full = q0.cnt == 32 ? 0xffffffffu : ((1u << q0.cnt) - 1u);
    if (q0.okm == full && ((reinterpret_cast<uintptr_t>(q0.out) | (q0.cnt * rec)) & 15) == 0)
      ag_consume16(wt, q0.o4, amap, q0.cnt, rec, q0.out, lane);
    else
      ag_consume(wt, q0.o4, q0.okm, q0.cnt, rec, q0.out, lane);
    __syncwarp();
    q0 = q1;
    q1 = q2;
    slot = slot == 2 ? 0 : slot + 1;
  }
  cp_async_wait<0>();
}
}  // namespace dpg

namespace dpg {
// ---------------------------------------------------------------------------
// Row-index window gather (l2run.cu): the same asynchronous window gather
// with one source base for the whole warp.  A group is described by each
// lane's 32-bit row index (~0u: row not copied) instead of a 64-bit address,
// so issuing a window word costs one shuffle and, when the source spans less
// than 4 GB (OFF32), 32-bit offset arithmetic; the lane constants of issue
// and consume are computed once per warp (byte addresses inside the tile),
// and the consume step reads the dword shifts of rows j and j + 1 with one
// shuffle of a packed value.
// ---------------------------------------------------------------------------
struct AgrLane {
  uintptr_t wbase;    // (base & ~15) + the lane's window word offset
  uint32_t bl;        // base & 15
  uint32_t frpi;      // rows per issue instruction (32 / window words)
  uint32_t flr;       // the lane's row inside an instruction (>= frpi: idle lane)
  int32_t lim;        // word flw is needed iff (addr & 15) + lim > 0
  uint32_t so0;       // the lane's byte offset inside a tile
};
__device__ __forceinline__ AgrLane agr_lane(uintptr_t base, uint32_t rec, uint32_t lane) {
  AgrLane L;
  const uint32_t fnw = (rec + 27) / 16;
  L.frpi = 32 / fnw;
  L.flr = lane / fnw;
  const uint32_t flw = lane - L.flr * fnw;
  L.wbase = (base & ~uintptr_t(15)) + 16 * flw;
  L.bl = (uint32_t)base & 15u;
  L.lim = (int32_t)rec - (int32_t)(16 * flw);
  L.so0 = L.flr * 128 + 16 * flw;
  return L;
}
template <bool OFF32>
__device__ __forceinline__ void agr_issue(uint32_t tile_s, uint32_t rec, uint32_t my_r, const AgrLane& L) {
  uint32_t j = L.flr;
  uint32_t so = tile_s + L.so0;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    if ((uint32_t)u * L.frpi >= 32) break;            // warp-uniform
    const uint32_t r = __shfl_sync(0xffffffffu, my_r, j & 31);
    if (OFF32) {
      const uint32_t x = L.bl + r * rec;               // offset from base & ~15
      if (j < 32 && (int32_t)(x & 15u) + L.lim > 0)
        cp_async16(so, reinterpret_cast<const void*>(L.wbase + (x & ~15u)), 16u);
    } else {
      const uint64_t x = L.bl + (uint64_t)r * rec;
      if (j < 32 && (int32_t)((uint32_t)x & 15u) + L.lim > 0)
        cp_async16(so, reinterpret_cast<const void*>(L.wbase + (x & ~uint64_t(15))), 16u);
    }
    j += L.frpi;
    so += L.frpi * 128;
  }
}
// Consume map of a full group, per lane: output word m = lane + 32 i reads
// dwords of row j0 (byte b0 in the tile before the row's shift) and, from
// dword `split` on, of row j0 + 1 (b1, minus the row length).
struct AgrMap {
  uint32_t b0[8];
  uint32_t b1[8];
  uint32_t jp[8];     // j0 | split << 8
};
__device__ __forceinline__ void agr_map_init(AgrMap& M, uint32_t rec, uint32_t lane) {
  const uint32_t RD = rec >> 2;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t d0 = 4 * (lane + 32 * i);
    const uint32_t j0 = min(d0 / RD, 31u);
    const uint32_t q0 = d0 - j0 * RD;
    const uint32_t j1 = min(j0 + 1, 31u);
    const bool in = d0 < 32 * RD;                   // words past a full group read the tile start
    M.b0[i] = in ? 4 * (j0 * 32 + q0) : 0u;
    M.b1[i] = in ? 4 * (j1 * 32 + q0 - RD) : 0u;
    M.jp[i] = in ? j0 | (min(RD - q0, 4u) << 8) : 4u << 8;
  }
}
// packed (lane j): bits 0-15 = 4 x dword shift of row j, bits 16-31 = of row j + 1.
// The loads of a batch of four output words are written before its stores:
// the streaming store is a compiler memory barrier, so this order is what
// lets the shuffles and shared loads of a batch overlap.  Every map entry
// addresses the tile, so the batch needs no guard; the stores are predicated.
__device__ __forceinline__ void agr_consume16(const uint8_t* tile, uint32_t packed, const AgrMap& M,
                                              uint32_t cnt, uint32_t rec, uint32_t* out,
                                              uint32_t lane) {
  const uint32_t nw = cnt * (rec >> 2) / 4;         // 16-byte output words
  uint4* o = reinterpret_cast<uint4*>(out) + lane;
#pragma unroll
  for (int h = 0; h < 8; h += 4) {
    if (32 * h >= nw) break;                        // warp-uniform
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t jp = M.jp[h + k];
      const uint32_t s = __shfl_sync(0xffffffffu, packed, jp & 31);
      const uint32_t split = jp >> 8;
      const uint8_t* r0 = tile + M.b0[h + k] + (s & 0xffffu);
      const uint8_t* r1 = tile + M.b1[h + k] + (s >> 16);
      v[k].x = *reinterpret_cast<const uint32_t*>(r0);
      v[k].y = *reinterpret_cast<const uint32_t*>((1 < split ? r0 : r1) + 4);
      v[k].z = *reinterpret_cast<const uint32_t*>((2 < split ? r0 : r1) + 8);
      v[k].w = *reinterpret_cast<const uint32_t*>((3 < split ? r0 : r1) + 12);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (lane + 32 * (h + k) < nw) __stcs(o + 32 * (h + k), v[k]);
  }
}
struct AgrGroup {
  uint32_t r;         // the lane's row index (a row not stored reads row 0)
  uint32_t cnt;       // rows in the group (<= 32)
  uint32_t okm;       // rows to store
  uint32_t* out;      // the group's output span (nullptr: rows go to several output segments)
  uint64_t g0;        // the group's first output row (for split)
};
// Three groups per warp in flight, as ag_pipeline.  OFF32: every row offset
// (base & 15) + r * rec of the source fits in 32 bits.  A group whose rows
// belong to several output segments (out == nullptr) is stored by
// split(group, tile, lane's dword shift).
template <bool OFF32, typename F, typename S>
__device__ __forceinline__ void agr_pipeline(uint32_t nt, F group, S split, uint8_t* wtiles, uint32_t wt_s,
                                             uint32_t tile_bytes, const AgrMap& amap, uintptr_t base,
                                             uint32_t rec, uint32_t lane, uint32_t dbg = 0) {
  // dbg (experiments, tools/engine_probe.py): bit 20 skips the consume step,
  // bit 21 the issue step (the output is then wrong)
  const bool no_consume = dbg & (1u << 20), no_issue = dbg & (1u << 21);
  const AgrLane L = agr_lane(base, rec, lane);
  AgrGroup q0{}, q1{}, q2{};
  if (0 < nt) { q0 = group(0); if (!no_issue) agr_issue<OFF32>(wt_s, rec, q0.r, L); }
  cp_async_commit();
  if (1 < nt) { q1 = group(1); if (!no_issue) agr_issue<OFF32>(wt_s + tile_bytes, rec, q1.r, L); }
  cp_async_commit();
  uint32_t slot = 0;
  for (uint32_t t = 0; t < nt; ++t) {
    const uint32_t slot2 = slot == 0 ? 2 : slot - 1;
    if (t + 2 < nt) {
      q2 = group(t + 2);
      if (!no_issue) agr_issue<OFF32>(wt_s + slot2 * tile_bytes, rec, q2.r, L);
    }
    cp_async_commit();
    const uint32_t o4 = (L.bl + q0.r * rec) >> 2 & 3u;   // (base + r*rec) >> 2 & 3
    const uint32_t nx = __shfl_down_sync(0xffffffffu, o4, 1);
    cp_async_wait<2>();
    __syncwarp();
    const uint8_t* ts = wtiles + slot * tile_bytes;
    const uint32_t full = q0.cnt == 32 ? 0xffffffffu : ((1u << q0.cnt) - 1u);
    if (no_consume) {
    } else if (!q0.out) {
      split(q0, reinterpret_cast<const uint32_t*>(ts), o4);
    } else if (q0.okm == full && ((reinterpret_cast<uintptr_t>(q0.out) | (q0.cnt * rec)) & 15) == 0)
      agr_consume16(ts, (o4 << 2) | (nx << 18), amap, q0.cnt, rec, q0.out, lane);
    else
      ag_consume(reinterpret_cast<const uint32_t*>(wtiles + slot * tile_bytes), o4, q0.okm, q0.cnt,
                 rec, q0.out, lane);
    __syncwarp();
    q0 = q1;
    q1 = q2;
    slot = slot == 2 ? 0 : slot + 1;
  }
  cp_async_wait<0>();
}

// Launch `k` with programmatic stream serialisation (PDL, see pdl_wait) when
// `pdl`, on clusters of `cluster` CTAs when > 1.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, uint32_t smem,
                              cudaStream_t st, bool pdl, uint32_t cluster, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[2];
  unsigned n = 0;
  if (pdl) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}
}  // namespace dpg
