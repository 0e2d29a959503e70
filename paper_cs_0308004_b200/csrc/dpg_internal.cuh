// dpg_internal.cuh -- device helpers and launcher declarations shared by the
// CUDA translation units of libdpg.so (product path; no oracle code here).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dpg.h"

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
    const uint32_t gen = ld_acquire_gpu(gbar + 1);
    __threadfence();
    if (atomicAdd(gbar, 1u) == G - 1) {
      atomicExch(gbar, 0u);
      __threadfence();
      atomicAdd(gbar + 1, 1u);
    } else {
      while (ld_acquire_gpu(gbar + 1) == gen) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
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
};

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
  uint32_t rd_magic;     // ceil(2^32 / (rec / 4)): dword -> row division of the gather
  uint32_t dbg;          // tuning flags (dpg_debug_flags): bit0 LSU stores of the tile,
                         // bit1 no tile store, bit2 no Phase II load, bit3 L2 prefetch first
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
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Launchers (return cudaError_t of the launch).
cudaError_t launch_fused(const FusedArgs& a, uint32_t W, uint32_t grid, uint32_t smem,
                         cudaStream_t st, uint32_t* nlaunch);
cudaError_t launch_l2run(const L2RunArgs& a, uint32_t W, uint32_t grid, cudaStream_t st,
                         uint32_t* nlaunch);
uint32_t l2run_smem_bytes(uint64_t chunk_rids);
cudaError_t launch_distribute(const DistArgs& a, bool rid64, cudaStream_t st, uint32_t* nlaunch);
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
                            uint32_t* nlaunch);
cudaError_t launch_scatter_rows(const uint8_t* rows, uint32_t rec, const uint32_t* pos,
                                uint64_t n, uint8_t* dst, uint64_t n_dst, uint32_t W,
                                int sm_count, cudaStream_t st, uint32_t* nlaunch);
cudaError_t launch_split_entries(const DistArgs& a, uint32_t* local_out, uint32_t* pos_out,
                                 uint64_t* counts, cudaStream_t st, uint32_t* nlaunch);
cudaError_t launch_unpack_pairs(const DistArgs& a, uint64_t* pairs_out, uint64_t* run_start_out,
                                cudaStream_t st, uint32_t* nlaunch);

}  // namespace dpg
