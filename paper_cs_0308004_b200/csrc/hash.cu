// hash.cu -- batch lookup of keys in a hash index with DPG (section 4,
// "Batch Lookup in Hash Indexes").
//
// The index (built by the caller; datagen/gen.c builds the test inputs): a
// primary array of M = 2^m slots and an overflow pool, 16-byte entries
// {key, rid, next, 0}; key k lives in slot h(k) = (k * 0x9E3779B1) >> (32 - m)
// or in the chain of pool entries linked from it ("a second hash array ...
// stores pointers to overflow key-rid pairs"); rid 0xFFFFFFFF
// marks an empty slot, next 0xFFFFFFFF the end of a chain.
//
//   direct     k_hash_direct: each query reads its slot (a random 16-byte
//              access into the array) and walks the chain -- the lookup the
//              paper calls uneconomical when the index does not fit in cache.
//   DPG        "The hash array is partitioned into sets of L hash slots.  In
//              the distribute phase, the hash value acts as an index into the
//              hash array":
//     Phase I   the keys are distributed into runs by partition (h >> s) --
//               k_l2k_distribute in hash mode: run-major keys + each query's
//               slot in the run order (inv);
//     Phase II  k_hash_probe, one cooperative kernel over all runs: run b's
//               partition of the hash array is staged into the L2 (the cache
//               of this design, reading A17; TMA bulk copies, evict_last), a
//               grid barrier, then every key of run b looks up its slot (an
//               L2 hit) and its chain; the rids go to a temporary partition
//               in run order ("saved in a temporary partition, in the same
//               order ...");
//     Phase III dpg_gather_rows: out[i] = tmp[inv[i]] in query order.
#include "dpg_internal.cuh"

namespace dpg {

static constexpr int kHThreads = 512;
static constexpr uint32_t kNotFound = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t hslot(uint32_t key, uint32_t m) {
  return (uint32_t)(key * 0x9E3779B1u) >> (32 - m);
}

// The rest of a lookup once the key's slot s has been read.
__device__ __forceinline__ uint32_t hash_chain(uint4 s, uint32_t key, const uint4* __restrict__ pool) {
  if (s.y == kNotFound) return kNotFound;               // empty slot: no chain either
  if (s.x == key) return s.y;
  for (uint32_t nx = s.z; nx != kNotFound;) {
    const uint4 p = __ldg(pool + nx);
    if (p.x == key) return p.y;
    nx = p.z;
  }
  return kNotFound;
}

__global__ void __launch_bounds__(256) k_hash_direct(const uint4* __restrict__ table, uint32_t m,
                                                      const uint4* __restrict__ pool,
                                                      const uint32_t* __restrict__ keys, uint64_t n,
                                                      uint32_t* __restrict__ out) {
  constexpr int U = 4;                                  // slot loads in flight per thread
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    uint32_t k[U];
    uint4 s[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = i0 + u * stride;
      k[u] = i < n ? __ldcs(keys + i) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < n) s[u] = __ldg(table + hslot(k[u], m));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < n) __stcs(out + i, hash_chain(s[u], k[u], pool));
    }
  }
}

struct HashProbeArgs {
  const uint4* table;
  uint32_t m;              // log2 slots
  uint32_t s;              // log2 slots per partition (run)
  uint32_t K;              // runs
  const uint4* pool;
  const uint32_t* qkeys;   // keys, run-major (Phase I)
  const uint32_t* run_start;   // [K + 1]
  uint32_t* tmp;           // rids, run-major
  uint32_t* gbar;          // grid barrier words (count, generation; zero-restored)
  const uint32_t* counts;  // fixed-capacity layout: run b at [b*cap, b*cap + min(counts[b], cap))
  uint32_t cap;            //   (counts == nullptr: run b at [run_start[b], run_start[b+1]))
};

// Phase II over all runs.  Lane 0 of warp 0 of every CTA streams its slice
// of partition b into the L2 through a shared-memory ring; the grid barrier
// makes the partition resident for everyone; then the CTA looks up its share
// of run b's keys.  The next run's staging follows without a second barrier.
__global__ void __launch_bounds__(kHThreads, 1) k_hash_probe(HashProbeArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  uint8_t* ring = smem + 128;
  constexpr uint32_t CH = 32u << 10, NS = 4;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t c = blockIdx.x, G = gridDim.x;
  if (tid == 0) {
    for (uint32_t q = 0; q < NS; ++q) mbar_init(&bar[q], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = policy_evict_last();
  const uint64_t L = 1ull << a.s;
  uint32_t jring = 0;
  for (uint32_t b = 0; b < a.K; ++b) {
    if (warp == 0) {
      if (lane == 0)
        jring = l2_stage_slice(reinterpret_cast<const uint8_t*>(a.table + b * L), L * 16, c, G, ring,
                               bar, CH, NS, pol, jring);
      __syncwarp();
    }
    grid_barrier(a.gbar, G);
    uint64_t e0, e1;
    if (a.counts) {
      e0 = (uint64_t)b * a.cap;
      e1 = e0 + min(__ldcg(a.counts + b), a.cap);
    } else {
      e0 = __ldg(a.run_start + b);
      e1 = __ldg(a.run_start + b + 1);
    }
    const uint64_t per = ((e1 - e0 + G - 1) / G + 31) & ~uint64_t(31);
    const uint64_t lo = min_u64(e1, e0 + (uint64_t)c * per), hi = min_u64(e1, lo + per);
    constexpr int U = 16;     // keys in flight per thread (the probe is latency-bound)
    for (uint64_t e = lo + tid; e < hi; e += U * kHThreads) {
      uint32_t k[U];
      uint4 sl[U];
#pragma unroll
      for (int u = 0; u < U; ++u) k[u] = e + u * kHThreads < hi ? __ldcs(a.qkeys + e + u * kHThreads) : 0u;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (e + u * kHThreads < hi) sl[u] = __ldcg(a.table + hslot(k[u], a.m));
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (e + u * kHThreads < hi) __stcg(a.tmp + e + u * kHThreads, hash_chain(sl[u], k[u], a.pool));
    }
  }
}

// Phase III of the batch lookup: out[i] = tmp[inv[i]] (4-byte words; inv
// in range by construction).  Eight lookups in flight per thread: the reads
// of tmp are K interleaved sequential streams (one per run), L2-served.
__global__ void __launch_bounds__(256) k_gather_u32(const uint32_t* __restrict__ tmp,
                                                     const uint32_t* __restrict__ inv, uint64_t n,
                                                     uint32_t* __restrict__ out) {
  constexpr int U = 8;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    uint32_t j[U], v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) j[u] = i0 + u * stride < n ? __ldcs(inv + i0 + u * stride) : 0u;
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = i0 + u * stride < n && j[u] != kNotFound ? __ldcg(tmp + j[u]) : 0u;
#pragma unroll
    for (int u = 0; u < U; ++u)   // (inv = 0xFFFFFFFF: an overflow key, looked up directly)
      if (i0 + u * stride < n && j[u] != kNotFound) __stcs(out + i0 + u * stride, v[u]);
  }
}

// Phase I in one pass (the hash spreads the keys evenly over the partitions,
// so every run gets a fixed capacity): per tile of 8192 keys (16 per thread,
// read once) a shared-memory rank inside (tile, run), one global reservation
// per (tile, run), and each key written at b*cap + base + rank with its slot
// in inv; a key beyond its run's capacity goes to an overflow list (looked up
// directly after Phase III).
static constexpr int kHdKpt = 16;
__global__ void __launch_bounds__(kHThreads, 1) k_hash_distribute(
    const uint32_t* __restrict__ keys, uint64_t n, uint64_t chunk, uint32_t m, uint32_t s, uint32_t K,
    uint32_t cap, uint32_t* __restrict__ cursor, uint32_t* __restrict__ qkeys, uint32_t* __restrict__ inv,
    uint64_t* __restrict__ ovf, uint32_t* __restrict__ n_ovf) {
  __shared__ uint32_t cnt[512], base[512];
  const int tid = threadIdx.x;
  const uint64_t lo = min_u64(n, (uint64_t)blockIdx.x * chunk), hi = min_u64(n, lo + chunk);
  for (uint64_t t0 = lo; t0 < hi; t0 += kHThreads * kHdKpt) {
    for (uint32_t b = tid; b < K; b += kHThreads) cnt[b] = 0;
    __syncthreads();
    uint32_t k[kHdKpt], rk[kHdKpt];
#pragma unroll
    for (int u = 0; u < kHdKpt; ++u) {
      const uint64_t i = t0 + (uint64_t)u * kHThreads + tid;
      k[u] = i < hi ? __ldcs(keys + i) : 0u;
    }
#pragma unroll
    for (int u = 0; u < kHdKpt; ++u) {
      const uint64_t i = t0 + (uint64_t)u * kHThreads + tid;
      if (i < hi) rk[u] = atomicAdd(&cnt[hslot(k[u], m) >> s], 1u);
    }
    __syncthreads();
    for (uint32_t b = tid; b < K; b += kHThreads) base[b] = cnt[b] ? atomicAdd(cursor + b, cnt[b]) : 0u;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kHdKpt; ++u) {
      const uint64_t i = t0 + (uint64_t)u * kHThreads + tid;
      if (i >= hi) continue;
      const uint32_t b = hslot(k[u], m) >> s;
      const uint32_t slot = base[b] + rk[u];
      if (slot < cap) {
        const uint32_t e = b * cap + slot;
        qkeys[e] = k[u];
        __stcs(inv + i, e);
      } else {
        const uint32_t o = atomicAdd(n_ovf, 1u);
        ovf[o] = (i << 32) | k[u];
        __stcs(inv + i, kNotFound);
      }
    }
    __syncthreads();
  }
}

// The overflow keys of the one-pass Phase I: looked up directly.
__global__ void __launch_bounds__(256) k_hash_overflow(const uint4* __restrict__ table, uint32_t m,
                                                        const uint4* __restrict__ pool,
                                                        const uint64_t* __restrict__ ovf,
                                                        const uint32_t* __restrict__ n_ovf,
                                                        uint32_t* __restrict__ out) {
  const uint32_t no = *n_ovf;
  for (uint32_t o = blockIdx.x * blockDim.x + threadIdx.x; o < no; o += gridDim.x * blockDim.x) {
    const uint64_t e = ovf[o];
    const uint32_t key = (uint32_t)e;
    out[e >> 32] = hash_chain(__ldg(table + hslot(key, m)), key, pool);
  }
}

cudaError_t launch_hash_distribute(const uint32_t* keys, uint64_t n, uint32_t m, uint32_t s, uint32_t K,
                                   uint32_t cap, uint32_t* cursor, uint32_t* qkeys, uint32_t* inv,
                                   uint64_t* ovf, uint32_t* n_ovf, int sm, cudaStream_t st,
                                   uint32_t* nl) {
  ++*nl;
  const uint64_t chunk = (n + sm - 1) / sm;
  k_hash_distribute<<<sm, kHThreads, 0, st>>>(keys, n, chunk, m, s, K, cap, cursor, qkeys, inv, ovf,
                                              n_ovf);
  return cudaGetLastError();
}

cudaError_t launch_hash_overflow(const void* table, uint32_t m, const void* pool, const uint64_t* ovf,
                                 const uint32_t* n_ovf, uint32_t* out, int sm, cudaStream_t st,
                                 uint32_t* nl) {
  ++*nl;
  k_hash_overflow<<<sm * 2, 256, 0, st>>>((const uint4*)table, m, (const uint4*)pool, ovf, n_ovf, out);
  return cudaGetLastError();
}

cudaError_t launch_gather_u32(const uint32_t* tmp, const uint32_t* inv, uint64_t n, uint32_t* out,
                              int sm, cudaStream_t st, uint32_t* nl) {
  ++*nl;
  const uint32_t g = (uint32_t)max_u64(1, min_u64((n + 255) / 256, (uint64_t)sm * 8));
  k_gather_u32<<<g, 256, 0, st>>>(tmp, inv, n, out);
  return cudaGetLastError();
}

cudaError_t launch_hash_direct(const void* table, uint32_t m, const void* pool, const uint32_t* keys,
                               uint64_t n, uint32_t* out, int sm, cudaStream_t st, uint32_t* nl) {
  ++*nl;
  const uint32_t g = (uint32_t)max_u64(1, min_u64((n + 255) / 256, (uint64_t)sm * 8));
  k_hash_direct<<<g, 256, 0, st>>>((const uint4*)table, m, (const uint4*)pool, keys, n, out);
  return cudaGetLastError();
}

cudaError_t launch_hash_probe(const void* table, uint32_t m, uint32_t s, uint32_t K, const void* pool,
                              const uint32_t* qkeys, const uint32_t* run_start, uint32_t* tmp,
                              uint32_t* gbar, int sm, cudaStream_t st, uint32_t* nl,
                              const uint32_t* counts, uint32_t cap) {
  ++*nl;
  HashProbeArgs a;
  a.counts = counts;
  a.cap = cap;
  a.table = (const uint4*)table;
  a.m = m;
  a.s = s;
  a.K = K;
  a.pool = (const uint4*)pool;
  a.qkeys = qkeys;
  a.run_start = run_start;
  a.tmp = tmp;
  a.gbar = gbar;
  const int smem = 128 + 4 * (32 << 10);
  cudaError_t e = cudaFuncSetAttribute(k_hash_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  void* params[] = {&a};
  return cudaLaunchCooperativeKernel((const void*)k_hash_probe, dim3(sm), dim3(kHThreads), params,
                                     smem, st);
}

}  // namespace dpg
