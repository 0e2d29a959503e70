// l2k.cu -- DPG with K L2-sized runs (Fig. 1 with the L2 as the cache) for
// sources larger than the L2 budget (config 3, config 4's dimension table).
//
//   Phase I  (k_l2k_distribute, one cooperative kernel): every rid r goes to
//            run b = r >> s, with L = 2^s records per run sized to the L2
//            (constraint (1)).  Each CTA owns a chunk of output
//            positions, its warps take 32-row groups round-robin; pass 1
//            counts per (warp, run), a grid barrier makes the (run, CTA)
//            totals visible, every CTA derives the start of its blocks, and
//            pass 2 appends each rid ("Append r to RID_RUN[run_num]",
//            P:410): local[slot] = r - b*L and inv[i] = slot.  Inside a run,
//            CTA blocks follow the CTA order and a block is the concatenation
//            of its warps' rows, each warp's in output order -- so Phase III,
//            walking the outputs in the same warp/group order, reads every
//            INTERNAL run as 16 x 148 sequential streams.
//   Phase II (K launches of the L2-run kernel, l2run.cu): run b is staged
//            into L2 (TMA, evict_last), then probed: INTERNAL[slot] =
//            R[b*L + local[slot]] for the run's slots in order (P:287-302,
//            413-422); the slot range comes from the device (run_start).
//   Phase III (one launch of the same kernel without staging): dst[i] =
//            INTERNAL[inv[i]] in output order.
// DRAM traffic per record: rid 2x, local 2x, inv 2x (4 B each), the source
// once and INTERNAL twice (sequential), the output once -- no random HBM
// access.
#include "dpg_internal.cuh"

namespace dpg {

static constexpr int kKThreads = 512;
static constexpr int kKWarps = kKThreads / 32;

// HASH: the entries are query keys of the batch index lookup:
// the "rid" is the key's hash slot, the run its partition of the hash array,
// and the appended value is the key itself.
template <typename RidT, bool HASH>
__global__ void __launch_bounds__(kKThreads, 1) k_l2k_distribute(L2KArgs a) {
  const RidT* rids = reinterpret_cast<const RidT*>(a.rids);
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* wrun = sm;                                  // [kKWarps][K] counts, then cursors
  uint32_t* base = sm + kKWarps * a.K;                  // [K] start of this CTA's block of run b
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t c = blockIdx.x, G = gridDim.x, K = a.K;
  const uint64_t lo = min_u64(a.n_out, (uint64_t)c * a.chunk);
  const uint64_t hi = min_u64(a.n_out, lo + a.chunk);
  const uint32_t ngroups = (uint32_t)((hi - lo + 31) / 32);
  for (uint32_t k = tid; k < kKWarps * K; k += kKThreads) wrun[k] = 0;
  __syncthreads();
  uint32_t* my = wrun + warp * K;

  // ---- pass 1: rows per (warp, run) ----
  for (uint32_t g0 = warp; g0 < ngroups; g0 += 8 * kKWarps) {
    RidT r[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t g = g0 + u * kKWarps;
      const uint64_t i = lo + 32 * (uint64_t)g + lane;
      r[u] = (g < ngroups && i < hi) ? __ldcg(rids + i) : ~RidT(0);
      if (HASH && g < ngroups && i < hi) r[u] = (uint32_t)(r[u] * 0x9E3779B1u) >> (32 - a.hash_m);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t g = g0 + u * kKWarps;
      if (g >= ngroups) break;
      const uint64_t i = lo + 32 * (uint64_t)g + lane;
      const bool valid = r[u] < a.n_src;
      if (!HASH && i < hi && !valid) report_bad(a.status, i);
      // (a count needs no rank: warp-private counters, shared-memory atomics)
      if (valid) atomicAdd(&my[(uint32_t)(r[u] >> a.s)], 1u);
    }
  }
  __syncthreads();
  // (run, CTA) totals, and the warps' exclusive offsets inside the CTA's block
  for (uint32_t b = tid; b < K; b += kKThreads) {
    uint32_t t = 0;
    for (int w = 0; w < kKWarps; ++w) {
      const uint32_t x = wrun[w * K + b];
      wrun[w * K + b] = t;
      t += x;
    }
    a.counts[(uint64_t)b * G + c] = t;
  }
  grid_barrier_mono(a.gbar, G);
  // start of this CTA's block in each run: rows of all earlier runs, then of
  // the earlier CTAs in this run; CTA 0 publishes run_start[0..K]
  {
    __shared__ uint32_t s_carry;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (uint32_t b0 = 0; b0 < K; b0 += kKThreads) {
      const uint32_t b = b0 + tid;
      uint32_t tot = 0, pre = 0;
      if (b < K) {
        const uint32_t* row = a.counts + (uint64_t)b * G;
        for (uint32_t q = 0; q < G; ++q) {
          const uint32_t x = __ldcg(row + q);
          tot += x;
          if (q < c) pre += x;
        }
      }
      // exclusive scan of tot over b (block-wide, in warp chunks)
      uint32_t y = tot;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, y, d);
        if (lane >= d) y += t;
      }
      __shared__ uint32_t wsum[kKWarps];
      if (lane == 31) wsum[warp] = y;
      __syncthreads();
      uint32_t woff = s_carry;
      for (int w = 0; w < warp; ++w) woff += wsum[w];
      const uint32_t start = woff + y - tot;
      if (b < K) {
        base[b] = start + pre;
        if (c == 0) {
          a.run_start[b] = start;
          if (a.counts64) a.counts64[b] = tot;
        }
      }
      __syncthreads();
      if (tid == 0) {
        uint32_t t = s_carry;
        for (int w = 0; w < kKWarps; ++w) t += wsum[w];
        s_carry = t;
      }
      __syncthreads();
    }
    if (c == 0 && tid == 0) a.run_start[K] = s_carry;
  }
  __syncthreads();
  // cursors: block start + the warp's offset
  for (uint32_t k = tid; k < kKWarps * K; k += kKThreads) wrun[k] += base[k % K];
  __syncthreads();

  // ---- pass 2: append (the same groups, the same order) ----
  const RidT lmask = (RidT)((1ull << a.s) - 1ull);
  for (uint32_t g0 = warp; g0 < ngroups; g0 += 8 * kKWarps) {
    RidT r[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t g = g0 + u * kKWarps;
      const uint64_t i = lo + 32 * (uint64_t)g + lane;
      r[u] = (g < ngroups && i < hi) ? __ldcs(rids + i) : ~RidT(0);
    }
    RidT key[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      key[u] = r[u];
      const uint32_t g = g0 + u * kKWarps;
      const uint64_t i = lo + 32 * (uint64_t)g + lane;
      if (HASH && g < ngroups && i < hi) r[u] = (uint32_t)(r[u] * 0x9E3779B1u) >> (32 - a.hash_m);
    }
    // the rank groups of all eight rows first (independent match.any issues)
    uint32_t pm[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool valid = r[u] < a.n_src;
      pm[u] = __match_any_sync(0xffffffffu, valid ? (uint32_t)(r[u] >> a.s) : 0xFFFFFFFFu);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t g = g0 + u * kKWarps;
      if (g >= ngroups) break;
      const uint64_t i = lo + 32 * (uint64_t)g + lane;
      const bool valid = r[u] < a.n_src;
      const uint32_t b = valid ? (uint32_t)(r[u] >> a.s) : 0xFFFFFFFFu;
      const uint32_t peers = pm[u];
      uint32_t slot = 0;
      if (valid) slot = my[b] + __popc(peers & lanemask_lt());
      __syncwarp();
      if (valid && (peers & lanemask_lt()) == 0) my[b] += __popc(peers);
      if (i < hi) {
        a.inv[i] = valid ? slot : 0xFFFFFFFFu;
        if (valid)
          a.local[slot] = HASH ? (uint32_t)key[u]
                               : a.payload ? __ldcs(a.payload + i) : (uint32_t)(r[u] & lmask);
      }
    }
  }
}

uint32_t l2k_smem_bytes(uint32_t K) { return (kKWarps + 1) * K * 4 + 64; }

cudaError_t launch_l2k_distribute(const L2KArgs& a, uint32_t grid, cudaStream_t st, uint32_t* nl) {
  ++*nl;
  const uint32_t smem = l2k_smem_bytes(a.K);
  auto fn = a.hash_m ? k_l2k_distribute<uint32_t, true>
                     : a.rid_bytes == 8 ? k_l2k_distribute<uint64_t, false> : k_l2k_distribute<uint32_t, false>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  L2KArgs arg = a;
  void* params[] = {&arg};
  return cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(kKThreads), params, smem, st);
}

}  // namespace dpg
