// fused.cu -- the whole DPG path in one persistent cooperative kernel.
//
//   Phase I   Distribute (Fig. 1)
//     B  count : each CTA histograms its contiguous chunk of the rid list by
//                run r >> s into warp-private 16-bit counters (warp-level
//                __match_any_sync aggregation, no shared-memory atomics), then
//                reserves its share of every run with one global atomicAdd per
//                run ("count the number of elements destined for each
//                bucket").
//     -- grid barrier --
//     C  scan + scatter : every CTA scans the K run totals ("set bucket
//                boundaries according to the statistics") and
//                appends each rid to its run ("Append r to RID_RUN[run_num]",
//                P:410).
//     -- grid barrier --
//   Phase II  Probe (Fig. 1): warp 0 is a TMA producer
//        that bulk-copies each run of INPUT owned by this CTA ("load the i-th
//        INPUT run entirely into cache") plus the run's RID-run
//        entries into one of S shared-memory stages (full/empty mbarrier
//        ring); the other warps consume the stages asynchronously.  The
//        source runs of the first two items are prefetched before Phase I, so
//        the distribute overlaps the first source reads.
//   Phase III Gather (Fig. 1), in one of two modes:
//     mode 0 (fused):  the probe writes each staged record straight to its
//        output row; the RID-run entry carries the row (pos).  No INTERNAL
//        file.  Right when rows are whole 32-byte sectors (rec % 32 == 0):
//        B200's L2 then absorbs the scattered rows without read-modify-write.
//     mode 1 (three-phase, as Fig. 1): the probe appends records to the run's
//        INTERNAL segment sequentially (L2 evict_last: for L2-sized inputs
//        INTERNAL stays on chip), a grid barrier, then each CTA gathers its own
//        chunk of output rows, "the next record from the j-th INTERNAL run"
//         being INTERNAL[inv[i]], and writes the rows sequentially.
//        Right for records that straddle sectors (e.g. 100 B), whose scattered
//        writes would each cost a DRAM read-modify-write.
//
// Shared memory: [header | bucket_start[K+1] | stage 0 | ... | stage S-1];
// during Phase I the last two stages hold the warp histograms and CTA bases.
#include "dpg_internal.cuh"

namespace dpg {

static constexpr int kFusedThreads = 512;
static constexpr int kWarps = kFusedThreads / 32;
static constexpr int kConsumers = kWarps - 1;
static constexpr uint32_t kHdr = 512;
static constexpr int kMaxStages = 8;

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

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ const uint8_t* adn(const uint8_t* p) {
  return reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15));
}
__device__ __forceinline__ const uint8_t* aup(const uint8_t* p) {
  return reinterpret_cast<const uint8_t*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
}

// Item sequence of one CTA over its runs b = c, c+G, ...: first the leading
// chunk (up to slot_pairs entries) of every run, then -- only for runs heavier
// than one stage (skew) -- their remaining chunks.  Item t < #runs
// is therefore always run c + t*G, which lets the source of the first runs be
// prefetched before Phase I knows the run sizes.
struct Items {
  uint32_t b, j, pass, c, G, K, sp;
  const uint32_t* bs;
  __device__ void init(uint32_t c_, uint32_t G_, uint32_t K_, uint32_t sp_, const uint32_t* bs_) {
    c = c_; b = c_; j = 0; pass = 0; G = G_; K = K_; sp = sp_; bs = bs_;
    if (b >= K) { pass = 1; b = K; }
  }
  __device__ bool valid() const { return b < K; }
  __device__ uint32_t p0() const { return bs[b] + j * sp; }
  __device__ uint32_t p1() const { return min(bs[b + 1], bs[b] + (j + 1) * sp); }
  __device__ void settle() {
    while (b < K && j * sp >= bs[b + 1] - bs[b]) { b += G; j = 1; }
  }
  __device__ void next() {
    if (pass == 0) {
      b += G;
      if (b >= K) { pass = 1; b = c; j = 1; settle(); }
    } else {
      ++j;
      settle();
    }
  }
};

// Producer-warp helpers --------------------------------------------------------
// Copy the unaligned head/tail bytes of run b's byte range into the stage
// (whole warp), so that the bulk copy can take the 16-byte-aligned interior.
__device__ __forceinline__ void issue_region(const FusedArgs& a, uint32_t b, uint8_t* stage,
                                             uint64_t* full, int lane, uint64_t pol) {
  const uint64_t rec0 = (uint64_t)b << a.s;
  const uint64_t rec1 = min_u64(a.n_src, rec0 + (1ull << a.s));
  const uint8_t* r0 = a.src + rec0 * a.rec;
  const uint8_t* r1 = a.src + rec1 * a.rec;
  const uint8_t* rb = adn(r0);
  const uint8_t* ra0 = aup(r0);
  const uint8_t* ra1 = adn(r1);
  if (ra1 <= ra0) {
    for (const uint8_t* p = r0 + lane; p < r1; p += 32) stage[p - rb] = *p;
    ra1 = ra0;
  } else {
    for (const uint8_t* p = r0 + lane; p < ra0; p += 32) stage[p - rb] = *p;
    for (const uint8_t* p = ra1 + lane; p < r1; p += 32) stage[p - rb] = *p;
  }
  __syncwarp();
  if (lane == 0) {
    const uint32_t bytes = (uint32_t)(ra1 - ra0);
    mbar_arrive_expect_tx(full, bytes);
    if (bytes) bulk_g2s(stage + (ra0 - rb), ra0, bytes, full, pol);
  }
}

__device__ __forceinline__ void issue_pairs(const FusedArgs& a, uint32_t p0, uint32_t p1,
                                            uint8_t* stage, uint64_t* full, int lane,
                                            uint64_t pol) {
  if (lane == 0) {
    if (p1 > p0) {
      const uint8_t* pb = reinterpret_cast<const uint8_t*>(a.pairs);
      const uint8_t* q0 = adn(pb + (uint64_t)p0 * a.pair_bytes);
      const uint8_t* q1 = aup(pb + (uint64_t)p1 * a.pair_bytes);
      const uint32_t bytes = (uint32_t)(q1 - q0);
      mbar_arrive_expect_tx(full, bytes);
      bulk_g2s(stage + a.region_cap, q0, bytes, full, pol);
    } else {
      mbar_arrive(full);
    }
  }
}

// mode 0 entry: (pos << s | local) in 4 bytes or (local, pos) in 8 bytes;
// mode 1 entry: local only (2 or 4 bytes).
template <typename PairT, int MODE>
__device__ __forceinline__ void unpack(PairT p, uint32_t s, uint32_t& local, uint32_t& pos) {
  if (MODE == 1) {
    local = (uint32_t)p;
    pos = 0;
  } else if (sizeof(PairT) == 4) {
    local = (uint32_t)p & ((1u << s) - 1u);
    pos = (uint32_t)p >> s;
  } else {
    local = (uint32_t)(uint64_t)p;
    pos = (uint32_t)((uint64_t)p >> 32);
  }
}

template <int W, typename PairT, int MODE>
__global__ void __launch_bounds__(kFusedThreads, 1) k_dpg_fused(FusedArgs a) {
  using T = typename Word<W>::T;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  uint32_t* wsum = reinterpret_cast<uint32_t*>(smem + 128);
  uint32_t* bs = reinterpret_cast<uint32_t*>(smem + kHdr);
  const uint32_t bs_bytes = ((a.K + 1) * 4 + 127) & ~127u;
  uint8_t* stages = smem + kHdr + bs_bytes;
  const uint32_t S = a.nstages;
  // Phase I scratch: the stages not prefetched into
  uint16_t* hw = reinterpret_cast<uint16_t*>(stages + (size_t)a.npre * a.stage_bytes);
  uint32_t* cbase = reinterpret_cast<uint32_t*>(hw + (size_t)a.hist_warps * a.K);
  uint32_t* rcache = cbase + ((a.K + 3) & ~3u);       // this CTA's rid chunk (optional)
  uint64_t* ridbar = reinterpret_cast<uint64_t*>(smem + 384);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t c = blockIdx.x, G = gridDim.x;
  const uint64_t pol_first = policy_evict_first();
#define DPG_STAMP(k) \
  if (a.ts && tid == 0) a.ts[(size_t)c * 8 + (k)] = globaltimer();
  DPG_STAMP(0);

  const uint64_t lo = (uint64_t)c * a.chunk;
  const uint64_t hi = min_u64(a.n_out, lo + a.chunk);
  const uint64_t span = hi > lo ? hi - lo : 0;
  if (tid == 0) {
    for (uint32_t k = 0; k < S; ++k) {
      mbar_init(&full[k], 2);          // region arrival + entries arrival
      mbar_init(&empty[k], kConsumers);
    }
    mbar_init(ridbar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  // ---- A: one bulk copy of this CTA's rid chunk; prefetch of its first runs -----
  const uint64_t span16 = a.rid_cache ? (span & ~3ull) : 0;   // 16-byte multiple
  if (tid == 0 && a.rid_cache) {
    mbar_arrive_expect_tx(ridbar, (uint32_t)(span16 * 4));
    if (span16) bulk_g2s(rcache, a.rids + lo, (uint32_t)(span16 * 4), ridbar, pol_first);
  }
  if (warp == 0) {
    for (uint32_t t = 0; t < a.npre; ++t) {
      const uint32_t b = c + t * G;
      if (b < a.K) issue_region(a, b, stages + (size_t)t * a.stage_bytes, &full[t], lane, pol_first);
    }
  }
  {
    uint4* h4 = reinterpret_cast<uint4*>(hw);
    const uint32_t n4 = (a.hist_warps * a.K * 2 + 15) / 16;
    for (uint32_t k = tid; k < n4; k += blockDim.x) h4[k] = make_uint4(0, 0, 0, 0);
    if (a.rid_cache && (uint64_t)tid < span - span16) rcache[span16 + tid] = a.rids[lo + span16 + tid];
  }
  if (a.rid_cache) mbar_wait(ridbar, 0);
  __syncthreads();

  // ---- B: count -----------------------------------------------------------------
  const uint32_t HW = a.hist_warps;   // warps with a private histogram (Phase I)
  const uint64_t sub = ((span + HW - 1) / HW + 31) & ~31ull;
  const uint64_t wlo = min_u64(hi, lo + (uint64_t)warp * sub);
  const uint64_t whi = min_u64(hi, wlo + sub);
  uint16_t* myh = hw + (size_t)warp * a.K;
  auto rid_at = [&](uint64_t i) -> uint32_t {
    return a.rid_cache ? rcache[i - lo] : __ldg(a.rids + i);
  };
  constexpr int U = 8;
  for (uint64_t i0 = wlo; i0 < whi; i0 += 32 * U) {
    uint32_t r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = i0 + u * 32 + lane;
      r[u] = i < whi ? rid_at(i) : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = i0 + u * 32 + lane;
      const bool in = i < whi;
      const bool ok = in && r[u] < a.n_src;
      if (in && !ok) report_bad(a.status, i);
      const uint32_t d = ok ? (r[u] >> a.s) : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
      if (ok && lane == __ffs(peers) - 1) myh[d] = (uint16_t)(myh[d] + __popc(peers));
    }
  }
  __syncthreads();
  {
    // CTA totals per run, warp-exclusive prefixes in place, and one global
    // reservation per (run, CTA); the atomics of a thread are all in flight
    // together.
    constexpr int BPT = 8;
    for (uint32_t b0 = tid; b0 < a.K; b0 += BPT * blockDim.x) {
      uint32_t sum[BPT];
#pragma unroll
      for (int q = 0; q < BPT; ++q) {
        const uint32_t b = b0 + q * blockDim.x;
        sum[q] = 0;
        if (b < a.K) {
#pragma unroll 4
          for (uint32_t w = 0; w < HW; ++w) {
            const uint32_t h = hw[(size_t)w * a.K + b];
            hw[(size_t)w * a.K + b] = (uint16_t)sum[q];
            sum[q] += h;
          }
        }
      }
      uint32_t base[BPT];
#pragma unroll
      for (int q = 0; q < BPT; ++q) {
        const uint32_t b = b0 + q * blockDim.x;
        base[q] = (b < a.K && sum[q]) ? atomicAdd(&a.total[b], sum[q]) : 0u;
      }
#pragma unroll
      for (int q = 0; q < BPT; ++q) {
        const uint32_t b = b0 + q * blockDim.x;
        if (b < a.K) cbase[b] = base[q];
      }
    }
  }
  DPG_STAMP(1);
  grid_barrier(a.gbar, G);
  DPG_STAMP(2);

  // ---- C: scan of run totals, then scatter ----------------------------------------
  {
    const uint32_t ipt = (a.K + blockDim.x - 1) / blockDim.x;
    const uint32_t k0 = tid * ipt;
    uint32_t local = 0;
    for (uint32_t k = k0; k < min(a.K, k0 + ipt); ++k) local += __ldcg(a.total + k);
    uint32_t x = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      const uint32_t v = lane < kWarps ? wsum[lane] : 0;
      uint32_t ws = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, ws, o);
        if (lane >= o) ws += y;
      }
      if (lane < kWarps) wsum[lane] = ws - v;
      if (lane == kWarps - 1) wsum[32] = ws;
    }
    __syncthreads();
    uint32_t run = wsum[warp] + x - local;
    for (uint32_t k = k0; k < min(a.K, k0 + ipt); ++k) {
      bs[k] = run;
      run += __ldcg(a.total + k);
    }
    if (tid == 0) bs[a.K] = wsum[32];
    __syncthreads();
  }
  {
    PairT* pairs = reinterpret_cast<PairT*>(a.pairs);
    const uint32_t lmask = (1u << a.s) - 1u;
    const uint32_t lt = lanemask_lt();
    for (uint64_t i0 = wlo; i0 < whi; i0 += 32 * U) {
      uint32_t r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t i = i0 + u * 32 + lane;
        r[u] = i < whi ? rid_at(i) : 0xFFFFFFFFu;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t i = i0 + u * 32 + lane;
        const bool ok = i < whi && r[u] < a.n_src;
        const uint32_t d = ok ? (r[u] >> a.s) : 0xFFFFFFFFu;
        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (ok && lane == leader) {
          const uint32_t h = myh[d];
          base = bs[d] + cbase[d] + h;
          myh[d] = (uint16_t)(h + __popc(peers));
        }
        base = __shfl_sync(0xFFFFFFFFu, base, leader);
        if (ok) {
          const uint32_t slot = base + __popc(peers & lt);
          const uint32_t loc = r[u] & lmask;
          if (MODE == 1) {
            pairs[slot] = (PairT)loc;
            a.inv[i] = slot;
          } else if (sizeof(PairT) == 4) {
            pairs[slot] = (PairT)(((uint32_t)i << a.s) | loc);
          } else {
            pairs[slot] = (PairT)((uint64_t)loc | ((uint64_t)i << 32));
          }
        } else if (MODE == 1 && i < whi) {
          a.inv[i] = 0xFFFFFFFFu;      // row left unwritten (invalid rid)
        }
      }
    }
  }
  DPG_STAMP(3);
  grid_barrier(a.gbar, G);
  DPG_STAMP(4);

  // ---- Phase II (+ III in mode 0) --------------------------------------------------
  for (uint32_t b = c; b < a.K; b += G) a.total[b] = 0;   // restore the zero invariant

  Items it;
  it.init(c, G, a.K, a.slot_pairs, bs);
  if (warp == 0) {
    // producer
    fence_proxy_async_global();  // RID-run entries were written by generic stores
    for (uint32_t t = 0; it.valid(); ++t, it.next()) {
      const uint32_t st = t % S;
      uint8_t* stage = stages + (size_t)st * a.stage_bytes;
      const bool pre = t < a.npre && it.pass == 0;
      if (t >= S) mbar_wait(&empty[st], ((t / S) & 1) ^ 1);
      const uint32_t p0 = it.p0(), p1 = it.p1();
      if (!pre) {
        if (p1 > p0) {
          issue_region(a, it.b, stage, &full[st], lane, pol_first);
        } else if (lane == 0) {
          mbar_arrive(&full[st]);
        }
      }
      issue_pairs(a, p0, p1, stage, &full[st], lane, pol_first);
    }
  } else {
    // consumers
    const uint32_t rank = warp - 1;
    const uint32_t R = a.row_bytes / W;
    const uint32_t RPI = R <= 32 ? 32 / R : 1;
    const uint32_t lr = R <= 32 ? lane / R : 0;
    const uint32_t lw = R <= 32 ? lane % R : 0;
    const bool lane_on = R <= 32 ? (uint32_t)lane < RPI * R : true;
    const uint64_t pol_last = policy_evict_last();
    uint32_t q0 = 0;
    for (uint32_t t = 0; it.valid(); ++t, it.next()) {
      const uint32_t st = t % S;
      const uint8_t* stage = stages + (size_t)st * a.stage_bytes;
      const uint32_t p0 = it.p0(), p1 = it.p1();
      const uint32_t n = p1 - p0;
      const uint32_t ng = (n + 31) / 32;
      mbar_wait(&full[st], (t / S) & 1);
      const uint8_t* r0 = a.src + ((uint64_t)it.b << a.s) * a.rec;
      const uint8_t* region = stage + (r0 - adn(r0));
      const uint8_t* pb = reinterpret_cast<const uint8_t*>(a.pairs) + (uint64_t)p0 * a.pair_bytes;
      const PairT* prs = reinterpret_cast<const PairT*>(stage + a.region_cap + (pb - adn(pb)));
      for (uint32_t g = (rank + kConsumers - (q0 % kConsumers)) % kConsumers; g < ng;
           g += kConsumers) {
        const uint32_t g0 = g * 32;
        uint32_t my_local = 0, my_pos = 0;
        if (g0 + lane < n) unpack<PairT, MODE>(prs[g0 + lane], a.s, my_local, my_pos);
        const uint32_t cnt = min(32u, n - g0);
        // destination of entry rr of this group: mode 0 its output row, mode 1
        // the next slot of the run's INTERNAL segment
        uint8_t* const obase = MODE == 1 ? a.internal + (uint64_t)(p0 + g0) * a.rec : a.dst;
        if (R <= 32) {
          constexpr int B = W >= 16 ? 4 : 8;
          for (uint32_t k0 = 0; k0 < cnt; k0 += RPI * B) {
            T v[B];
            uint32_t ps[B];
#pragma unroll
            for (int u = 0; u < B; ++u) {
              const uint32_t rr = k0 + u * RPI + lr;
              const uint32_t loc = __shfl_sync(0xFFFFFFFFu, my_local, rr & 31);
              ps[u] = MODE == 1 ? rr : __shfl_sync(0xFFFFFFFFu, my_pos, rr & 31);
              if (lane_on && rr < cnt)
                v[u] = *reinterpret_cast<const T*>(region + (size_t)loc * a.rec + lw * W);
            }
#pragma unroll
            for (int u = 0; u < B; ++u) {
              const uint32_t rr = k0 + u * RPI + lr;
              if (lane_on && rr < cnt) {
                uint8_t* d = obase + (uint64_t)ps[u] * a.row_bytes + lw * W;
                if (MODE == 1) HintIO<W>::st(d, v[u], pol_last);
                else *reinterpret_cast<T*>(d) = v[u];
              }
            }
          }
        } else {
          for (uint32_t rr = 0; rr < cnt; ++rr) {
            const uint32_t loc = __shfl_sync(0xFFFFFFFFu, my_local, rr);
            const uint32_t pos = MODE == 1 ? rr : __shfl_sync(0xFFFFFFFFu, my_pos, rr);
            const uint8_t* srow = region + (size_t)loc * a.rec;
            uint8_t* drow = obase + (uint64_t)pos * a.row_bytes;
#pragma unroll 4
            for (uint32_t w = lane; w < R; w += 32) {
              const T v = *reinterpret_cast<const T*>(srow + w * W);
              if (MODE == 1) HintIO<W>::st(drow + w * W, v, pol_last);
              else *reinterpret_cast<T*>(drow + w * W) = v;
            }
          }
        }
      }
      q0 += ng;
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  }

  // Mode 1: Phase III (gather from INTERNAL) is a separate launch of the
  // direct-gather kernel over (INTERNAL, inv), at full occupancy (api.cu).
  if (a.ts) {
    __syncthreads();
    DPG_STAMP(7);
  }
#undef DPG_STAMP
}

template <int W, typename PairT, int MODE>
static cudaError_t launch_t(const FusedArgs& a, uint32_t grid, uint32_t smem, cudaStream_t st) {
  auto fn = k_dpg_fused<W, PairT, MODE>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  FusedArgs arg = a;
  void* params[] = {&arg};
  return cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(kFusedThreads), params,
                                     smem, st);
}

template <int W>
static cudaError_t launch_w(const FusedArgs& a, uint32_t grid, uint32_t smem, cudaStream_t st) {
  if (a.mode == 1)
    return a.pair_bytes == 2 ? launch_t<W, uint16_t, 1>(a, grid, smem, st)
                             : launch_t<W, uint32_t, 1>(a, grid, smem, st);
  return a.pair_bytes == 4 ? launch_t<W, uint32_t, 0>(a, grid, smem, st)
                           : launch_t<W, uint64_t, 0>(a, grid, smem, st);
}

cudaError_t launch_fused(const FusedArgs& a, uint32_t W, uint32_t grid, uint32_t smem,
                         cudaStream_t st, uint32_t* nl) {
  ++*nl;
  switch (W) {
    case 16: return launch_w<16>(a, grid, smem, st);
    case 8: return launch_w<8>(a, grid, smem, st);
    case 4: return launch_w<4>(a, grid, smem, st);
    case 2: return launch_w<2>(a, grid, smem, st);
    default: return launch_w<1>(a, grid, smem, st);
  }
}

}  // namespace dpg
