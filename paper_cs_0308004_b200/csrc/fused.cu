// fused.cu -- the whole DPG path in one persistent cooperative kernel.
//
//   Phase I   Distribute (Fig. 1).  Every rid r goes to
//        run r >> s ("the high order bits").  Per tile of the CTA's
//        chunk: each rid takes its rank inside (CTA, run) from a shared-memory
//        atomicAdd, the CTA reserves its share of every run with one global
//        atomicAdd per run, and each rid appends (r - run*L, i) at base + rank
//        ("Append r to RID_RUN[run_num]", plus the position i Phase
//        III needs).  Runs have a fixed capacity CAP: a
//        permutation puts exactly L rids into every run (the paper's sorting
//        case), rids drawn with replacement exceed L only by a
//        Poisson tail, and the rare excess -- or a skewed rid list (section
//        2.3) -- goes to an overflow list served after Phase II by
//        direct copies.  No scan: one grid barrier ends Phase I.
//   Phase II  Probe (Fig. 1): warp 0 is a TMA producer
//        that bulk-copies each run of INPUT owned by this CTA ("load the i-th
//        INPUT run entirely into cache") plus the run's entries
//        into one of S shared-memory stages (full/empty mbarrier ring); the
//        other warps consume the stages asynchronously.  The source runs of
//        the first items are prefetched before Phase I, so the distribute
//        overlaps the first source reads.
//   Phase III Gather (Fig. 1), in one of two modes:
//     mode 0 (fused):  the probe writes each staged record straight to its
//        output row; the entry carries the row (pos).  No INTERNAL file.
//     mode 1 (three-phase, as Fig. 1): the probe appends records to the run's
//        INTERNAL segment sequentially, then (separate launch, api.cu) the
//        output rows are gathered from INTERNAL and written sequentially.
//
// Shared memory: [header | own-run counts | stage 0 | ... | stage S-1]; the
// CTA's rid chunk is cached in a stage that is not prefetched into.
#include "dpg_internal.cuh"

namespace dpg {

static constexpr int kFusedThreads = 512;
static constexpr int kWarps = kFusedThreads / 32;
static constexpr int kConsumers = kWarps - 1;
static constexpr uint32_t kHdr = 512;
static constexpr int kMaxStages = 8;

__device__ __forceinline__ const uint8_t* adn(const uint8_t* p) {
  return reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15));
}
__device__ __forceinline__ const uint8_t* aup(const uint8_t* p) {
  return reinterpret_cast<const uint8_t*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
}

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

__device__ __forceinline__ void issue_pairs(const FusedArgs& a, uint64_t p0, uint64_t p1,
                                            uint8_t* stage, uint64_t* full, int lane,
                                            uint64_t pol) {
  if (lane == 0) {
    if (p1 > p0) {
      const uint8_t* pb = reinterpret_cast<const uint8_t*>(a.pairs);
      const uint8_t* q0 = adn(pb + p0 * a.pair_bytes);
      const uint8_t* q1 = aup(pb + p1 * a.pair_bytes);
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
  uint32_t* stage_run = reinterpret_cast<uint32_t*>(smem + 128);   // [kMaxStages] run in stage
  uint32_t* stage_n = reinterpret_cast<uint32_t*>(smem + 160);     // [kMaxStages] its entries
  uint64_t* ridbar = reinterpret_cast<uint64_t*>(smem + 384);
  uint32_t* own_cnt = reinterpret_cast<uint32_t*>(smem + kHdr);   // entries of run c + t*G
  const uint32_t own_bytes = (a.max_own * 4 + 127) & ~127u;
  uint8_t* stages = smem + kHdr + own_bytes;
  const uint32_t S = a.nstages;
  uint32_t* rcache = reinterpret_cast<uint32_t*>(stages + (size_t)a.npre * a.stage_bytes);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t c = blockIdx.x, G = gridDim.x;
  const uint64_t pol_first = policy_evict_first();
#define DPG_STAMP(k) \
  if (a.ts && tid == 0) a.ts[(size_t)c * 16 + (k)] = globaltimer();
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
  // ---- A: prefetch of the source runs of this CTA's first items: issued right
  // after the first rid tile's bulk copy (below), so that copy is not queued
  // behind them.
  auto prefetch_runs = [&]() {
    if (warp == 0) {
      for (uint32_t t = 0; t < a.npre && t < a.n_static; ++t) {
        const uint32_t b = c + t * G;
        if (b < a.K) issue_region(a, b, stages + (size_t)t * a.stage_bytes, &full[t], lane, pol_first);
      }
    }
  };
  if (lo >= hi) prefetch_runs();

  // ---- B: distribute ---------------------------------------------------------------
  // The CTA's chunk of the rid list is processed in tiles (each staged into
  // shared memory by one bulk copy when rid_cache is set).  Pass 1: every rid
  // takes its rank inside (this CTA, its run) from a shared-memory atomicAdd on
  // the run's counter ("count the number of elements destined for each
  // bucket").  The CTA then reserves its share of every run with one
  // global atomicAdd per run ("set bucket boundaries according to the
  // statistics").  Pass 2 appends each rid to its run at base +
  // rank ("Append r to RID_RUN[run_num]"); no further atomics.
  uint32_t* hc = rcache + a.rcache_words;                        // [K] counts, then bases
  uint16_t* rank = reinterpret_cast<uint16_t*>(hc + ((a.K + 3) & ~3u));   // [tile]
  PairT* pairs = reinterpret_cast<PairT*>(a.pairs);
  const uint32_t lmask = (1u << a.s) - 1u;
  constexpr int U = 8;
  uint32_t tile_no = 0;
  for (uint64_t tlo = lo; tlo < hi; tlo += a.tile, ++tile_no) {
    const uint64_t thi = min_u64(hi, tlo + a.tile);
    const uint32_t tspan = (uint32_t)(thi - tlo);
    if (tile_no) __syncthreads();                  // previous tile fully consumed
    if (a.rid_cache) {
      const uint32_t t16 = tspan & ~3u;            // 16-byte multiple (tlo % 4 == 0)
      if (tid == 0) {
        mbar_arrive_expect_tx(ridbar, t16 * 4);
        if (t16) bulk_g2s(rcache, a.rids + tlo, t16 * 4, ridbar, pol_first);
      }
      if ((uint32_t)tid < tspan - t16) rcache[t16 + tid] = a.rids[tlo + t16 + tid];
    }
    if (tile_no == 0) prefetch_runs();
    for (uint32_t b = tid; b < a.K; b += blockDim.x) hc[b] = 0;
    if (a.rid_cache) mbar_wait(ridbar, tile_no & 1);
    __syncthreads();
    if (tile_no == 0) DPG_STAMP(1);
    auto rid_at = [&](uint32_t j) -> uint32_t {
      return a.rid_cache ? rcache[j] : __ldg(a.rids + tlo + j);
    };
    // pass 1: rank within (CTA, run)
    for (uint32_t j0 = tid; j0 < tspan; j0 += U * blockDim.x) {
      uint32_t r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t j = j0 + u * blockDim.x;
        r[u] = j < tspan ? rid_at(j) : 0xFFFFFFFFu;
      }
      uint32_t rmax = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) rmax = max(rmax, r[u]);
      if (j0 + (U - 1) * blockDim.x < tspan && rmax < a.n_src) {
        // (the common case, without per-rid branches: U valid rids)
#pragma unroll
        for (int u = 0; u < U; ++u)
          rank[j0 + u * blockDim.x] = (uint16_t)atomicAdd(&hc[r[u] >> a.s], 1u);
        continue;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t j = j0 + u * blockDim.x;
        if (j >= tspan) continue;
        if (r[u] < a.n_src) {
          rank[j] = (uint16_t)atomicAdd(&hc[r[u] >> a.s], 1u);
        } else {
          report_bad(a.status, tlo + j);
          if (MODE == 1) a.inv[tlo + j] = 0xFFFFFFFFu;   // row left unwritten
        }
      }
    }
    __syncthreads();
    if (tile_no == 0) DPG_STAMP(6);
    {
      constexpr int BPT = 8;    // a thread's reservations are all in flight together
      const uint32_t rot = (a.dbg & 2) ? (uint32_t)(((uint64_t)c * a.K) / G) : 0u;
      for (uint32_t b0 = tid; b0 < a.K; b0 += BPT * blockDim.x) {
        uint32_t base[BPT];
#pragma unroll
        for (int q = 0; q < BPT; ++q) {
          uint32_t b = b0 + q * blockDim.x;
          if (rot && b < a.K) b = b + rot < a.K ? b + rot : b + rot - a.K;
          const uint32_t n = b < a.K ? hc[b] : 0u;
          base[q] = n ? atomicAdd(&a.total[b], n) : 0u;
        }
#pragma unroll
        for (int q = 0; q < BPT; ++q) {
          uint32_t b = b0 + q * blockDim.x;
          if (rot && b < a.K) b = b + rot < a.K ? b + rot : b + rot - a.K;
          if (b < a.K) hc[b] = base[q];
        }
      }
    }
    __syncthreads();
    if (tile_no == 0) DPG_STAMP(7);
    // pass 2: append each rid to its run
    for (uint32_t j0 = tid; j0 < tspan; j0 += U * blockDim.x) {
      uint32_t r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t j = j0 + u * blockDim.x;
        r[u] = j < tspan ? rid_at(j) : 0xFFFFFFFFu;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t j = j0 + u * blockDim.x;
        if (j >= tspan || r[u] >= a.n_src) continue;
        const uint64_t i = tlo + j;
        const uint32_t b = r[u] >> a.s;
        const uint32_t slot = hc[b] + rank[j];
        const uint32_t loc = r[u] & lmask;
        if (slot < a.cap) {
          const uint64_t e = (uint64_t)b * a.cap + slot;
          if (MODE == 1) {
            pairs[e] = (PairT)loc;
            a.inv[i] = (uint32_t)e;
          } else if (sizeof(PairT) == 4) {
            pairs[e] = (PairT)(((uint32_t)i << a.s) | loc);
          } else {
            pairs[e] = (PairT)((uint64_t)loc | ((uint64_t)i << 32));
          }
        } else {
          // run over capacity (skew): served after Phase II by a direct copy
          const uint32_t o = atomicAdd(a.gbar + 2, 1u);
          a.ovf[o] = (uint64_t)i | ((uint64_t)r[u] << 32);
          if (MODE == 1) a.inv[i] = 0xFFFFFFFFu;
        }
      }
    }
    if (tile_no == 0) DPG_STAMP(8);
  }
  DPG_STAMP(2);
  grid_barrier(a.gbar, G);
  DPG_STAMP(3);

  // entries of this CTA's static runs; restore the zero invariant of the cursors
  for (uint32_t t = tid; t < a.n_static && c + (uint64_t)t * G < a.K; t += blockDim.x) {
    const uint32_t b = c + t * G;
    own_cnt[t] = min(__ldcg(a.total + b), a.cap);
    a.total[b] = 0;
  }
  __syncthreads();

  // ---- Phase II (+ III in mode 0) --------------------------------------------------
  // Run schedule: the CTA's static runs c + t*G (t < n_static; the first npre
  // of them were prefetched before Phase I), then runs claimed dynamically
  // from the pool [n_static*G, K) through a global counter, so that CTAs that
  // finish early take the remaining runs (the SMs' write rates differ by
  // +-15% under this scattered-store load).  The producer publishes each
  // stage's run and entry count in shared memory before its arrivals; a
  // sentinel run ends the consumers' loop.
  constexpr uint32_t kNoRun = 0xFFFFFFFFu;
  const uint32_t n_stat = c < a.K ? min(a.n_static, (a.K - c + G - 1) / G) : 0;
  const uint32_t dyn0 = a.n_static * G;
  if (warp == 0) {
    // producer
    fence_proxy_async_global();  // the entries were written by generic stores in Phase I
    for (uint32_t t = 0;; ++t) {
      uint32_t b, n;
      if (t < n_stat) {
        b = c + t * G;
        n = own_cnt[t];
      } else {
        uint32_t idx = 0;
        if (lane == 0) idx = dyn0 < a.K ? atomicAdd(a.gbar + 4, 1u) : 0xFFFFFFFFu;
        idx = __shfl_sync(0xFFFFFFFFu, idx, 0);
        b = (idx < a.K - min(dyn0, a.K)) ? dyn0 + idx : kNoRun;
        n = 0;
        if (b != kNoRun && lane == 0) {
          n = min(__ldcg(a.total + b), a.cap);
          a.total[b] = 0;
        }
        n = __shfl_sync(0xFFFFFFFFu, n, 0);
      }
      const uint32_t st = t % S;
      uint8_t* stage = stages + (size_t)st * a.stage_bytes;
      if (t >= S) mbar_wait(&empty[st], ((t / S) & 1) ^ 1);
      if (lane == 0) {
        stage_run[st] = b;
        stage_n[st] = n;
      }
      if (b == kNoRun) {
        if (lane == 0) { mbar_arrive(&full[st]); mbar_arrive(&full[st]); }
        break;
      }
      const uint64_t p0 = (uint64_t)b * a.cap, p1 = p0 + n;
      if (t >= a.npre || t >= n_stat) {
        if (p1 > p0) issue_region(a, b, stage, &full[st], lane, pol_first);
        else if (lane == 0) mbar_arrive(&full[st]);
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
    for (uint32_t t = 0;; ++t) {
      const uint32_t st = t % S;
      const uint8_t* stage = stages + (size_t)st * a.stage_bytes;
      mbar_wait(&full[st], (t / S) & 1);
      const uint32_t b = stage_run[st];
      if (b == kNoRun) break;
      const uint32_t n = stage_n[st];
      const uint64_t p0 = (uint64_t)b * a.cap;
      const uint32_t ng = (n + 31) / 32;
      const uint8_t* r0 = a.src + ((uint64_t)b << a.s) * a.rec;
      const uint8_t* region = stage + (r0 - adn(r0));
      const uint8_t* pb = reinterpret_cast<const uint8_t*>(a.pairs) + p0 * a.pair_bytes;
      const PairT* prs = reinterpret_cast<const PairT*>(stage + a.region_cap + (pb - adn(pb)));
      for (uint32_t g = (rank + kConsumers - (q0 % kConsumers)) % kConsumers; g < ng;
           g += kConsumers) {
        const uint32_t g0 = g * 32;
        uint32_t my_local = 0, my_pos = 0;
        if (g0 + lane < n) unpack<PairT, MODE>(prs[g0 + lane], a.s, my_local, my_pos);
        const uint32_t cnt = min(32u, n - g0);
        // destination of entry rr of this group: mode 0 its output row, mode 1
        // the next slot of the run's INTERNAL segment
        uint8_t* const obase = MODE == 1 ? a.internal + (p0 + g0) * a.rec : a.dst;
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
                uint8_t* d = (MODE == 1 ? obase + (uint64_t)ps[u] * a.row_bytes
                                        : seg_row(a.seg, a.dst, ps[u], a.row_bytes)) + lw * W;
                // rows with L2 evict_last: a row's partially written sectors stay
                // in L2 until the neighbouring rows complete them (measured: -15%)
                if (!(a.dbg & 1)) HintIO<W>::st(d, v[u], pol_last);
                else *reinterpret_cast<T*>(d) = v[u];
              }
            }
          }
        } else {
          for (uint32_t rr = 0; rr < cnt; ++rr) {
            const uint32_t loc = __shfl_sync(0xFFFFFFFFu, my_local, rr);
            const uint32_t pos = MODE == 1 ? rr : __shfl_sync(0xFFFFFFFFu, my_pos, rr);
            const uint8_t* srow = region + (size_t)loc * a.rec;
            uint8_t* drow = MODE == 1 ? obase + (uint64_t)pos * a.row_bytes
                                      : seg_row(a.seg, a.dst, pos, a.row_bytes);
#pragma unroll 4
            for (uint32_t w = lane; w < R; w += 32) {
              const T v = *reinterpret_cast<const T*>(srow + w * W);
              if (!(a.dbg & 1)) HintIO<W>::st(drow + w * W, v, pol_last);
              else *reinterpret_cast<T*>(drow + w * W) = v;
            }
          }
        }
      }
      q0 += ng;
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (a.ts && tid == 32) a.ts[(size_t)c * 16 + 9] = globaltimer();
  }
  DPG_STAMP(4);

  // ---- overflow entries (runs over capacity): direct copies ------------------------
  {
    const uint32_t n_ovf = __ldcg(a.gbar + 2);   // final since the grid barrier
    if (n_ovf) {
      const uint32_t R = a.rec / W;
      for (uint64_t j = (uint64_t)c * kWarps + warp; j < n_ovf; j += (uint64_t)G * kWarps) {
        const uint64_t e = __ldcg(a.ovf + j);
        const uint64_t i = (uint32_t)e, r = e >> 32;
        const uint8_t* s = a.src + r * a.rec;
        uint8_t* d = seg_row(a.seg, a.dst, i, a.row_bytes);
        for (uint32_t w = lane; w < R; w += 32)
          *reinterpret_cast<T*>(d + w * W) = *reinterpret_cast<const T*>(s + w * W);
      }
    }
    // rows written into peer memory (output segments mapped from other GPUs)
    // are made visible system-wide before the kernel ends
    if (a.seg.n) __threadfence_system();
    // the last CTA through here resets the overflow count for the next call
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      if (atomicAdd(a.gbar + 3, 1u) == G - 1) {
        atomicExch(a.gbar + 2, 0u);
        atomicExch(a.gbar + 4, 0u);
        atomicExch(a.gbar + 3, 0u);
      }
    }
  }
  if (a.ts) {
    __syncthreads();
    DPG_STAMP(5);
  }
#undef DPG_STAMP
}

template <int W, typename PairT, int MODE>
static cudaError_t launch_t(const FusedArgs& a, uint32_t grid, uint32_t smem, cudaStream_t st) {
  auto fn = k_dpg_fused<W, PairT, MODE>;
  // opt in to the dynamic shared memory once per device and size
  static int set_dev = -1;
  static uint32_t set_smem = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (set_dev != dev || set_smem < smem) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    set_dev = dev;
    set_smem = smem;
  }
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
