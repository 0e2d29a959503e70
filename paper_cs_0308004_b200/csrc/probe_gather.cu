// probe_gather.cu -- DPG Phases II + III fused, "Probe" and "Gather"
// (Fig. 1).
//
// Phase II: "every time, one loads the i-th INPUT run entirely into cache"
// and copies INPUT[r] for every rid r of RID run i.
// Phase III: "if the i-th rid was distributed to the j-th RID run ..., then at
// the i-th step of the Gather phase, the next record from the j-th INTERNAL
// run is copied to the destination array".
//
// B200 form: one persistent CTA per SM walks
// the items (run b, pair chunk j) i = blockIdx.x, blockIdx.x + grid, ...; each
// item's source records [bL, (b+1)L) and its pair chunk are staged into one of two shared-memory
// stages by TMA bulk copies (cp.async.bulk + mbarrier complete_tx, L2
// evict-first), double buffered so the next run streams in while this one is
// written out.  Each pair (local, pos) then copies the staged record straight
// to dst row pos: the INTERNAL file of Fig. 1 is never materialised, because
// the pair already names the gather destination and B200's L2 absorbs the
// scattered, fire-and-forget row writes (sector byte masks, no
// read-for-ownership).  A row may carry a payload from the pair (DPG-Move join:
// out row = fact row ++ dim record).
#include "dpg_internal.cuh"

namespace dpg {

static constexpr int kProbeThreads = 512;
static constexpr uint32_t kBarBytes = 128;

struct Item {
  uint32_t b;       // run (kItemDone: no more items)
  uint32_t chunk;   // pair chunk within the run
  uint32_t p0, p1;  // pair range [p0, p1)
  uint32_t more;    // 1: a later chunk of the run stages the same region
};
constexpr uint32_t kItemDone = 0xFFFFFFFFu;
constexpr uint32_t kNoLocal = 0xFFFFFFFFu;   // a pair whose rid was out of range

// The items are the (run, chunk) pairs in run order -- chunk j of run b holds
// its pairs [rs[b] + j*SP, min(rs[b+1], rs[b] + (j+1)*SP)) -- and item i runs
// on CTA i mod G, so a run with many rids (data skew) is spread
// over the CTAs instead of queueing on one.  items[i] = {b, j, p0, p1}
// (launch_items, distribute.cu): one independent load per item, so thread 0
// fetches the item after next while the CTA copies rows.
struct ItemIter {
  uint32_t i, stride, n;
  const uint4* items;
  __device__ bool first(uint32_t c, uint32_t G, const ProbeArgs& a, Item& it) {
    stride = G;
    items = reinterpret_cast<const uint4*>(a.item_run);
    n = __ldg(a.item_start + a.K);
    i = c;
    return settle(it);
  }
  __device__ bool settle(Item& it) {
    if (i >= n) return false;
    const uint4 d = __ldg(items + i);
    it.b = d.x;
    it.chunk = d.y & 0x7FFFFFFFu;
    it.more = d.y >> 31;
    it.p0 = d.z;
    it.p1 = d.w;
    return true;
  }
  __device__ bool next(Item& it) { i += stride; return settle(it); }
};

struct SlotPtrs {
  uint8_t* region;  // staged bytes start here (16-aligned base)
  uint8_t* pairs;
  uint8_t* pay;
};

__device__ __forceinline__ SlotPtrs slot_ptrs(uint8_t* smem, const ProbeArgs& a, int slot) {
  uint8_t* base = smem + kBarBytes + (size_t)slot * a.slot_bytes;
  SlotPtrs p;
  p.region = base;
  p.pairs = base + a.region_cap;
  p.pay = p.pairs + ((a.slot_pairs * a.pair_bytes + 32 + 15) & ~15u);
  return p;
}

// Byte range [start, end) of `item` in global memory for each staged array.
struct Ranges {
  const uint8_t *r0, *r1;   // region
  const uint8_t *q0, *q1;   // pairs
  const uint8_t *y0, *y1;   // payload
};

__device__ __forceinline__ Ranges item_ranges(const ProbeArgs& a, const Item& it) {
  Ranges g;
  uint64_t rec0 = a.bmap ? (uint64_t)__ldg(a.bmap + it.b) : (uint64_t)it.b << a.s;
  uint64_t rec1 = a.bmap ? (uint64_t)__ldg(a.bmap + it.b + 1) : min_u64(a.n_src, rec0 + (1ull << a.s));
  g.r0 = a.src + rec0 * a.rec;
  g.r1 = a.src + rec1 * a.rec;
  const uint8_t* pb = reinterpret_cast<const uint8_t*>(a.pairs);
  g.q0 = pb + (uint64_t)it.p0 * a.pair_bytes;
  g.q1 = pb + (uint64_t)it.p1 * a.pair_bytes;
  g.y0 = a.pay + (uint64_t)it.p0 * a.pay_bytes;
  g.y1 = a.pay + (uint64_t)it.p1 * a.pay_bytes;
  return g;
}

__device__ __forceinline__ const uint8_t* align_dn(const uint8_t* p) {
  return reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15));
}
__device__ __forceinline__ const uint8_t* align_up(const uint8_t* p) {
  return reinterpret_cast<const uint8_t*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
}

// Thread 0: stage `it` into `slot`.  The region's 16-byte-aligned interior is
// bulk-copied; its unaligned head/tail bytes (if any) are copied by threads
// after the wait.  Pair and payload arrays live in padded workspace, so their
// chunks are bulk-copied from aligned-down to aligned-up addresses.
__device__ __forceinline__ void issue(const ProbeArgs& a, const Item& it, uint8_t* smem, int slot,
                                      uint64_t* bar, uint64_t pol, uint64_t pol_keep) {
  SlotPtrs sp = slot_ptrs(smem, a, slot);
  Ranges g = item_ranges(a, it);
  const uint8_t* rb = align_dn(g.r0);
  const uint8_t* ra0 = align_up(g.r0);
  const uint8_t* ra1 = align_dn(g.r1);
  uint32_t tx = 0;
  uint32_t rbytes = ra1 > ra0 ? (uint32_t)(ra1 - ra0) : 0;
  const uint8_t* qa0 = align_dn(g.q0);
  uint32_t qbytes = (uint32_t)(align_up(g.q1) - qa0);
  const uint8_t* ya0 = align_dn(g.y0);
  uint32_t ybytes = a.pay_bytes ? (uint32_t)(align_up(g.y1) - ya0) : 0;
  tx = rbytes + qbytes + ybytes;
  fence_proxy_async_smem();
  mbar_arrive_expect_tx(bar, tx);
  // a region another chunk of the run will stage again (on a neighbouring
  // CTA, at about the same time) is kept in L2 until that chunk reads it
  if (rbytes) bulk_g2s(sp.region + (ra0 - rb), ra0, rbytes, bar, it.more ? pol_keep : pol);
  bulk_g2s(sp.pairs, qa0, qbytes, bar, pol);
  if (ybytes) bulk_g2s(sp.pay, ya0, ybytes, bar, pol);
}

template <typename PairT>
__device__ __forceinline__ void unpack(PairT p, uint32_t s, uint32_t& local, uint32_t& pos) {
  if (sizeof(PairT) == 4) {
    local = (uint32_t)p & ((1u << s) - 1u);
    pos = (uint32_t)p >> s;
  } else {
    local = (uint32_t)(uint64_t)p;
    pos = (uint32_t)((uint64_t)p >> 32);
  }
}

template <int W, typename PairT, bool PAY>
__global__ void __launch_bounds__(kProbeThreads, 1) k_probe_gather(const __grid_constant__ ProbeArgs a) {
  using T = typename Word<W>::T;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  const uint32_t R = a.row_bytes / W;      // words per output row
  const uint32_t PR = PAY ? a.pay_bytes / W : 0;
  const uint32_t recW = a.rec / W;

  __shared__ Item sit[2];   // the item staged in each slot (written by thread 0 before its arrive)
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();

  uint64_t pol = policy_evict_first();
  uint64_t pol_keep = policy_evict_last();
  ItemIter prod;
  Item pit;
  bool phave = false;
  // thread 0 fills a slot: the next item's copies, or the end mark
  auto post = [&](int slot) {
    if (phave) {
      sit[slot] = pit;
      issue(a, pit, smem, slot, &bars[slot], pol, pol_keep);
      phave = prod.next(pit);   // (loads in flight while the CTA copies rows)
    } else {
      sit[slot].b = kItemDone;
      mbar_arrive(&bars[slot]);
    }
  };
  if (tid == 0) {
    phave = prod.first(blockIdx.x, gridDim.x, a, pit);
    post(0);
    post(1);
  }

  // Per-lane word mapping for rows of R <= 32 words: RPI rows per warp step.
  const uint32_t RPI = R <= 32 ? 32 / R : 1;
  const uint32_t lr = R <= 32 ? lane / R : 0;
  const uint32_t lw = R <= 32 ? lane % R : 0;
  const bool lane_on = R <= 32 ? (uint32_t)lane < RPI * R : true;

  uint32_t it_idx = 0;
  while (true) {
    const int slot = it_idx & 1;
    const uint32_t parity = (it_idx >> 1) & 1;
    mbar_wait(&bars[slot], parity);
    const Item cit = sit[slot];
    if (cit.b == kItemDone) break;
    SlotPtrs sp = slot_ptrs(smem, a, slot);
    Ranges g = item_ranges(a, cit);
    const uint8_t* rb = align_dn(g.r0);
    // Unaligned head / tail bytes of the region, copied by warp 0.
    if (warp == 0) {
      const uint8_t* ra0 = align_up(g.r0);
      const uint8_t* ra1 = align_dn(g.r1);
      if (ra1 <= ra0) {
        for (const uint8_t* p = g.r0 + lane; p < g.r1; p += 32) sp.region[p - rb] = *p;
      } else {
        for (const uint8_t* p = g.r0 + lane; p < ra0; p += 32) sp.region[p - rb] = *p;
        for (const uint8_t* p = ra1 + lane; p < g.r1; p += 32) sp.region[p - rb] = *p;
      }
    }
    __syncthreads();

    const uint8_t* region = sp.region + (g.r0 - rb);
    const PairT* prs = reinterpret_cast<const PairT*>(sp.pairs + (g.q0 - align_dn(g.q0)));
    const uint8_t* pay = PAY ? sp.pay + (g.y0 - align_dn(g.y0)) : nullptr;
    const uint32_t n = cit.p1 - cit.p0;

    for (uint32_t g0 = (uint32_t)warp * 32; g0 < n; g0 += (uint32_t)nwarps * 32) {
      uint32_t my_local = 0, my_pos = 0;
      if (g0 + lane < n) {
        if (sizeof(PairT) == 8 && a.rid_pairs) {
          // radix Phase I elements (rid << 32) | position; a bad rid is skipped
          const uint64_t e = (uint64_t)prs[g0 + lane];
          const uint32_t r = (uint32_t)(e >> 32);
          my_pos = (uint32_t)e;
          my_local = r < a.n_src ? (r & ((1u << a.s) - 1u)) : kNoLocal;
        } else {
          unpack<PairT>(prs[g0 + lane], a.s, my_local, my_pos);
        }
      }
      const uint32_t cnt = min(32u, n - g0);
      if (R <= 32) {
#pragma unroll 4
        for (uint32_t k = 0; k < 32; k += RPI) {
          const uint32_t rr = k + lr;
          const uint32_t loc = __shfl_sync(0xffffffffu, my_local, rr & 31);
          const uint32_t pos = __shfl_sync(0xffffffffu, my_pos, rr & 31);
          if (lane_on && rr < cnt && loc != kNoLocal) {
            T v;
            if (PAY && lw < PR)
              v = *reinterpret_cast<const T*>(pay + (size_t)(g0 + rr) * a.pay_bytes + lw * W);
            else
              v = *reinterpret_cast<const T*>(region + (size_t)loc * a.rec + (lw - PR) * W);
            *reinterpret_cast<T*>(seg_row(a.seg, a.dst, pos, a.row_bytes) + lw * W) = v;
          }
        }
      } else {
        for (uint32_t rr = 0; rr < cnt; ++rr) {
          const uint32_t loc = __shfl_sync(0xffffffffu, my_local, rr);
          const uint32_t pos = __shfl_sync(0xffffffffu, my_pos, rr);
          if (loc == kNoLocal) continue;
          uint8_t* drow = seg_row(a.seg, a.dst, pos, a.row_bytes);
          const uint8_t* srow = region + (size_t)loc * a.rec;
#pragma unroll 4
          for (uint32_t w = lane; w < R; w += 32) {
            T v;
            if (PAY && w < PR)
              v = *reinterpret_cast<const T*>(pay + (size_t)(g0 + rr) * a.pay_bytes + w * W);
            else
              v = *reinterpret_cast<const T*>(srow + (w - PR) * W);
            *reinterpret_cast<T*>(drow + w * W) = v;
          }
        }
      }
    }
    (void)recW;
    __syncthreads();  // every thread is done reading this stage (and its item)
    if (tid == 0) post(slot);
    ++it_idx;
  }
  // rows written into peer memory (output segments mapped from other GPUs)
  // are made visible system-wide before the kernel ends
  if (a.seg.n) __threadfence_system();
}

template <int W, typename PairT, bool PAY>
static cudaError_t launch_t(const ProbeArgs& a, uint32_t grid, uint32_t smem, cudaStream_t st) {
  auto fn = k_probe_gather<W, PairT, PAY>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fn<<<grid, kProbeThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <int W>
static cudaError_t launch_w(const ProbeArgs& a, uint32_t grid, uint32_t smem, cudaStream_t st) {
  if (a.pair_bytes == 4)
    return a.pay_bytes ? launch_t<W, uint32_t, true>(a, grid, smem, st)
                       : launch_t<W, uint32_t, false>(a, grid, smem, st);
  return a.pay_bytes ? launch_t<W, uint64_t, true>(a, grid, smem, st)
                     : launch_t<W, uint64_t, false>(a, grid, smem, st);
}

cudaError_t launch_probe_gather(const ProbeArgs& a, uint32_t W, uint32_t grid, uint32_t smem,
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
