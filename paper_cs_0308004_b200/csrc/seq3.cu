// seq3.cu -- DPG with shared-memory runs in three sequential passes (path 6).
//
// Fig. 1 of the paper with every phase a sequential stream and
// the random accesses inside on-chip memory -- the form the paper argues for
// (P:227-230, 278-281, 299-302, 317-319), and the one that pays on B200 where
// a random access costs more than the record: a whole HBM transfer unit and
// one L2 request per record, while the L2 serves only ~175-210 G requests/s
// (profiles/r02_ncu_seq3_v1.md).
//
// Tile-major layout.  The rid list is cut into tiles of T rids (T * rec fits
// one shared-memory buffer).  Every intermediate is stored tile by tile, and
// inside a tile run by run:
//
//   RID_RUN   loc[t*T + pre[t][b] + k] = k-th rid of tile t in run b, as its
//             local offset rid - b*L (16 bits)
//   INTERNAL  internal[(t*T + pre[t][b] + k) * rec] = that rid's record
//   tinv[i]   position of row i's entry inside its tile (16 bits; 0xFFFF for
//             an invalid rid)
//   pre[t][b] exclusive prefix over runs of tile t's run counts (b <= K; the
//             entries of invalid rids sit after pre[t][K]); preT its transpose
//
//   Phase I  (distribute), k3_distribute: a CTA takes a
//            tile (rids staged by one TMA bulk copy), counts its runs in
//            shared memory, scans the counts, places every rid's local offset
//            at its run's next slot in shared memory, and writes the sorted
//            tile, tinv and pre[t] as contiguous blocks.  One pass over the
//            rids; every global write is coalesced.  Run b's RID_RUN is the
//            concatenation of its pieces (t, b), t = 0, 1, ...
//   Phase II (probe), k3_probe: a CTA stages run b --
//            records [b*L, (b+1)*L), at most one stage -- into shared memory
//            with one TMA bulk copy (its next run is prefetched into L2
//            meanwhile), reads run b's column of preT, and for every entry of
//            every piece copies INPUT[local] to the entry's INTERNAL slot.
//   Phase III (gather), k3_gather: a CTA loads tile t's
//            INTERNAL block (one TMA bulk copy, double-buffered) and writes
//            the tile's output rows in order, dst[i] = block[tinv[i]]
//            (join: pay[i] ++ block[tinv[i]]), coalesced.
//
// Bytes per row: Phase I 4 + 2 + 2 (rids, RID_RUN, tinv), Phase II 2 + rec +
// rec, Phase III 2 + rec + rec (+ pay read): 12 + 4 rec, plus the pre tables
// ((K + 1) * 4 / T bytes per row).  Inside a piece the entries follow shared-
// memory atomic order (reading A15): the pieces are in tile order, the set of
// each piece is unique, and every row's slot is recorded, so the output does
// not depend on the order.
#include <algorithm>

#include "dpg_internal.cuh"

namespace dpg {

static constexpr uint16_t kNoSlot = 0xFFFF;

// ---- Phase I: distribute each tile into its runs ----------------------------
static constexpr int k3DistThreads = 512;
// the plan's kernels after the first are launched with PDL (pdl_wait), no
// early trigger: each starts as its predecessor's CTAs exit, hiding the launch
// gap (path 6, 4 launches: -5 to -9 us per call; triggering at kernel start
// was slower, up to +100 us at 32-byte records: profiles/r02_pdl.md).  The
// tuning flag 0x40000 launches them plainly (A/B)
static bool seq3_pdl(const Seq3Args& a) { return !(a.dbg & 0x40000u); }

uint32_t seq3_dist_smem(uint32_t T, uint32_t K) {
  return (uint32_t)(256 + (uint64_t)T * 4 + (((uint64_t)T * 2 + 15) & ~15ull) +
                    2 * (((uint64_t)K + 1) * 4 + 16));
}

// Exclusive scan of v[0, n) in place (one CTA); returns the total.
__device__ uint32_t block_scan_inplace(uint32_t* v, uint32_t n, uint32_t* warp_tot) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nth = blockDim.x;
  const uint32_t per = (n + nth - 1) / nth;
  const uint32_t b0 = min(n, tid * per), b1 = min(n, b0 + per);
  uint32_t s = 0;
  for (uint32_t j = b0; j < b1; ++j) s += v[j];
  uint32_t x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const uint32_t nw = nth >> 5;
    const uint32_t w = lane < nw ? warp_tot[lane] : 0;
    uint32_t ws = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, ws, o);
      if (lane >= o) ws += y;
    }
    if (lane < nw) warp_tot[lane] = ws - w;
    if (lane == 31) warp_tot[32] = ws;
  }
  __syncthreads();
  uint32_t run = warp_tot[warp] + x - s;
  for (uint32_t j = b0; j < b1; ++j) {
    const uint32_t c = v[j];
    v[j] = run;
    run += c;
  }
  const uint32_t total = warp_tot[32];
  __syncthreads();
  return total;
}

template <bool DBG>
__global__ void __launch_bounds__(k3DistThreads) k3_distribute(Seq3Args a) {
  extern __shared__ __align__(128) uint8_t smd[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smd);
  uint32_t* wtot = reinterpret_cast<uint32_t*>(smd + 16);       // [33]
  uint32_t* srid = reinterpret_cast<uint32_t*>(smd + 256);      // [T]
  uint16_t* sloc = reinterpret_cast<uint16_t*>(srid + a.T);     // [T]
  uint32_t* hist = reinterpret_cast<uint32_t*>(smd + 256 + (uint64_t)a.T * 4 +
                                               (((uint64_t)a.T * 2 + 15) & ~15ull));  // [K+1]
  uint32_t* scur = hist + ((a.K + 1 + 3) & ~3u);                // [K+1]
  const uint32_t tid = threadIdx.x, nth = blockDim.x, K = a.K, T = a.T, sh = a.s;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol_first = policy_evict_first();
  const uint32_t lmask = (1u << sh) - 1u;
  // rids are uint32: valid iff rid <= n_src - 1 (n_src <= 2^32)
  const uint32_t rid_max = (uint32_t)min_u64(a.n_src - 1, 0xFFFFFFFFull);
  const bool tma_ok = ((uintptr_t)a.rids % 16) == 0;
  uint32_t phase = 0;
  for (uint32_t t = blockIdx.x; t < a.nsub; t += gridDim.x) {
    const uint64_t i0 = (uint64_t)t * T;
    const uint32_t nt = (uint32_t)min_u64(T, a.n_out - i0);
    // the tile's rids into shared memory (one bulk copy of the aligned part)
    const uint32_t nbulk = tma_ok ? (nt & ~3u) : 0;
    if (tid == 0) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(bar, nbulk * 4);
      for (uint32_t off = 0; off < nbulk * 4; off += 32768)
        bulk_g2s(reinterpret_cast<uint8_t*>(srid) + off,
                 reinterpret_cast<const uint8_t*>(a.rids + i0) + off,
                 min(32768u, nbulk * 4 - off), bar, pol_first);
    }
    for (uint32_t j = nbulk + tid; j < ((nt + 3) & ~3u); j += nth)
      srid[j] = j < nt ? a.rids[i0 + j] : 0xFFFFFFFFu;      // pad to 4: bucket K, not stored
    for (uint32_t b = tid; b <= K; b += nth) hist[b] = 0;
    mbar_wait(bar, phase);
    phase ^= 1;
    __syncthreads();
    const uint32_t n4 = (nt + 3) / 4, nfull = nt / 4;
    const uint4* srid4 = reinterpret_cast<const uint4*>(srid);
    // count: run b = rid >> s; invalid rids go to bucket K
    for (uint32_t q = tid; q < n4; q += nth) {
      const uint4 r4 = srid4[q];
      if (q < nfull && max(max(r4.x, r4.y), max(r4.z, r4.w)) <= rid_max) {
        // (the common case, without per-rid branches: four valid rids)
        atomicAdd(&hist[r4.x >> sh], 1u);
        atomicAdd(&hist[r4.y >> sh], 1u);
        atomicAdd(&hist[r4.z >> sh], 1u);
        atomicAdd(&hist[r4.w >> sh], 1u);
        continue;
      }
      const uint32_t r[4] = {r4.x, r4.y, r4.z, r4.w};
      if (q < nfull) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const bool ok = r[k] <= rid_max;
          if (!ok) report_bad(a.status, i0 + 4 * q + k);
          atomicAdd(&hist[ok ? (r[k] >> sh) : K], 1u);
        }
      } else {
        for (int k = 0; k < 4; ++k) {
          if (4 * q + k >= nt) break;
          const bool ok = r[k] <= rid_max;
          if (!ok) report_bad(a.status, i0 + 4 * q + k);
          atomicAdd(&hist[ok ? (r[k] >> sh) : K], 1u);
        }
      }
    }
    __syncthreads();
    block_scan_inplace(hist, K + 1, wtot);            // hist -> pre[t][b]
    uint16_t* pre_g = a.pre + (uint64_t)t * (K + 1);
    for (uint32_t b = tid; b <= K; b += nth) {
      const uint32_t p = hist[b];
      scur[b] = p;
      pre_g[b] = (uint16_t)p;
    }
    __syncthreads();
    // place: "Append r to RID_RUN[run_num]", inside the tile's block
    uint2* tinv4 = reinterpret_cast<uint2*>(a.tinv + i0);   // i0 % 4 == 0 (T % 16 == 0)
    for (uint32_t q = tid; q < n4; q += nth) {
      const uint4 r4 = srid4[q];
      if (!DBG && q < nfull && max(max(r4.x, r4.y), max(r4.z, r4.w)) <= rid_max) {
        const uint32_t s0 = atomicAdd(&scur[r4.x >> sh], 1u);
        const uint32_t s1 = atomicAdd(&scur[r4.y >> sh], 1u);
        const uint32_t s2 = atomicAdd(&scur[r4.z >> sh], 1u);
        const uint32_t s3 = atomicAdd(&scur[r4.w >> sh], 1u);
        sloc[s0] = (uint16_t)(r4.x & lmask);
        sloc[s1] = (uint16_t)(r4.y & lmask);
        sloc[s2] = (uint16_t)(r4.z & lmask);
        sloc[s3] = (uint16_t)(r4.w & lmask);
        tinv4[q] = make_uint2(s0 | (s1 << 16), s2 | (s3 << 16));
        continue;
      }
      const uint32_t r[4] = {r4.x, r4.y, r4.z, r4.w};
      const uint32_t kn = q < nfull ? 4u : nt - 4 * q;
      uint32_t sl[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool ok = r[k] <= rid_max;
        sl[k] = kNoSlot;
        if (k < (int)kn) {
          const uint32_t slot = atomicAdd(&scur[ok ? (r[k] >> sh) : K], 1u);
          sloc[slot] = (uint16_t)(r[k] & lmask);
          if (ok) sl[k] = slot;
          if (DBG && ok) a.dbg_pairs[i0 + slot] = (uint64_t)(r[k] & lmask) | ((i0 + 4 * q + k) << 32);
        }
      }
      const uint2 v = make_uint2(sl[0] | (sl[1] << 16), sl[2] | (sl[3] << 16));
      if (kn == 4) {
        tinv4[q] = v;
      } else {
        for (int k = 0; k < (int)kn; ++k) a.tinv[i0 + 4 * q + k] = (uint16_t)sl[k];
      }
    }
    __syncthreads();
    // the sorted tile leaves as one block (16-byte words; T % 8 == 0)
    const uint32_t nv = hist[K];
    uint4* lo = reinterpret_cast<uint4*>(a.loc + i0);
    const uint4* ls = reinterpret_cast<const uint4*>(sloc);
    for (uint32_t w = tid; w < (nv + 7) / 8; w += nth) lo[w] = ls[w];
    __syncthreads();
  }
}

// pre (nsub x (K+1), u16) -> preT ((K+1) x nsub), 32 x 32 tiles
__global__ void k3_transpose(const uint16_t* __restrict__ in, uint16_t* __restrict__ out,
                             uint32_t rows, uint32_t cols) {
  __shared__ uint16_t tile[32][33];
  const uint32_t c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  pdl_wait();
  for (uint32_t y = threadIdx.y; y < 32; y += blockDim.y) {
    const uint32_t r = r0 + y, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[y][threadIdx.x] = in[(uint64_t)r * cols + c];
  }
  __syncthreads();
  for (uint32_t y = threadIdx.y; y < 32; y += blockDim.y) {
    const uint32_t c = c0 + y, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[(uint64_t)c * rows + r] = tile[threadIdx.x][y];
  }
}

cudaError_t launch_seq3_distribute(const Seq3Args& a, uint32_t grid, cudaStream_t st,
                                   uint32_t* nl) {
  const uint32_t smem = seq3_dist_smem(a.T, a.K);
  auto kern = a.dbg_pairs ? k3_distribute<true> : k3_distribute<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, k3DistThreads, smem, st>>>(a);
  ++*nl;
  dim3 tg((a.K + 1 + 31) / 32, (a.nsub + 31) / 32);
  e = launch_pdl(k3_transpose, tg, dim3(32, 8), 0, st, seq3_pdl(a), 1, a.pre, a.preT, a.nsub,
                 a.K + 1);
  ++*nl;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// ---- Phase II: probe each run in shared memory into INTERNAL -----------------
static constexpr int k3ProbeThreads = 1024;
static constexpr uint32_t k3Reg = 512;      // entries of one warp's list

uint32_t seq3_probe_smem(uint64_t stage_bytes) {
  return (uint32_t)(256 + (k3ProbeThreads / 32) * k3Reg * 4 + ((stage_bytes + 127) & ~127ull));
}

// Phase II.  Per run: the stage by TMA (the CTA's next run prefetched into L2
// meanwhile); then every warp takes 32 pieces at a time (lane q: piece (t, b)
// with t = 32 g + q, its start and length from run b's column of preT),
// scans their lengths with shuffles, writes the pieces' RID_RUN slots into
// its own shared-memory list (pieces that do not fit go in the next round),
// and copies the records of the list: INTERNAL[slot] = stage[RID_RUN[slot]].
// Consecutive list entries of a piece are consecutive slots, so a warp's
// loads of RID_RUN and stores of INTERNAL touch a few contiguous ranges.
// (Measured alternatives -- per-warp mbarrier pipelines over the stage, lists
// filled by cp.async, one lane group per piece, CTA-wide entry windows -- were
// slower: profiles/r02_seq3_phase2_variants.md.)
// Cluster-wide barrier (all threads of every CTA of the cluster), release /
// acquire: the shared memory of every CTA is then visible cluster-wide.
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// Generic address of `p` (this CTA's shared memory) in CTA `rank` of the cluster.
__device__ __forceinline__ const uint8_t* map_cluster(const uint8_t* p, uint32_t rank) {
  uint64_t r;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(r) : "l"(p), "r"(rank));
  return reinterpret_cast<const uint8_t*>(r);
}

// CL > 1 (section 8(f) #1 of the survey: larger on-chip regions): a cluster
// of CL CTAs on CL SMs holds one run of L = 2^s records together, CTA r its
// slice [r L/CL, (r+1) L/CL) in its own stage; a lookup of local offset l
// reads the stage of CTA l / (L/CL) through distributed shared memory.  The
// run's pieces are shared among all the cluster's warps; cluster barriers
// order every slice's landing before the lookups and every lookup before the
// next run's bulk copies.
template <int WB, int M, int CL>
__global__ void __launch_bounds__(k3ProbeThreads, 1) k3_probe(Seq3Args a) {
  using W = typename Word<WB>::T;
  extern __shared__ __align__(128) uint8_t smp[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smp);
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  uint32_t* reg = reinterpret_cast<uint32_t*>(smp + 256) + warp * k3Reg;
  uint8_t* stage = smp + 256 + (k3ProbeThreads / 32) * k3Reg * 4;
  pdl_wait();
  const uint32_t cr = CL > 1 ? cluster_ctarank() : 0;
  const uint32_t cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  const uint8_t* sbase[CL];
#pragma unroll
  for (int r = 0; r < CL; ++r) sbase[r] = CL > 1 ? map_cluster(stage, r) : stage;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol_first = policy_evict_first();
  // the next run, prefetched into L2 while this one is probed, is kept there
  // until its bulk copy reads it (evict_first lost ~half of it at 2^26 records)
  const uint64_t pol_keep = policy_evict_last();
  const uint64_t L = 1ull << a.s;
  const uint64_t Ls = L / CL;                     // records of one CTA's slice
  const uint32_t ls_shift = a.s - (CL == 8 ? 3 : CL == 4 ? 2 : CL == 2 ? 1 : 0);
  const uint32_t rec = a.rec, m = M ? M : rec / WB, T = a.T, nsub = a.nsub;
  uint32_t phase = 0, it = 0;
  for (uint32_t b = cid; b < a.K; b += ncl, ++it) {
    const uint64_t r0 = ((uint64_t)b << a.s) + cr * Ls;      // this CTA's slice of run b
    const uint32_t bytes = r0 < a.n_src ? (uint32_t)(min_u64(Ls, a.n_src - r0) * rec) : 0u;
    const uint32_t bulk = bytes & ~15u;
    const uint8_t* gsrc = a.src + r0 * rec;
    if (a.ts && tid == 0 && it < 16) a.ts[(blockIdx.x * 16 + it) * 4 + 0] = globaltimer();
    if (tid == 0) {
      // "Read into memory all records in the i-th run of INPUT_REC"
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(bar, bulk);
      for (uint32_t off = 0; off < bulk; off += 32768)
        bulk_g2s(stage + off, gsrc + off, min(32768u, bulk - off), bar, pol_first);
      const uint32_t bn = b + ncl;           // the cluster's next run, on its way to L2
      if (bn < a.K) {
        const uint64_t rn = ((uint64_t)bn << a.s) + cr * Ls;
        const uint32_t nb = rn < a.n_src ? (uint32_t)(min_u64(Ls, a.n_src - rn) * rec) & ~15u : 0u;
        for (uint32_t off = 0; off < nb; off += 32768)
          bulk_prefetch_l2(a.src + rn * rec + off, min(32768u, nb - off), pol_keep);
      }
    }
    for (uint32_t t = bulk + tid; t < bytes; t += blockDim.x) stage[t] = gsrc[t];   // < 16 B
    const uint16_t* colA = a.preT + (uint64_t)b * nsub;
    const uint16_t* colB = colA + nsub;
    // this warp's pieces: an equal share [p_lo, p_hi) of the run's nsub pieces
    // among the cluster's warps, 32 at a time; the first group's column
    // entries loaded before the stage wait
    const uint32_t gw = cr * nwarp + warp, ngw = nwarp * CL;
    const uint32_t ppw = (nsub + ngw - 1) / ngw;
    const uint32_t p_lo = min(nsub, gw * ppw), p_hi = min(nsub, p_lo + ppw);
    uint32_t g = p_lo;
    uint32_t t = g + lane;
    uint32_t pa = t < p_hi ? colA[t] : 0u, pb = t < p_hi ? colB[t] : 0u;
    mbar_wait(bar, phase);
    phase ^= 1;
    if (CL > 1) cluster_sync_all();   // every slice of run b landed (and the tail bytes)
    else __syncthreads();             // (the tail bytes)
    if (a.ts && tid == 0 && it < 16) a.ts[(blockIdx.x * 16 + it) * 4 + 1] = globaltimer();
    // "For each rid r in RID_RUN[i]: append INPUT_REC[r] to RECORD_RUN[i]"
    //
    for (; g < p_hi; g += 32) {
      const uint32_t len = pb - pa, st = t * T + pa;
      // the next group's column entries, in flight during this group
      const uint32_t tn = g + 32 + lane;
      pa = tn < p_hi ? colA[tn] : 0u;
      pb = tn < p_hi ? colB[tn] : 0u;
      t = tn;
      uint32_t inc = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      // lanes [lo, hi) whose pieces fit the list together, in turn
      for (uint32_t lo = 0; lo < 32;) {
        const uint32_t off = lo ? __shfl_sync(0xffffffffu, inc, lo - 1) : 0u;
        const uint32_t rinc = inc - off;
        const uint32_t hi = lo + __popc(__ballot_sync(0xffffffffu, lane >= lo && rinc <= k3Reg));
        if (hi == lo) {
          // a piece longer than the list (skewed rids): lanes over its words
          const uint32_t sq = __shfl_sync(0xffffffffu, st, lo);
          const uint32_t lq = __shfl_sync(0xffffffffu, len, lo);
          for (uint32_t j = lane; j < lq * m; j += 32) {
            const uint32_t e = j / m, w = j - e * m;
            const uint32_t l = __ldcs(a.loc + sq + e);
            const uint8_t* from = CL > 1 ? sbase[l >> ls_shift] + (l & (Ls - 1)) * rec
                                         : stage + l * rec;
            reinterpret_cast<W*>(a.internal + (uint64_t)(sq + e) * rec)[w] =
                reinterpret_cast<const W*>(from)[w];
          }
          ++lo;
          continue;
        }
        if (lane >= lo && lane < hi)
          for (uint32_t e = 0; e < len; ++e) reg[rinc - len + e] = st + e;
        __syncwarp();
        const uint32_t nw = __shfl_sync(0xffffffffu, rinc, hi - 1) * m;
        constexpr int U = 12;   // a list's RID_RUN loads in flight together
        for (uint32_t j0 = lane; j0 < nw; j0 += 32 * U) {
          uint32_t sl[U], l[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t j = j0 + 32 * u;
            sl[u] = j < nw ? reg[M == 1 ? j : j / m] : 0u;
            // (dbg 0x10000 / 0x20000: tuning experiments that drop the RID_RUN
            // loads / the INTERNAL stores; the output is then wrong)
            l[u] = j < nw ? ((a.dbg & 0x10000) ? (sl[u] & 1023u) : (uint32_t)__ldcs(a.loc + sl[u])) : 0u;
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t j = j0 + 32 * u;
            if (j >= nw) continue;
            const uint32_t w = M == 1 ? 0 : j - (j / m) * m;
            const uint8_t* from = CL > 1 ? sbase[l[u] >> ls_shift] + (l[u] & (Ls - 1)) * rec
                                         : stage + l[u] * rec;
            const W v = reinterpret_cast<const W*>(from)[w];
            if (a.dbg & 0x20000) {
              if (l[u] == 0xFFFFFFFFu) reinterpret_cast<W*>(a.internal)[0] = v;
            } else {
              // (streaming store: INTERNAL is read back only after the whole
              // Phase II, so it need not displace the staged runs' lines)
              __stcs(reinterpret_cast<W*>(a.internal + (uint64_t)sl[u] * rec) + w, v);
            }
          }
        }
        __syncwarp();
        lo = hi;
      }
    }
    // the stage is rewritten for the next run (CL > 1: once no CTA of the
    // cluster reads it any more)
    if (CL > 1) cluster_sync_all();
    else __syncthreads();
    if (a.ts && tid == 0 && it < 16) a.ts[(blockIdx.x * 16 + it) * 4 + 2] = globaltimer();
  }
}

template <int WB, int M, int CL>
static cudaError_t launch_probe_wc(const Seq3Args& a, uint32_t grid, uint32_t smem,
                                   cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(k3_probe<WB, M, CL>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (CL == 1)
    return launch_pdl(k3_probe<WB, M, 1>, dim3(grid), dim3(k3ProbeThreads), smem, st,
                      seq3_pdl(a), 1, a);
  // clusters of CL CTAs, as many as can be resident at once
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(k3ProbeThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(CL);
  int nclusters = 0;
  e = cudaOccupancyMaxActiveClusters(&nclusters, (void*)k3_probe<WB, M, CL>, &cfg);
  if (e != cudaSuccess || nclusters <= 0) {
    cudaGetLastError();
    nclusters = (int)(grid / CL);
  }
  const uint32_t runs = a.K;
  const uint32_t ncl = (uint32_t)std::max(1, std::min<int>(nclusters, (int)std::max(1u, runs)));
  return launch_pdl(k3_probe<WB, M, CL>, dim3(ncl * CL), dim3(k3ProbeThreads), smem, st,
                    seq3_pdl(a), CL, a);
}

template <int WB, int M>
static cudaError_t launch_probe_w(const Seq3Args& a, uint32_t grid, uint32_t smem,
                                  cudaStream_t st) {
  switch (a.cl) {
    case 2: return launch_probe_wc<WB, M, 2>(a, grid, smem, st);
    case 4: return launch_probe_wc<WB, M, 4>(a, grid, smem, st);
    case 8: return launch_probe_wc<WB, M, 8>(a, grid, smem, st);
    default: return launch_probe_wc<WB, M, 1>(a, grid, smem, st);
  }
}

cudaError_t launch_seq3_probe(const Seq3Args& a, uint32_t W, uint32_t grid, cudaStream_t st,
                              uint32_t* nl) {
  // each CTA stages a slice of L / cl records
  const uint32_t smem = seq3_probe_smem((((uint64_t)1 << a.s) / std::max(1u, a.cl)) * a.rec);
  cudaError_t e;
  const uint32_t m = a.rec / W;
  if (W == 4 && m == 1) e = launch_probe_w<4, 1>(a, grid, smem, st);
  else if (W == 8 && m == 1) e = launch_probe_w<8, 1>(a, grid, smem, st);
  else if (W == 16 && m == 1) e = launch_probe_w<16, 1>(a, grid, smem, st);
  else if (W == 4) e = launch_probe_w<4, 0>(a, grid, smem, st);
  else if (W == 8) e = launch_probe_w<8, 0>(a, grid, smem, st);
  else if (W == 16) e = launch_probe_w<16, 0>(a, grid, smem, st);
  else return cudaErrorInvalidValue;
  ++*nl;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// ---- Phase III: each tile's INTERNAL block -> the tile's output rows ---------
static constexpr int k3GatherThreads = 512;

__host__ __device__ static uint64_t gather_buf_bytes(uint32_t T, uint32_t rec) {
  return (((uint64_t)T * rec + 127) & ~127ull) + (((uint64_t)T * 2 + 127) & ~127ull);
}
uint32_t seq3_gather_smem(uint32_t T, uint32_t rec, uint32_t nbuf) {
  return (uint32_t)(128 + nbuf * gather_buf_bytes(T, rec));
}

// q = n / d for n < 2^32 via a 64-bit reciprocal (exact for d < 2^16).
struct FastDiv {
  uint64_t mul;
  uint32_t d;
};
static FastDiv make_div(uint32_t d) { return {UINT64_MAX / d + 1, d}; }
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return f.d == 1 ? n : (uint32_t)__umul64hi((uint64_t)n, f.mul);
}

// Tile t's INTERNAL block and its tinv both arrive by TMA into one buffer;
// output word j of the tile: row j / mr, word j % mr; words [0, mp) from
// pay[i], the rest from the block at tinv[i].
template <int WB>
__global__ void __launch_bounds__(k3GatherThreads, 1)
    k3_gather(Seq3Args a, FastDiv fr, uint32_t mp, uint32_t nbuf) {
  using W = typename Word<WB>::T;
  extern __shared__ __align__(128) uint8_t smg[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smg);   // [nbuf]
  const uint32_t T = a.T, rec = a.rec, mr = fr.d;
  const uint64_t blksz = ((uint64_t)T * rec + 127) & ~127ull;
  const uint64_t bufsz = gather_buf_bytes(T, rec);
  const uint32_t tid = threadIdx.x;
  if (tid == 0) {
    for (uint32_t k = 0; k < nbuf; ++k) mbar_init(&bar[k], 1);
    fence_mbar_init();
  }
  pdl_wait();
  __syncthreads();
  const uint64_t pol_first = policy_evict_first();
  auto issue = [&](uint32_t t, uint32_t k) {
    const uint32_t nv = a.pre[(uint64_t)t * (a.K + 1) + a.K];      // valid entries of tile t
    const uint32_t bytes = (uint32_t)(((uint64_t)nv * rec + 15) & ~15ull);
    const uint32_t nt = (uint32_t)min_u64(T, a.n_out - (uint64_t)t * T);
    const uint32_t tb = (nt * 2 + 15) & ~15u;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&bar[k], bytes + tb);
    const uint8_t* g = a.internal + (uint64_t)t * T * rec;
    uint8_t* s = smg + 128 + k * bufsz;
    for (uint32_t off = 0; off < bytes; off += 32768)
      bulk_g2s(s + off, g + off, min(32768u, bytes - off), &bar[k], pol_first);
    bulk_g2s(s + blksz, a.tinv + (uint64_t)t * T, tb, &bar[k], pol_first);
  };
  uint32_t it = 0;
  if (tid == 0 && blockIdx.x < a.nsub) issue(blockIdx.x, 0);
  for (uint32_t t = blockIdx.x; t < a.nsub; t += gridDim.x, ++it) {
    const uint32_t k = it % nbuf;
    if (nbuf > 1 && tid == 0 && t + gridDim.x < a.nsub) issue(t + gridDim.x, (it + 1) % nbuf);
    mbar_wait(&bar[k], (it / nbuf) & 1);
    const uint8_t* blk = smg + 128 + k * bufsz;
    const uint16_t* stinv = reinterpret_cast<const uint16_t*>(blk + blksz);
    const uint64_t i0 = (uint64_t)t * T;
    const uint32_t nt = (uint32_t)min_u64(T, a.n_out - i0);
    W* out = reinterpret_cast<W*>(a.dst) + i0 * mr;
    if (mp == 0 && mr == 1) {
      // one word per row: dst[i] = block[tinv[i]]
      const W* bw = reinterpret_cast<const W*>(blk);
      for (uint32_t i = tid; i < nt; i += blockDim.x) {
        const uint32_t sl = stinv[i];
        if (sl != kNoSlot) __stcs(out + i, bw[sl]);
      }
    } else {
      const uint32_t nw = nt * mr;
      const W* pay = reinterpret_cast<const W*>(a.pay) + i0 * mp;
      constexpr int U = 4;
      for (uint32_t j0 = tid; j0 < nw; j0 += U * blockDim.x) {
        W v[U];
        bool on[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t j = j0 + u * blockDim.x;
          const uint32_t i = fdiv(j, fr), q = j - i * mr;
          const uint32_t sl = j < nw ? stinv[i] : kNoSlot;
          on[u] = sl != kNoSlot;
          if (on[u])
            v[u] = q < mp ? __ldcs(pay + (uint64_t)i * mp + q)
                          : reinterpret_cast<const W*>(blk + (uint64_t)sl * rec)[q - mp];
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (on[u]) __stcs(out + j0 + u * blockDim.x, v[u]);
      }
    }
    __syncthreads();   // buffer k is reloaded nbuf tiles later
    if (nbuf == 1 && tid == 0 && t + gridDim.x < a.nsub) issue(t + gridDim.x, 0);
  }
}

cudaError_t launch_seq3_gather(const Seq3Args& a, uint32_t W, uint32_t grid, uint32_t nbuf,
                               cudaStream_t st, uint32_t* nl) {
  const uint32_t mr = (a.pay_bytes + a.rec) / W;
  const FastDiv fr = make_div(mr);
  const uint32_t mp = a.pay_bytes / W;
  const uint32_t smem = seq3_gather_smem(a.T, a.rec, nbuf);
  cudaError_t e = cudaSuccess;
#define DPG_SEQ3_GATHER(WB)                                                                   \
  case WB:                                                                                    \
    e = cudaFuncSetAttribute(k3_gather<WB>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                             (int)smem);                                                      \
    if (e == cudaSuccess)                                                                     \
      e = launch_pdl(k3_gather<WB>, dim3(grid), dim3(k3GatherThreads), smem, st, seq3_pdl(a),  \
                     1, a, fr, mp, nbuf);                                                      \
    break;
  switch (W) {
    DPG_SEQ3_GATHER(4)
    DPG_SEQ3_GATHER(8)
    DPG_SEQ3_GATHER(16)
    default: return cudaErrorInvalidValue;
  }
#undef DPG_SEQ3_GATHER
  ++*nl;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace dpg
