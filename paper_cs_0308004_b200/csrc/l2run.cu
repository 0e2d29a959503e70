// l2run.cu -- DPG with the run sized to the L2 cache.
//
// The paper sizes a run so that "one data run plus a rid-run buffer fit in
// cache" (section 2.1, constraints P:247-255; Fig. 1 `L <- CACHE_SIZE/2`,
// P:396), and on its IBM p690 the cache that mattered was the 128 MB L3
// (P:796-799, 846-847).  B200 has a 126 MB L2 in front of HBM.  When the
// whole source fits the L2 budget there is one run (K = 1), and the three
// phases become:
//   Phase I   Distribute: with one run, RID_RUN[0] is the rid list itself
//             (Fig. 1 P:406-411 appends every rid to run 0); nothing to do.
//   Phase II  Probe: "load the i-th INPUT run entirely into cache"
//             (P:299-302, 415-416): every CTA streams its slice of the source
//             through TMA bulk copies (L2 evict_last), so the run is read from
//             HBM once, sequentially, and stays resident in L2; a grid
//             barrier ends the load.  The CTA's chunk of the rid list is bulk-
//             copied into shared memory at the same time (the rid-run buffer).
//   Phase III Gather, fused with the probe's copy: in
//             rid order, each record is read from the L2-resident run and
//             written to the next output row, so the output is one sequential
//             write stream (stores L2 evict_first: the stream must not evict
//             the run).
// Every HBM access of the path is then sequential: the source once, the rids
// once, the output once (2*rec + 4 bytes per record).
//
// Lane layout of the gather: a warp owns 32 consecutive output rows, i.e. one
// contiguous span of 32*rec bytes of dst, viewed as 32*R words of W bytes
// (R = rec/W).  Lane l moves words l, l+32, l+64, ...: every store
// instruction writes 32 consecutive words (coalesced), and the word's row
// (w / R) selects the source record through a shuffle of the row's rid.
#include "dpg_internal.cuh"

namespace dpg {

static constexpr int kL2Threads = 512;
static constexpr int kL2Warps = kL2Threads / 32;
static constexpr uint32_t kL2Slots = 16;           // max ring slots of Phase II bulk copies
static constexpr uint32_t kL2Region = 192u << 10;  // Phase II ring, then the gather tiles
static constexpr uint32_t kL2WarpTile = 4096;                   // tile bytes per warp
static_assert(kL2WarpTile * kL2Warps <= kL2Region, "gather tiles exceed the ring");
static_assert(128 >= 8 * kL2Slots, "barrier area");


// REALIGN 0: rows are whole W-byte words (W = 16 when rec, src and dst allow):
//            flat word loop, loads and stores straight between L2 and dst.
// REALIGN 1: rows of any 4-byte multiple (e.g. the 100-byte records): each row
//            is read as the 16-byte words of its enclosing aligned window (a
//            16-byte load moves 4x the bytes of a 4-byte one per LSU
//            instruction -- measured 88 vs 34 Grow/s for L2-resident 100-byte
//            rows, profiles/r01_micro3_l2_rows.txt), realigned into the warp's
//            output tile in shared memory, and the tile (32 consecutive
//            output rows) leaves by one TMA bulk store.
// REALIGN 2: as 1 with byte granularity (rec or src not 4-byte aligned).
template <int W, int REALIGN>
__global__ void __launch_bounds__(kL2Threads, 1) k_dpg_l2run(const __grid_constant__ L2RunArgs a0) {
  L2RunArgs a = a0;
  const OutSegs& sg = a0.seg;   // (read in place: dynamic segment indices use the constant bank)
  if (a.dev_range) {
    // the rows [range[0], range[1]) of rids/dst, known on the device only (the
    // run of a K-run plan, l2k.cu): rids and dst are offset by range[0]
    const uint32_t r0 = __ldg(a.dev_range), r1 = __ldg(a.dev_range + 1);
    a.rids += r0;
    a.dst += (uint64_t)r0 * a.rec;
    a.n_out = r1 - r0;
    a.chunk = ((a.n_out + gridDim.x - 1) / gridDim.x + 31) & ~uint64_t(31);
  }
  using T = typename Word<W>::T;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);            // [kL2Slots] + rid barrier
  uint8_t* ring = smem + 128;                                    // Phase II ring / Phase III tiles
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t c = blockIdx.x, G = gridDim.x;
  if (a.ts && tid == 0) a.ts[(size_t)c * 16 + 0] = globaltimer();

  // this CTA's output rows (and rids): [lo, hi)
  const uint64_t lo = min_u64(a.n_out, (uint64_t)c * a.chunk);
  const uint64_t hi = min_u64(a.n_out, lo + a.chunk);
  if (tid == 0) {
    for (uint32_t k = 0; k < kL2Slots; ++k) mbar_init(&bar[k], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // ---- Phase II: load the run (the whole source) into L2 ----------------------
  // (one lane of warp 0 issues; the warp reconverges before any CTA barrier)
  if (warp == 0) {
  if (lane == 0) {
    const uint64_t pol_last = policy_evict_last();
    const uint64_t pol_first = policy_evict_first();
    // the CTA's slice of the source bytes, enclosing 16-byte blocks (a block
    // holding at least one source byte is mapped, so this never faults)
    const uintptr_t s0 = al_dn(reinterpret_cast<uintptr_t>(a.src));
    const uintptr_t s1 = al_up(reinterpret_cast<uintptr_t>(a.src) + a.n_src * (uint64_t)a.rec);
    const uint64_t total = a.stage_bytes ? min_u64(s1 - s0, a.stage_bytes) : s1 - s0;
    const uint64_t slice = ((total + G - 1) / G + 15) & ~uint64_t(15);
    const uint64_t b0 = min_u64(total, (uint64_t)c * slice), b1 = min_u64(total, b0 + slice);
    // ring geometry (tunable): NS slots of CH bytes, NS * CH <= kL2Region
    // (evict_normal or a 0.5 evict_last fraction kept less of the run:
    // profiles/r01_l2_stage_policy.txt)
    const uint64_t pol_stage = pol_last;
    const uint32_t CH = a.ring_chunk ? a.ring_chunk : (32u << 10);
    const uint32_t NS = a.ring_slots ? a.ring_slots : 6;
    uint32_t j = 0;
    if (a.stage && (a.dbg & 0x10000)) {
      // experiment: L2 prefetches of the slice (no shared memory, no completion)
      for (uint64_t off = b0; off < b1; off += CH)
        bulk_prefetch_l2(reinterpret_cast<const void*>(s0 + off), (uint32_t)min_u64(CH, b1 - off),
                         pol_stage);
    } else if (a.stage)
    for (uint64_t off = b0; off < b1; off += CH, ++j) {
      const uint32_t slot = j % NS;
      if (j >= NS) mbar_wait(&bar[slot], ((j / NS) - 1) & 1);
      const uint32_t bytes = (uint32_t)min_u64(CH, b1 - off);
      mbar_arrive_expect_tx(&bar[slot], bytes);
      bulk_g2s(ring + (size_t)slot * CH, reinterpret_cast<const void*>(s0 + off), bytes,
               &bar[slot], pol_stage);
    }
    // drain: the last min(j, NS) copies
    for (uint32_t q = (j > NS ? j - NS : 0); q < j; ++q)
      mbar_wait(&bar[q % NS], (q / NS) & 1);
  }
  __syncwarp();
  }
  if (a.ts && tid == 0) a.ts[(size_t)c * 16 + 1] = globaltimer();
  if (a.stage && !(a.dbg & 0x20000)) grid_barrier_mono(a.gbar + 16, G);   // (one poller: CTA 0)
  if (a.ts && tid == 0) a.ts[(size_t)c * 16 + 2] = globaltimer();

  // The rid run (this CTA's chunk of the rid list) is read group by group,
  // one coalesced 128-byte load per 32 rows, issued one group ahead.
  const uint64_t ngroups = (hi - lo + 31) / 32;
  auto rid_of = [&](uint64_t g) -> uint32_t {
    const uint64_t i = lo + g * 32 + lane;
    return (g < ngroups && i < hi) ? ldg_first(a.rids + i) : 0xFFFFFFFFu;
  };

  // ---- Phase II probe + Phase III gather, in rid order ---------------------------
  const uint64_t pol_last = policy_evict_last();
  const uint64_t pol_first = policy_evict_first();
  // loads: evict_last when the run was staged in L2 (Phase II), else evict_first
  const uint64_t pol_load = a.stage ? pol_last : pol_first;
  // the window gather: hits leave the staged lines' priority alone; a miss's
  // fill is evict_first so it does not displace the staged run (tunable)
  const uint64_t pol_gather = (a.dbg & 64) ? pol_last : pol_first;
  if (REALIGN == 0) {
    const uint32_t R = a.rec / W;
    const uint32_t q32 = 32 / R, r32 = 32 % R;     // advance of (row, word) per 32 words
    constexpr int U = W >= 16 ? 4 : 8;
    uint32_t nxt = rid_of(warp);
    for (uint64_t g = warp; g < ngroups; g += kL2Warps) {
      const uint64_t g0 = lo + g * 32;
      const uint32_t cnt = (uint32_t)min_u64(32, hi - g0);
      const uint32_t cur = nxt;
      nxt = rid_of(g + kL2Warps);
      uint32_t my_r = 0, ok = 0;
      if ((uint32_t)lane < cnt) {
        my_r = cur;
        if (my_r < a.n_src) ok = 1;
        else report_bad(a.status, g0 + lane);
      }
      const uint32_t okm = __ballot_sync(0xffffffffu, ok);
      const uint64_t nw = (uint64_t)cnt * R;          // words of this group
      uint8_t* gdst = a.dst + g0 * a.rec;
      uint32_t row = lane / R, off = lane % R;        // of word w = lane + 32*j
      for (uint64_t w0 = 0; w0 < nw; w0 += 32 * U) {
        T v[U];
        uint32_t rw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t w = w0 + 32 * u + lane;
          const uint32_t rrow = row < 32 ? row : 31;
          const uint32_t r = __shfl_sync(0xffffffffu, my_r, rrow);
          rw[u] = row;
          if (w < nw && ((okm >> rrow) & 1)) {
            const uint8_t* p = a.src + (uint64_t)r * a.rec + (uint64_t)off * W;
            v[u] = HintIO<W>::ld(p, pol_load);
          }
          row += q32;
          off += r32;
          if (off >= R) { off -= R; ++row; }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t w = w0 + 32 * u + lane;
          if (w < nw && ((okm >> (rw[u] < 32 ? rw[u] : 31)) & 1))
            HintIO<W>::st(gdst + w * W, v[u], pol_first);
        }
      }
    }
  } else if (REALIGN == 1 && a.rec >= 8 && a.rec <= 116 &&
             (reinterpret_cast<uintptr_t>(a.dst) & 3) == 0) {
    // the asynchronous window gather (dpg_internal.cuh): three groups of 32
    // rows per warp in flight through cp.async, rids loaded four groups ahead
    static_assert(3 * kAgTile * kL2Warps <= kL2Region, "window tiles exceed the region");
    uint8_t* wtiles = ring + (size_t)warp * 3 * kAgTile;
    const uint32_t wt_s = smem_u32(wtiles);
    const uintptr_t src_u = reinterpret_cast<uintptr_t>(a.src);
    AgrMap amap;
    agr_map_init(amap, a.rec, lane);
    const uint32_t ng = (uint32_t)ngroups;
    const uint32_t nt = ng > (uint32_t)warp ? (ng - warp + kL2Warps - 1) / kL2Warps : 0;
    auto rid_load = [&](uint32_t t) -> uint32_t {
      const uint64_t i = lo + 32 * (uint64_t)(warp + t * kL2Warps) + lane;
      return (t < nt && i < hi) ? ldg_first(a.rids + i) : 0xFFFFFFFFu;
    };
    uint32_t rq0 = rid_load(0), rq1 = rid_load(1), rq2 = rid_load(2), rq3 = rid_load(3);
    auto grp = [&](uint32_t t) -> AgrGroup {
      const uint32_t r = rq0;
      rq0 = rq1;
      rq1 = rq2;
      rq2 = rq3;
      rq3 = rid_load(t + 4);
      AgrGroup q;
      const uint64_t g0 = lo + 32 * (uint64_t)(warp + t * kL2Warps);
      q.cnt = (uint32_t)min_u64(32, hi - g0);
      const bool on = r < a.n_src;
      if ((uint32_t)lane < q.cnt && !on) report_bad(a.status, g0 + lane);
      q.r = on ? r : 0u;          // (row 0 is read, not stored)
      q.okm = __ballot_sync(0xffffffffu, on);
      q.g0 = g0;
      if (!sg.n) {
        q.out = reinterpret_cast<uint32_t*>(a.dst + g0 * a.rec);
      } else {
        // output segments: the group's rows in one segment store as usual
        const uint32_t qa = seg_of(sg, g0), qb = seg_of(sg, g0 + q.cnt - 1);
        q.out = qa == qb ? reinterpret_cast<uint32_t*>(sg.out[qa] + (g0 - sg.start[qa]) * a.rec)
                         : nullptr;
      }
      return q;
    };
    // a group across output segments: one masked dword store per segment, the
    // span placed so that row j lands at its segment's row (g0 + j - start)
    auto split = [&](const AgrGroup& q, const uint32_t* tile, uint32_t o4) {
      const uint64_t g0 = q.g0;
      const uint32_t qa = seg_of(sg, g0), qb = seg_of(sg, g0 + q.cnt - 1);
      for (uint32_t sq = qa; sq <= qb; ++sq) {
        const uint64_t s0 = sg.start[sq], s1 = sg.start[sq + 1];
        const uint32_t j0 = (uint32_t)(max_u64(s0, g0) - g0), j1 = (uint32_t)min_u64(s1 - g0, 32);
        const uint32_t m = (j1 >= 32 ? 0xffffffffu : ((1u << j1) - 1u)) & ~((1u << j0) - 1u);
        uint8_t* out = sg.out[sq] + (int64_t)(g0 - s0) * (int64_t)a.rec;
        ag_consume(tile, o4, q.okm & m, q.cnt, a.rec, reinterpret_cast<uint32_t*>(out), lane);
      }
    };
    if (a.n_src * a.rec + 16 <= 0xFFFFFFFFull)
      agr_pipeline<true>(nt, grp, split, wtiles, wt_s, kAgTile, amap, src_u, a.rec, lane, a.dbg);
    else
      agr_pipeline<false>(nt, grp, split, wtiles, wt_s, kAgTile, amap, src_u, a.rec, lane, a.dbg);
    // rows written into peer memory (output segments mapped from other GPUs)
    // are made visible system-wide before the kernel ends
    if (sg.n) __threadfence_system();
  } else {
    const uint32_t rec = a.rec;
    const uint32_t NW = (rec + 30) / 16;            // 16-byte words of a row's window (max)
    const uint32_t RPI = 32 / NW;                   // rows per load instruction
    const uint32_t lr = lane / NW, lw = lane % NW;
    const uint32_t nbuf = rec <= 64 ? 2 : 1;
    const uint32_t tile_bytes = 32 * rec;
    uint8_t* tiles = ring + (size_t)warp * kL2WarpTile;
    constexpr int U = 8;
    // fast path (whole groups of valid rows, rec % 4 == 0, rec <= 116): each
    // 16-byte window word is stored by dwords straight into the output layout
    // of the warp's tile (row jj at byte jj*rec; the dwords outside the row
    // are dropped), then the tile leaves as aligned 16-byte words.
    const uintptr_t src_u = reinterpret_cast<uintptr_t>(a.src);
    const bool fast_ok = REALIGN == 1 && rec <= 116 && rec >= 8;
    const uint32_t FNW = (rec + 12 + 15) / 16;       // window words a row can need
    const uint32_t FRPI = 32 / FNW, flr = lane / FNW, flw = lane % FNW;
    uint32_t* ot = reinterpret_cast<uint32_t*>(tiles);
    const uint32_t ot_s = smem_u32(ot);
    const uint32_t RD = rec >> 2;                     // dwords per row
    uint32_t on_mask = 0;                             // bit u: lane holds a row in load u
#pragma unroll
    for (int u = 0; u < 8; ++u) on_mask |= (uint32_t)(flr < FRPI && u * FRPI + flr < 32) << u;
    uint32_t gi = 0;
    uint32_t nxt = rid_of(warp);
    for (uint64_t g = warp; g < ngroups; g += kL2Warps, ++gi) {
      const uint64_t g0 = lo + g * 32;
      const uint32_t cnt = (uint32_t)min_u64(32, hi - g0);
      const uint32_t cur = nxt;
      nxt = rid_of(g + kL2Warps);
      uint32_t my_r = 0, ok = 0;
      if ((uint32_t)lane < cnt) {
        my_r = cur;
        if (my_r < a.n_src) ok = 1;
        else report_bad(a.status, g0 + lane);
      }
      const uint32_t okm = __ballot_sync(0xffffffffu, ok);
      if (fast_ok && okm == 0xffffffffu &&
          ((reinterpret_cast<uintptr_t>(a.dst) + g0 * rec) & 15) == 0) {
        if (lane == 0) bulk_wait_read<0>();          // a slow-path tile store may read here
        __syncwarp();
        uint4 v[8];
        uint32_t o4p = 0;                               // 2-bit dword offsets, load u at bit 2u
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t jj = (u * FRPI + flr) & 31;
          const uint32_t r = __shfl_sync(0xffffffffu, my_r, jj);
          const uintptr_t ra = src_u + (uint64_t)r * rec;
          const uint32_t o4 = (uint32_t)(ra >> 2) & 3;
          o4p |= o4 << (2 * u);
          ld16_pred(v[u], reinterpret_cast<const void*>((ra & ~uintptr_t(15)) + 16 * flw),
                    ((on_mask >> u) & 1) && 4 * flw < o4 + RD, pol_gather);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          // dword k of this window word is row dword 4*flw + k - o4 (kept when
          // inside [0, RD)); row jj at dword jj*RD of the tile
          const uint32_t jj = (u * FRPI + flr) & 31;
          const uint32_t d0 = 4 * flw - ((o4p >> (2 * u)) & 3);   // may wrap below 0 (then > RD)
          const uint32_t sa = ot_s + 4 * (jj * RD + d0);
          const bool on = (on_mask >> u) & 1;
          sts32_pred(sa + 0, v[u].x, on && d0 + 0 < RD);
          sts32_pred(sa + 4, v[u].y, on && d0 + 1 < RD);
          sts32_pred(sa + 8, v[u].z, on && d0 + 2 < RD);
          sts32_pred(sa + 12, v[u].w, on && d0 + 3 < RD);
        }
        __syncwarp();
        uint8_t* gdst = a.dst + g0 * rec;
        const uint32_t nwo = 2 * rec;                 // 16-byte words of 32 rows
        for (uint32_t m = lane; m < nwo; m += 32)
          st16_cs(gdst + 16 * (uint64_t)m, reinterpret_cast<const uint4*>(ot)[m]);
        __syncwarp();
        continue;
      }
      uint8_t* tile = tiles + (size_t)(gi % nbuf) * ((tile_bytes + 127) & ~127u);
      if (nbuf == 2) { if (lane == 0) bulk_wait_read<1>(); }
      else { if (lane == 0) bulk_wait_read<0>(); }
      __syncwarp();
      for (uint32_t j0 = 0; j0 < cnt; j0 += RPI * U) {
        uint4 v[U];
        uint32_t o[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t j = j0 + u * RPI + lr;
          const uint32_t jj = j < 32 ? j : 31;
          const uint32_t r = __shfl_sync(0xffffffffu, my_r, jj);
          const uintptr_t ra = reinterpret_cast<uintptr_t>(a.src) + (uint64_t)r * rec;
          o[u] = (uint32_t)(ra & 15);
          v[u] = make_uint4(0, 0, 0, 0);
          if (lr < RPI && j < cnt && ((okm >> jj) & 1) && 16 * lw < o[u] + rec)
            v[u] = HintIO<16>::ld(reinterpret_cast<const void*>(al_dn(ra) + 16 * lw), pol_load);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t j = j0 + u * RPI + lr;
          if (!(lr < RPI && j < cnt)) continue;
          const int base = (int)(16 * lw) - (int)o[u];     // row byte of the word's first byte
          uint8_t* trow = tile + j * rec;
          if (REALIGN == 1) {
            const uint32_t vw[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int sb = base + 4 * k;
              if (sb >= 0 && sb < (int)rec) *reinterpret_cast<uint32_t*>(trow + sb) = vw[k];
            }
          } else {
            const uint32_t vw[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              const int sb = base + k;
              if (sb >= 0 && sb < (int)rec) trow[sb] = (uint8_t)(vw[k >> 2] >> (8 * (k & 3)));
            }
          }
        }
      }
      // the tile (cnt consecutive output rows) to dst
      uint8_t* gdst = a.dst + g0 * rec;
      const uint32_t bytes = cnt * rec;
      if (a.dbg & 2) {
        __syncwarp();
      } else if ((a.dbg & 1) && okm == (cnt == 32 ? 0xffffffffu : ((1u << cnt) - 1u)) &&
          (reinterpret_cast<uintptr_t>(gdst) & 15) == 0 && (bytes & 15) == 0) {
        __syncwarp();
        for (uint32_t b = lane * 16; b < bytes; b += 512)
          HintIO<16>::st(gdst + b, *reinterpret_cast<const uint4*>(tile + b), pol_first);
        __syncwarp();
      } else if (okm == (cnt == 32 ? 0xffffffffu : ((1u << cnt) - 1u)) &&
          (reinterpret_cast<uintptr_t>(gdst) & 15) == 0 && (bytes & 15) == 0) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) bulk_s2g(gdst, tile, bytes, pol_first);
      } else {
        __syncwarp();
        // rows with a bad rid stay unwritten
        for (uint32_t b = lane; b < bytes; b += 32) {
          const uint32_t j = b / rec;
          if ((okm >> j) & 1) gdst[b] = tile[b];
        }
        __syncwarp();
      }
    }
    if (lane == 0) bulk_wait_all();
  }
  if (a.ts) {
    __syncthreads();
    if (tid == 0) a.ts[(size_t)c * 16 + 3] = globaltimer();
  }
}

template <int W, int REALIGN>
static cudaError_t launch_l2_w(const L2RunArgs& a, uint32_t grid, uint32_t smem, cudaStream_t st) {
  auto fn = k_dpg_l2run<W, REALIGN>;
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
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kL2Threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  int na = 0;
  at[na].id = cudaLaunchAttributeCooperative;   // the grid barrier ends Phase II
  at[na].val.cooperative = a.stage ? 1 : 0;
  ++na;
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, fn, a);
}

uint32_t l2run_smem_bytes(uint64_t) { return 128 + kL2Region; }

cudaError_t launch_l2run(const L2RunArgs& a, uint32_t W, uint32_t grid, cudaStream_t st,
                         uint32_t* nl) {
  ++*nl;
  const uint32_t smem = l2run_smem_bytes(a.chunk);
  if (W == 16) return launch_l2_w<16, 0>(a, grid, smem, st);
  if (W == 8) return launch_l2_w<8, 0>(a, grid, smem, st);
  // rows of one 4-byte word (the rid gather of the batch lookup): the flat
  // word loop, one row per lane
  if (W == 4 && a.rec == 4) return launch_l2_w<4, 0>(a, grid, smem, st);
  if (a.rec <= 128) {
    const bool word4 = a.rec % 4 == 0 && reinterpret_cast<uintptr_t>(a.src) % 4 == 0;
    return word4 ? launch_l2_w<16, 1>(a, grid, smem, st) : launch_l2_w<16, 2>(a, grid, smem, st);
  }
  switch (W) {
    case 8: return launch_l2_w<8, 0>(a, grid, smem, st);
    case 4: return launch_l2_w<4, 0>(a, grid, smem, st);
    case 2: return launch_l2_w<2, 0>(a, grid, smem, st);
    default: return launch_l2_w<1, 0>(a, grid, smem, st);
  }
}

}  // namespace dpg
