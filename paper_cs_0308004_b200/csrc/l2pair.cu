// l2pair.cu -- DPG with two L2-sized runs (K = 2): Fig. 1 with the L2 as the
// cache, for sources that fit twice the L2 run budget (config 2: 105 MB).
//
// The run length follows the paper's constraint (1): one data run plus its
// rid-run buffer fit in the cache.  On B200 a run staged from all
// SMs stays L2-resident up to ~60 MB (profiles/r01_l2_retention_ncu.txt), so
// a 105 MB source takes two runs of L = 2^s records.  Each CTA owns a chunk
// of the output positions [lo, hi) (a multiple of 32 rows).
//
//   kernel PHASE 0  (Phase I + Phase II of run 0)
//     - thread 0 stages run 0 (source records [0, L)) into L2 by TMA bulk
//       copies ("load the i-th INPUT run entirely into cache");
//     - meanwhile warps 1..15 distribute the chunk's rids:
//       the rids of run 0 are appended, in output order, to the chunk's
//       RID_RUN[0] buffer in shared memory (a stable warp-ballot compaction);
//     - grid barrier (run 0 resident everywhere);
//     - probe: record rid of each RID_RUN[0] entry is
//       copied from the L2-resident run to the chunk's segment of INTERNAL
//       run 0, appended sequentially.
//   kernel PHASE 1  (Phase II of run 1 fused with Phase III)
//     - thread 0 stages run 1 (records [L, n_src)); warps 1..15 recount the
//       chunk's run-0 rids per 32-row group (the same compaction, so the
//       prefix of run-0 rows before each group is known);
//     - grid barrier;
//     - gather in output order: a run-1 row is copied
//       from the L2-resident run 1 (the probe of run 1 writes its record
//       straight to the output: the last run needs no INTERNAL), a run-0 row
//       takes the next record of the chunk's INTERNAL run-0 segment.
//
// DRAM traffic per record: source once (sequential), INTERNAL run 0 written
// and read once (sequential, half the records), output once (sequential),
// rids twice; no random HBM access.  Both kernels move rows with the window
// gather of l2run.cu: 16-byte loads of each row's enclosing aligned window,
// realigned by dwords into the warp's output tile in shared memory, and the
// tile stored as aligned 16-byte words.  Requires rec % 4 == 0, 8 <= rec <=
// 116, src / INTERNAL / dst 16-byte aligned (the planner checks).
#include "dpg_internal.cuh"

namespace dpg {

static constexpr int kPThreads = 512;
static constexpr int kPWarps = kPThreads / 32;
static constexpr uint32_t kPRegion = 192u << 10;   // staging ring, then the warps' window tiles
static constexpr uint32_t kPNB = 3;                 // window tiles (groups in flight) per warp
static constexpr uint32_t kPTile = kAgTile;
static constexpr uint32_t kPSlots = 6;
static constexpr uint32_t kPChunk = 32u << 10;
static_assert(kPNB * kPTile * kPWarps <= kPRegion, "tiles exceed the region");

// One cooperative kernel for the whole path (two grid barriers).
__global__ void __launch_bounds__(kPThreads, 1) k_dpg_l2pair(L2PairArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint32_t s_carry;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  uint8_t* region = smem + 128;                     // staging ring / window tiles
  uint32_t* gcnt = reinterpret_cast<uint32_t*>(region + kPRegion);   // [ngroups + 1] group bases
  uint32_t* ent = gcnt + a.max_groups + 1;          // [chunk] RID_RUN[0] of the chunk
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t c = blockIdx.x, G = gridDim.x;
  const uint64_t lo = min_u64(a.n_out, (uint64_t)c * a.chunk);
  const uint64_t hi = min_u64(a.n_out, lo + a.chunk);
  const uint32_t ngroups = (uint32_t)((hi - lo + 31) / 32);
  const uint64_t L = min_u64(a.L, a.n_src);
#define DPG_STAMP(k) if (a.ts && tid == 0) a.ts[(size_t)c * 16 + (k)] = globaltimer();
  DPG_STAMP(0);
  if (tid == 0) {
    for (uint32_t k = 0; k < kPSlots; ++k) mbar_init(&bar[k], 1);
    fence_mbar_init();
    gcnt[ngroups] = 0;                              // an empty chunk has an empty RID_RUN[0]
  }
  __syncthreads();
  uint32_t jring = 0;                               // bulk copies issued into the ring (lane 0 of warp 0)

  if (warp == 0) {
    // ---- Phase II (run 0), first step: stage run 0 into L2 (one lane issues) ----
    if (lane == 0)
      jring = l2_stage_slice(a.src, L * a.rec, c, G, region, bar, kPChunk, kPSlots,
                             policy_evict_last(), jring);
    __syncwarp();
  } else {
    // ---- Phase I (warps 1..15), "Append r to RID_RUN[run_num]":
    // per 32-row group the number of its rids in run 0, their exclusive scan,
    // then RID_RUN[0] of the chunk in output order (a stable ballot compaction);
    // rid loads batched 8 groups deep ----
    constexpr uint32_t kW = kPWarps - 1;
    constexpr int kR = 16;                           // groups per warp held in registers
    for (uint32_t gb = 0; gb < ngroups; gb += kR * kW) {
      uint32_t r[kR];
#pragma unroll
      for (int u = 0; u < kR; ++u) {
        const uint32_t g = gb + warp - 1 + u * kW;
        const uint64_t i = lo + 32 * (uint64_t)g + lane;
        r[u] = (g < ngroups && i < hi) ? ldg_first(a.rids + i) : 0xFFFFFFFFu;
      }
#pragma unroll
      for (int u = 0; u < kR; ++u) {
        const uint32_t g = gb + warp - 1 + u * kW;
        if (g >= ngroups) break;
        const uint32_t m0 = __ballot_sync(0xffffffffu, r[u] < L);
        if (lane == 0) gcnt[g] = __popc(m0);
        const uint64_t i = lo + 32 * (uint64_t)g + lane;
        if (i < hi && r[u] >= a.n_src) report_bad(a.status, i);
      }
      named_sync(1, kPThreads - 32);
      if (warp == 1) {
        // exclusive scan of this batch's group counts, continuing the previous batch
        uint32_t carry = gb ? s_carry : 0;           // total of the previous batches
        const uint32_t ge = min(ngroups, gb + kR * kW);
        for (uint32_t g0 = gb; g0 < ge; g0 += 32) {
          const uint32_t g = g0 + lane;
          const uint32_t x = g < ge ? gcnt[g] : 0;
          uint32_t y = x;
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const uint32_t tt = __shfl_up_sync(0xffffffffu, y, d);
            if (lane >= d) y += tt;
          }
          if (g < ge) gcnt[g] = carry + y - x;
          carry += __shfl_sync(0xffffffffu, y, 31);
        }
        if (lane == 0) {
          s_carry = carry;
          if (ge == ngroups) gcnt[ngroups] = carry;  // the chunk's RID_RUN[0] length
        }
      }
      named_sync(1, kPThreads - 32);
#pragma unroll
      for (int u = 0; u < kR; ++u) {
        const uint32_t g = gb + warp - 1 + u * kW;
        if (g >= ngroups) break;
        const bool in0 = r[u] < L;
        const uint32_t m0 = __ballot_sync(0xffffffffu, in0);
        if (in0) ent[gcnt[g] + __popc(m0 & lanemask_lt())] = r[u];
      }
      named_sync(1, kPThreads - 32);             // s_carry is read by the next batch
    }
  }
  __syncthreads();
  DPG_STAMP(1);
  grid_barrier_mono(a.gbar + 16, G);
  DPG_STAMP(2);

  // window tiles of this warp: 3 groups in flight (cp.async), one consumed
  uint8_t* wtiles = region + (size_t)warp * kPNB * kPTile;
  const uint32_t wt_s = smem_u32(wtiles);
  const uintptr_t src_u = reinterpret_cast<uintptr_t>(a.src);
  uint8_t* seg = a.internal + (uint64_t)c * a.chunk * a.rec;     // the chunk's INTERNAL run-0 segment
  const uintptr_t seg_u = reinterpret_cast<uintptr_t>(seg);
  AgMap amap;
  ag_map_init(amap, a.rec, lane);
  auto pipeline = [&](uint32_t nt, auto group) {
    ag_pipeline(nt, group, wtiles, wt_s, kPTile, amap, a.rec, lane);
  };

  // ---- Phase II (run 0), second step, the probe:
  // INTERNAL[seg + k] = R[RID_RUN[0][k]], appended sequentially ----
  {
    const uint32_t n0 = gcnt[ngroups];
    const uint32_t ng = (n0 + 31) / 32;
    const uint32_t nt = ng > (uint32_t)warp ? (ng - warp + kPWarps - 1) / kPWarps : 0;
    pipeline(nt, [&](uint32_t t) -> AgGroup {
      AgGroup q;
      const uint32_t k0 = 32 * (warp + t * kPWarps);
      q.cnt = min(32u, n0 - k0);
      q.on = (uint32_t)lane < q.cnt;
      q.addr = q.on ? src_u + (uint64_t)ent[k0 + lane] * a.rec : src_u;
      q.okm = q.cnt == 32 ? 0xffffffffu : ((1u << q.cnt) - 1u);
      q.out = reinterpret_cast<uint32_t*>(seg + (uint64_t)k0 * a.rec);
      q.o4 = (uint32_t)(q.addr >> 2) & 3;
      return q;
    });
  }
  __syncthreads();                                  // the window tiles are free: the ring again
  DPG_STAMP(3);
  // ---- Phase II (run 1), first step: stage run 1 (records [L, n_src)) ----
  if (warp == 0) {
    if (lane == 0 && a.n_src > L)
      jring = l2_stage_slice(a.src + L * a.rec, (a.n_src - L) * a.rec, c, G, region, bar, kPChunk,
                             kPSlots, policy_evict_last(), jring);
    __syncwarp();
  }
  __syncthreads();
  DPG_STAMP(4);
  grid_barrier_mono(a.gbar + 16, G);
  DPG_STAMP(5);

  // ---- Phase II (run 1) probe fused with Phase III, in
  // output order: a run-1 row comes from the L2-resident run 1 (the last run
  // needs no INTERNAL), a run-0 row is the next record of the chunk's
  // INTERNAL segment ----
  {
    const uint32_t nt = ngroups > (uint32_t)warp ? (ngroups - warp + kPWarps - 1) / kPWarps : 0;
    // the rids of a group are loaded two groups before its descriptor is built
    auto rid_load = [&](uint32_t t) -> uint32_t {
      const uint64_t i = lo + 32 * (uint64_t)(warp + t * kPWarps) + lane;
      return (t < nt && i < hi) ? ldg_first(a.rids + i) : 0xFFFFFFFFu;
    };
    uint32_t rq0 = rid_load(0), rq1 = rid_load(1), rq2 = rid_load(2), rq3 = rid_load(3);
    uint32_t next_t = 0;
    pipeline(nt, [&](uint32_t t) -> AgGroup {
      // groups are requested in order t = 0, 1, 2, ...: rotate the rid registers
      (void)next_t;
      const uint32_t r = rq0;
      rq0 = rq1;
      rq1 = rq2;
      rq2 = rq3;
      rq3 = rid_load(t + 4);
      AgGroup q;
      const uint32_t g = warp + t * kPWarps;
      const uint64_t g0 = lo + 32 * (uint64_t)g;
      q.cnt = (uint32_t)min_u64(32, hi - g0);
      const bool in0 = r < L;
      const uint32_t m0 = __ballot_sync(0xffffffffu, in0);
      const uint64_t k = gcnt[g] + __popc(m0 & lanemask_lt());
      q.on = r < a.n_src;
      q.addr = in0 ? seg_u + k * a.rec : (q.on ? src_u + (uint64_t)r * a.rec : src_u);
      q.okm = __ballot_sync(0xffffffffu, q.on);
      q.out = reinterpret_cast<uint32_t*>(a.dst + g0 * a.rec);
      q.o4 = (uint32_t)(q.addr >> 2) & 3;
      return q;
    });
  }
  if (a.ts) {
    __syncthreads();
    DPG_STAMP(6);
  }
#undef DPG_STAMP
}

uint32_t l2pair_smem_bytes(uint64_t chunk) {
  const uint64_t groups = (chunk + 31) / 32;
  return (uint32_t)(128 + kPRegion + 4 * (groups + 1) + 4 * chunk + 64);
}

cudaError_t launch_l2pair(const L2PairArgs& a, uint32_t grid, cudaStream_t st, uint32_t* nl) {
  ++*nl;
  auto fn = k_dpg_l2pair;
  const uint32_t smem = l2pair_smem_bytes(a.chunk);
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
  L2PairArgs arg = a;
  void* params[] = {&arg};
  return cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(kPThreads), params, smem, st);
}

}  // namespace dpg
