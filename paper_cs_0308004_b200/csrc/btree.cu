// btree.cu -- batch lookup of keys in an enhanced B+-tree with DPG (section
// 4, "Batch Lookup in B+ Tree Indexes").
//
// The index (built by the caller; datagen.btree_index builds the test
// inputs): level 0 = the N keys sorted, with rids[j] the rid of level-0 entry
// j; level t = every 16th entry of level t-1 (the first key of each 16-entry
// node below, "all slots of a B+ tree node are used"), up to a top
// level of at most 16 entries.  Every level is padded to a multiple of 16
// entries.  A lookup descends: in each node, the largest entry <= key.
//
//   direct   k_bt_direct: the whole descent per key -- "log_m N nodes of the
//            B+ tree must be accessed.  Each such access will be a random
//            access in main memory".
//   DPG      the two-pass lookup:
//     Phase I   "a lookup of each key, but only using the top half of the
//               B+ tree" -- k_bt_top descends to the level whose entries
//               root the lower subtrees; the key goes to the run of its
//               subtree group (k_l2k_distribute, payload mode: the run-major
//               keys and every query's slot);
//     Phase II  k_bt_probe, one cooperative kernel over the runs: the lower
//               levels of run b's subtrees (contiguous ranges of every level)
//               are staged into the L2 ("one loads a subtree from the lower
//               half"), a grid barrier, then every key of the run
//               completes its lookup (all node reads L2 hits); the rids go to a
//               temporary partition in run order;
//     Phase III k_gather_u32: the rids back in query order.
#include "dpg_internal.cuh"

namespace dpg {

static constexpr int kBtThreads = 512;
static constexpr uint32_t kBtNotFound = 0xFFFFFFFFu;

// Entries of node [first, first + 16) of a level of n entries that are <= q
// (a level is padded to 16 entries, so the node is one 64-byte line).
__device__ __forceinline__ uint32_t bt_count(const uint32_t* lvl, uint32_t n, uint32_t first, uint32_t q) {
  const uint4* p = reinterpret_cast<const uint4*>(lvl + first);
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint4 v = __ldg(p + k);
    const uint32_t i = first + 4 * k;
    c += (i + 0 < n && v.x <= q) + (i + 1 < n && v.y <= q) + (i + 2 < n && v.z <= q) +
         (i + 3 < n && v.w <= q);
  }
  return c;
}

// Descend from the top to level `stop`: the index of the entry of level
// `stop` whose subtree holds q, or kBtNotFound when q is below every key.
__device__ __forceinline__ uint32_t bt_descend(const BTreeIdx& T, uint32_t q, uint32_t stop) {
  const uint32_t top = T.levels - 1;
  const uint32_t c = bt_count(T.lv[top], T.n[top], 0, q);
  if (!c) return kBtNotFound;
  uint32_t j = c - 1;
  for (int t = (int)top - 1; t >= (int)stop; --t) j = 16 * j + bt_count(T.lv[t], T.n[t], 16 * j, q) - 1;
  return j;
}

__device__ __forceinline__ uint32_t bt_lookup(const BTreeIdx& T, uint32_t q) {
  const uint32_t j = bt_descend(T, q, 0);
  if (j == kBtNotFound) return kBtNotFound;
  return __ldg(T.lv[0] + j) == q ? __ldg(T.rids + j) : kBtNotFound;
}

__global__ void __launch_bounds__(256) k_bt_direct(const __grid_constant__ BTreeIdx T,
                                                    const uint32_t* __restrict__ keys, uint64_t n,
                                                    uint32_t* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    __stcs(out + i, bt_lookup(T, __ldcs(keys + i)));
}

// Phase I, first half: the run of each key = (its level-`stop` entry) >> shift
// (K = the runs; a key below every key of the index goes to run 0, where its
// lookup finds nothing).
__global__ void __launch_bounds__(256) k_bt_top(const __grid_constant__ BTreeIdx T, uint32_t stop,
                                                 uint32_t shift, const uint32_t* __restrict__ keys,
                                                 uint64_t n, uint32_t* __restrict__ run) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t j = bt_descend(T, __ldcs(keys + i), stop);
    __stcs(run + i, j == kBtNotFound ? 0u : j >> shift);
  }
}

struct BtProbeArgs {
  uint32_t K;              // runs
  uint32_t s;              // log2 level-0 entries per run
  uint32_t stop;           // the level whose entries root the subtrees (16^stop | 2^s)
  const uint32_t* qkeys;   // keys, run-major
  const uint32_t* run_start;   // [K + 1]
  uint32_t* tmp;           // rids, run-major
  uint32_t* gbar;
};

__global__ void __launch_bounds__(kBtThreads, 1) k_bt_probe(const __grid_constant__ BTreeIdx T,
                                                             const __grid_constant__ BtProbeArgs a) {
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
  uint32_t jring = 0;
  for (uint32_t b = 0; b < a.K; ++b) {
    if (warp == 0) {
      if (lane == 0) {
        // the run's range of every level below `stop`, and of the rids
        for (uint32_t t = 0; t < a.stop && t < T.levels; ++t) {
          const uint64_t r0 = min_u64(T.n[t], ((uint64_t)b << a.s) >> (4 * t));
          const uint64_t r1 = min_u64(T.n[t], ((uint64_t)(b + 1) << a.s) >> (4 * t));
          if (r1 > r0)
            jring = l2_stage_slice(reinterpret_cast<const uint8_t*>(T.lv[t] + r0), (r1 - r0) * 4, c, G,
                                   ring, bar, CH, NS, pol, jring);
          if (t == 0 && r1 > r0)
            jring = l2_stage_slice(reinterpret_cast<const uint8_t*>(T.rids + r0), (r1 - r0) * 4, c, G,
                                   ring, bar, CH, NS, pol, jring);
        }
      }
      __syncwarp();
    }
    grid_barrier(a.gbar, G);
    const uint64_t e0 = __ldg(a.run_start + b), e1 = __ldg(a.run_start + b + 1);
    const uint64_t per = ((e1 - e0 + G - 1) / G + 31) & ~uint64_t(31);
    const uint64_t lo = min_u64(e1, e0 + (uint64_t)c * per), hi = min_u64(e1, lo + per);
    for (uint64_t e = lo + tid; e < hi; e += kBtThreads)
      __stcg(a.tmp + e, bt_lookup(T, __ldcs(a.qkeys + e)));
  }
}

cudaError_t launch_bt_direct(const BTreeIdx& T, const uint32_t* keys, uint64_t n, uint32_t* out,
                             int sm, cudaStream_t st, uint32_t* nl) {
  ++*nl;
  const uint32_t g = (uint32_t)max_u64(1, min_u64((n + 255) / 256, (uint64_t)sm * 8));
  k_bt_direct<<<g, 256, 0, st>>>(T, keys, n, out);
  return cudaGetLastError();
}

cudaError_t launch_bt_top(const BTreeIdx& T, uint32_t stop, uint32_t shift, const uint32_t* keys,
                          uint64_t n, uint32_t* run, int sm, cudaStream_t st, uint32_t* nl) {
  ++*nl;
  const uint32_t g = (uint32_t)max_u64(1, min_u64((n + 255) / 256, (uint64_t)sm * 8));
  k_bt_top<<<g, 256, 0, st>>>(T, stop, shift, keys, n, run);
  return cudaGetLastError();
}

cudaError_t launch_bt_probe(const BTreeIdx& T, uint32_t K, uint32_t s, uint32_t stop,
                            const uint32_t* qkeys, const uint32_t* run_start, uint32_t* tmp,
                            uint32_t* gbar, int sm, cudaStream_t st, uint32_t* nl) {
  ++*nl;
  BtProbeArgs a;
  a.K = K;
  a.s = s;
  a.stop = stop;
  a.qkeys = qkeys;
  a.run_start = run_start;
  a.tmp = tmp;
  a.gbar = gbar;
  BTreeIdx t = T;
  const int smem = 128 + 4 * (32 << 10);
  cudaError_t e = cudaFuncSetAttribute(k_bt_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  void* params[] = {&t, &a};
  return cudaLaunchCooperativeKernel((const void*)k_bt_probe, dim3(sm), dim3(kBtThreads), params, smem,
                                     st);
}

}  // namespace dpg
