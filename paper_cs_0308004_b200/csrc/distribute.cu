// distribute.cu -- DPG Phase I, "Distribute" (Fig. 1).
//
// "One distributes the rids of RID_LIST into appropriate RID runs according
// to the values of the rids"; the run of rid r is given by its
// high-order bits: run(r) = r >> s, L = 2^s (reading A1) -- or,
// under data skew, by boundaries from a sorted sample of the rids merged with
// the multiples of L (section 2.3; bounds_run, reading A23).
//
// B200 form: a counting distribution over K runs and G contiguous chunks of
// the rid list (one CTA per chunk), in three steps:
//   (1) k_count   : per-chunk run histogram (count step of the paper's count
//                   bucket sort), stored run-major counts[b*G + c];
//   (2) k_scan_*  : exclusive scan of counts in run-major order, giving each
//                   (run, chunk) its first slot and run_start[b] ("set bucket
//                   boundaries according to the statistics");
//   (3) k_scatter : each rid writes the pair (r - b*L, i) -- the paper's
//                   "Append r to RID_RUN[run_num]" plus the position i
//                   that Phase III needs -- into its run.
// Within one (run, chunk) cell the order of pairs follows shared-memory atomic
// order; the set of pairs of each run is unique, and the retrieved output is
// unique regardless (each pair names its own destination).
#include "dpg_internal.cuh"

namespace dpg {

static constexpr int kDistThreads = 512;

template <typename RidT>
__device__ __forceinline__ uint64_t load_rid(const void* rids, uint64_t i) {
  return (uint64_t)__ldg(reinterpret_cast<const RidT*>(rids) + i);
}

// (1) per-chunk histogram ------------------------------------------------------
template <typename RidT>
__global__ void __launch_bounds__(kDistThreads) k_count(DistArgs a) {
  extern __shared__ uint32_t hist[];
  const uint32_t c = blockIdx.x;
  const uint64_t lo = (uint64_t)c * a.chunk;
  const uint64_t hi = min_u64(a.n_out, lo + a.chunk);
  if (a.hist_smem) {
    for (uint32_t b = threadIdx.x; b < a.K; b += blockDim.x) hist[b] = 0;
    __syncthreads();
  }
  constexpr int U = 4;
  for (uint64_t base = lo + threadIdx.x; base < hi; base += (uint64_t)U * blockDim.x) {
    uint64_t r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t i = base + (uint64_t)u * blockDim.x;
      r[u] = i < hi ? load_rid<RidT>(a.rids, i) : ~0ull;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t i = base + (uint64_t)u * blockDim.x;
      if (i >= hi) continue;
      if (r[u] >= a.n_src) { report_bad(a.status, i); continue; }
      uint32_t b0;
      uint32_t b = a.bmap ? bounds_run(a.bmap, a.btab, a.s, r[u], &b0) : (uint32_t)(r[u] >> a.s);
      if (a.hist_smem) atomicAdd(&hist[b], 1u);
      else atomicAdd(&a.counts[(uint64_t)b * a.G + c], 1u);
    }
  }
  if (a.hist_smem) {
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < a.K; b += blockDim.x)
      a.counts[(uint64_t)b * a.G + c] = hist[b];
  }
}

// (2) exclusive scan of counts[0, M), M = K*G, run-major ------------------------
static constexpr int kScanThreads = 1024;
static constexpr int kScanItems = 4;
static constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* warp_sums,
                                                         uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    uint32_t w = lane < nw ? warp_sums[lane] : 0;
    uint32_t ws = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, ws, o);
      if (lane >= o) ws += y;
    }
    if (lane < nw) warp_sums[lane] = ws - w;
    if (lane == nw - 1) warp_sums[32] = ws;
  }
  __syncthreads();
  uint32_t r = warp_sums[warp] + x - v;
  *total = warp_sums[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint32_t* in, uint64_t M,
                                                              uint32_t* partial) {
  __shared__ uint32_t ws[33];
  uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    uint64_t i = base + (uint64_t)k * kScanThreads + threadIdx.x;
    if (i < M) s += in[i];
  }
  uint32_t tot;
  block_exclusive_scan(s, ws, &tot);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_partials(uint32_t* partial, uint32_t n) {
  __shared__ uint32_t ws[33];
  uint32_t carry = 0;
  for (uint32_t base = 0; base < n; base += kScanThreads) {
    uint32_t i = base + threadIdx.x;
    uint32_t v = i < n ? partial[i] : 0;
    uint32_t tot;
    uint32_t e = block_exclusive_scan(v, ws, &tot);
    if (i < n) partial[i] = carry + e;
    carry += tot;
  }
}

// In-place exclusive scan of the tile, plus run_start[b] = offs[b*G],
// run_start[K] = total.
__global__ void __launch_bounds__(kScanThreads) k_scan_down(uint32_t* io, uint64_t M,
                                                            const uint32_t* partial, uint32_t G,
                                                            uint32_t K, uint32_t* run_start) {
  __shared__ uint32_t ws[33];
  uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    uint64_t i = base + k;
    v[k] = i < M ? io[i] : 0;
    s += v[k];
  }
  uint32_t tot;
  uint32_t e = block_exclusive_scan(s, ws, &tot) + partial[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    uint64_t i = base + k;
    if (i < M) {
      io[i] = e;
      if (i % G == 0) run_start[i / G] = e;
      if (i == M - 1) run_start[K] = e + v[k];
    }
    e += v[k];
  }
}

// (3) scatter pairs ---------------------------------------------------------------
__device__ __forceinline__ void copy_bytes(uint8_t* d, const uint8_t* s, uint32_t n) {
  if ((((uintptr_t)d | (uintptr_t)s | n) & 15) == 0) {
    for (uint32_t k = 0; k < n; k += 16)
      *reinterpret_cast<uint4*>(d + k) = __ldg(reinterpret_cast<const uint4*>(s + k));
  } else if ((((uintptr_t)d | (uintptr_t)s | n) & 3) == 0) {
    for (uint32_t k = 0; k < n; k += 4)
      *reinterpret_cast<uint32_t*>(d + k) = __ldg(reinterpret_cast<const uint32_t*>(s + k));
  } else {
    for (uint32_t k = 0; k < n; ++k) d[k] = s[k];
  }
}

template <typename RidT, typename PairT>
__global__ void __launch_bounds__(kDistThreads) k_scatter(DistArgs a) {
  extern __shared__ uint32_t cur[];
  const uint32_t c = blockIdx.x;
  const uint64_t lo = (uint64_t)c * a.chunk;
  const uint64_t hi = min_u64(a.n_out, lo + a.chunk);
  if (a.hist_smem) {
    for (uint32_t b = threadIdx.x; b < a.K; b += blockDim.x)
      cur[b] = a.counts[(uint64_t)b * a.G + c];
    __syncthreads();
  }
  const uint64_t lmask = (1ull << a.s) - 1;
  PairT* pairs = reinterpret_cast<PairT*>(a.pairs);
  constexpr int U = 4;
  for (uint64_t base = lo + threadIdx.x; base < hi; base += (uint64_t)U * blockDim.x) {
    uint64_t r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t i = base + (uint64_t)u * blockDim.x;
      r[u] = i < hi ? load_rid<RidT>(a.rids, i) : ~0ull;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t i = base + (uint64_t)u * blockDim.x;
      if (i >= hi || r[u] >= a.n_src) continue;
      uint32_t b0 = 0;
      uint32_t b = a.bmap ? bounds_run(a.bmap, a.btab, a.s, r[u], &b0) : (uint32_t)(r[u] >> a.s);
      uint32_t slot = a.hist_smem ? atomicAdd(&cur[b], 1u)
                                  : atomicAdd(&a.counts[(uint64_t)b * a.G + c], 1u);
      uint64_t local = a.bmap ? r[u] - b0 : r[u] & lmask;
      if (sizeof(PairT) == 4)
        pairs[slot] = (PairT)((i << a.s) | local);
      else
        pairs[slot] = (PairT)(local | (i << 32));
      if (a.pay_bytes)
        copy_bytes(a.pay_dst + (uint64_t)slot * a.pay_bytes, a.pay_src + i * a.pay_bytes,
                   a.pay_bytes);
    }
  }
}

// Test helper: pairs -> uint64 (local | pos << 32), run_start -> uint64.
template <typename PairT>
__global__ void k_unpack(const PairT* pairs, uint64_t n, uint32_t s, const uint32_t* rs,
                         uint32_t K, uint64_t* out, uint64_t* rs_out) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = t; j < n; j += stride) {
    uint64_t p = pairs[j];
    if (sizeof(PairT) == 4)
      out[j] = (p & ((1ull << s) - 1)) | ((p >> s) << 32);
    else
      out[j] = p;
  }
  for (uint64_t b = t; b <= K; b += stride) rs_out[b] = rs[b];
}

// Steps (1) and (2): counts[b*G + c] become the first slot of (run b, chunk c)
// in run-major order; run_start[K+1] the runs' boundaries.
template <typename RidT>
static cudaError_t launch_count_scan_t(const DistArgs& a, cudaStream_t st, uint32_t* nl) {
  size_t hsm = a.hist_smem ? (size_t)a.K * sizeof(uint32_t) : 0;
  if (hsm > 48 * 1024)
    cudaFuncSetAttribute(k_count<RidT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
  k_count<RidT><<<a.G, kDistThreads, hsm, st>>>(a);
  ++*nl;
  const uint64_t M = (uint64_t)a.K * a.G;
  const uint32_t nt = (uint32_t)((M + kScanTile - 1) / kScanTile);
  // partial sums live just past run_start (allocated by the caller: K+1+nt).
  uint32_t* partial = a.run_start + a.K + 1;
  k_scan_reduce<<<nt, kScanThreads, 0, st>>>(a.counts, M, partial);
  k_scan_partials<<<1, kScanThreads, 0, st>>>(partial, nt);
  k_scan_down<<<nt, kScanThreads, 0, st>>>(a.counts, M, partial, a.G, a.K, a.run_start);
  *nl += 3;
  return cudaGetLastError();
}

cudaError_t launch_count_scan(const DistArgs& a, cudaStream_t st, uint32_t* nl) {
  return launch_count_scan_t<uint32_t>(a, st, nl);
}

uint32_t count_scan_partials(uint64_t K, uint64_t G) {
  return (uint32_t)((K * G + kScanTile - 1) / kScanTile);
}

// Work items of the probe-gather kernel: ic[b] = chunks of SP pairs in run b,
// item_start = their exclusive scan, items[item_start[b] + j] = {b, j | more << 31, p0, p1}
// (more: a later chunk of the run follows).
__global__ void k_item_counts(const uint32_t* __restrict__ rs, uint32_t K, uint32_t sp,
                              uint32_t* __restrict__ ic) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < K; b += gridDim.x * blockDim.x)
    ic[b] = (rs[b + 1] - rs[b] + sp - 1) / sp;
}

__global__ void k_item_expand(const uint32_t* __restrict__ is, const uint32_t* __restrict__ rs,
                              uint32_t K, uint32_t sp, uint4* __restrict__ items) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < K;
       b += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t i0 = is[b], r0 = rs[b], r1 = rs[b + 1];
    for (uint32_t j = lane; i0 + j < is[b + 1]; j += 32) {
      const uint32_t p0 = r0 + j * sp;
      const uint32_t more = p0 + sp < r1 ? 0x80000000u : 0u;   // a later chunk restages the region
      items[i0 + j] = make_uint4(b, j | more, p0, min(r1, p0 + sp));
    }
  }
}

cudaError_t launch_items(const uint32_t* run_start, uint32_t K, uint32_t sp, uint32_t* item_cnt,
                         uint32_t* partial, uint32_t* item_start, uint32_t* item_run,
                         cudaStream_t st, uint32_t* nl) {
  const uint32_t g = (uint32_t)min_u64(1024, (K + 255) / 256);
  k_item_counts<<<g, 256, 0, st>>>(run_start, K, sp, item_cnt);
  const uint32_t nt = count_scan_partials(K, 1);
  k_scan_reduce<<<nt, kScanThreads, 0, st>>>(item_cnt, K, partial);
  k_scan_partials<<<1, kScanThreads, 0, st>>>(partial, nt);
  k_scan_down<<<nt, kScanThreads, 0, st>>>(item_cnt, K, partial, 1, K, item_start);
  k_item_expand<<<(uint32_t)min_u64(4096, (K + 7) / 8), 256, 0, st>>>(
      item_start, run_start, K, sp, reinterpret_cast<uint4*>(item_run));
  *nl += 5;
  return cudaGetLastError();
}

template <typename RidT>
static cudaError_t launch_distribute_t(const DistArgs& a, cudaStream_t st, uint32_t* nl) {
  size_t hsm = a.hist_smem ? (size_t)a.K * sizeof(uint32_t) : 0;
  if (hsm > 48 * 1024) {
    cudaFuncSetAttribute(k_scatter<RidT, uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)hsm);
    cudaFuncSetAttribute(k_scatter<RidT, uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)hsm);
  }
  cudaError_t e = launch_count_scan_t<RidT>(a, st, nl);
  if (e != cudaSuccess) return e;
  if (a.pair_bytes == 4)
    k_scatter<RidT, uint32_t><<<a.G, kDistThreads, hsm, st>>>(a);
  else
    k_scatter<RidT, uint64_t><<<a.G, kDistThreads, hsm, st>>>(a);
  ++*nl;
  return cudaGetLastError();
}

cudaError_t launch_distribute(const DistArgs& a, bool rid64, cudaStream_t st, uint32_t* nl) {
  return rid64 ? launch_distribute_t<uint64_t>(a, st, nl) : launch_distribute_t<uint32_t>(a, st, nl);
}

cudaError_t launch_unpack_pairs(const DistArgs& a, uint64_t* pairs_out, uint64_t* rs_out,
                                cudaStream_t st, uint32_t* nl) {
  uint64_t n = a.run_start ? a.n_out : 0;
  uint32_t grid = (uint32_t)min_u64(4096, (max_u64(n, a.K + 1) + 255) / 256);
  if (a.pair_bytes == 4)
    k_unpack<uint32_t><<<grid, 256, 0, st>>>((const uint32_t*)a.pairs, a.n_out, a.s, a.run_start,
                                             a.K, pairs_out, rs_out);
  else
    k_unpack<uint64_t><<<grid, 256, 0, st>>>((const uint64_t*)a.pairs, a.n_out, a.s, a.run_start,
                                             a.K, pairs_out, rs_out);
  ++*nl;
  return cudaGetLastError();
}

// Owner partition (multi-GPU): 8-byte entries (local | pos << 32) grouped by
// owner -> separate request (local) and position arrays + per-owner counts.
__global__ void k_split_entries(const uint64_t* pairs, const uint32_t* rs, uint32_t K,
                                uint32_t* local_out, uint32_t* pos_out, uint64_t* counts) {
  const uint64_t n = rs[K];
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = t; j < n; j += stride) {
    const uint64_t p = pairs[j];
    local_out[j] = (uint32_t)p;
    pos_out[j] = (uint32_t)(p >> 32);
  }
  for (uint64_t b = t; b < K; b += stride) counts[b] = rs[b + 1] - rs[b];
}

cudaError_t launch_split_entries(const DistArgs& a, uint32_t* local_out, uint32_t* pos_out,
                                 uint64_t* counts, cudaStream_t st, uint32_t* nl) {
  const uint32_t grid = (uint32_t)min_u64(4096, max_u64(1, (a.n_out + 255) / 256));
  k_split_entries<<<grid, 256, 0, st>>>((const uint64_t*)a.pairs, a.run_start, a.K, local_out,
                                        pos_out, counts);
  ++*nl;
  return cudaGetLastError();
}

}  // namespace dpg
