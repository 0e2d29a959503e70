// skew.cu -- data skew check by sampling the rid sequence (section 2.3,
// "sample the rids from the rid sequence ... partitions of the
// rids are chosen so as to evenly partition the sampled set").
//
// The shared-memory-run plan gives every run of L source records a fixed
// capacity of entries (expectation + L/4); a rid list that puts many more
// rids into some runs overflows them (the excess is served by direct copies
// after Phase II).  Before such a plan runs on a large input, S rids sampled
// at evenly spaced positions are counted per group of runs; the estimated
// number of rids beyond the runs' capacity decides whether the plan keeps its
// fixed runs or switches to the count-based L2 runs (exact run sizes, no
// capacity: the "other basis" for the partitions the paper asks for).
#include "dpg_internal.cuh"

namespace dpg {

// hist[g] += samples whose run r >> s falls in group g (runs b with b / gsz == g)
__global__ void k_skew_sample(const uint32_t* __restrict__ rids, uint64_t n_out, uint64_t n_src,
                              uint32_t S, uint32_t s, uint32_t gsz, uint32_t* __restrict__ hist) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < S; k += gridDim.x * blockDim.x) {
    const uint64_t i = (uint64_t)k * n_out / S;
    const uint32_t r = __ldg(rids + i);
    if (r < n_src) atomicAdd(&hist[(r >> s) / gsz], 1u);
  }
}

// out[0] = estimated rids beyond capacity: sum over groups of
// gsz * max(0, est_per_run - cap), est_per_run = hist[g] * n_out / (S * runs_in_g);
// the histogram is cleared for the next call.
__global__ void k_skew_reduce(uint32_t* __restrict__ hist, uint32_t ng, uint32_t K, uint32_t gsz,
                              uint64_t n_out, uint32_t S, uint32_t cap,
                              unsigned long long* __restrict__ out) {
  __shared__ unsigned long long acc;
  if (threadIdx.x == 0) acc = 0;
  __syncthreads();
  unsigned long long mine = 0;
  for (uint32_t g = threadIdx.x; g < ng; g += blockDim.x) {
    const uint32_t runs = min(gsz, K - g * gsz);
    const double est = (double)hist[g] * (double)n_out / ((double)S * runs);
    if (est > cap) mine += (unsigned long long)((est - cap) * runs);
    hist[g] = 0;
  }
  atomicAdd(&acc, mine);
  __syncthreads();
  if (threadIdx.x == 0) *out = acc;
}

cudaError_t launch_skew_check(const uint32_t* rids, uint64_t n_out, uint64_t n_src, uint32_t s,
                              uint32_t K, uint32_t cap, uint32_t S, uint32_t* hist,
                              unsigned long long* out, cudaStream_t st, uint32_t* nl) {
  // groups large enough for ~64 expected samples each (a uniform list then
  // stays within its capacity by several standard deviations)
  const uint32_t gsz = (uint32_t)max_u64(1, ((uint64_t)K * 64 + S - 1) / S);
  const uint32_t ng = (K + gsz - 1) / gsz;
  *nl += 2;
  k_skew_sample<<<(S + 255) / 256, 256, 0, st>>>(rids, n_out, n_src, S, s, gsz, hist);
  k_skew_reduce<<<1, 1024, 0, st>>>(hist, ng, K, gsz, n_out, S, cap, out);
  return cudaGetLastError();
}

}  // namespace dpg

namespace dpg {

// Run boundaries from a sorted sample of the rids (section 2.3, P:466-475;
// reading A23), one CTA: S rids drawn at SplitMix64 positions, sorted
// (bitonic, in shared memory, padded to P2 = 2^k >= S with 0xFFFFFFFF), the
// cut candidates c_i = sample[i*S/K] kept when c_i < n_src and c_i > c_(i-1)
// (c_0 = the smallest sampled rid; the candidates ascend, so this is "above
// the last kept cut"), compacted by a block scan.  bounds[0..n] = 0, cuts...,
// n_src; *n_runs = n.
constexpr int kSkewPartThreads = 1024;

__global__ void __launch_bounds__(kSkewPartThreads)
k_skew_partition(const uint32_t* __restrict__ rids, uint64_t n_out, uint32_t n_src, uint32_t K,
                 uint32_t S, uint32_t P2, uint64_t seed, uint32_t* __restrict__ bounds,
                 uint32_t* __restrict__ n_runs) {
  extern __shared__ uint32_t sv[];
  __shared__ uint32_t wsum[33];
  for (uint32_t k = threadIdx.x; k < P2; k += blockDim.x) {
    uint32_t v = 0xFFFFFFFFu;
    if (k < S) {
      uint64_t z = seed + (uint64_t)(k + 1) * 0x9E3779B97F4A7C15ull;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      z ^= z >> 31;
      const uint32_t r = __ldg(rids + __umul64hi(z, n_out));
      v = r < n_src ? r : n_src;
    }
    sv[k] = v;
  }
  __syncthreads();
  for (uint32_t size = 2; size <= P2; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t t = threadIdx.x; t < P2 / 2; t += blockDim.x) {
        const uint32_t i = 2 * t - (t & (stride - 1)), j = i + stride;
        const bool up = (i & size) == 0;
        const uint32_t x = sv[i], y = sv[j];
        if ((x > y) == up) { sv[i] = y; sv[j] = x; }
      }
      __syncthreads();
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t base = 0;
  for (uint32_t i0 = 1; i0 < K; i0 += blockDim.x) {
    const uint32_t i = i0 + threadIdx.x;
    uint32_t keep = 0, q = 0;
    if (i < K) {
      q = sv[(uint64_t)i * S / K];
      keep = q < n_src && q > sv[(uint64_t)(i - 1) * S / K];
    }
    uint32_t x = keep;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      const uint32_t w = wsum[lane];
      uint32_t ws = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, ws, o);
        if (lane >= o) ws += y;
      }
      wsum[lane] = ws - w;
      if (lane == 31) wsum[32] = ws;
    }
    __syncthreads();
    if (keep) bounds[1 + base + wsum[warp] + x - 1] = q;
    base += wsum[32];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    bounds[0] = 0;
    bounds[base + 1] = n_src;
    *n_runs = base + 1;
  }
}

cudaError_t launch_skew_partition(const uint32_t* rids, uint64_t n_out, uint32_t n_src, uint32_t K,
                                  uint32_t S, uint64_t seed, uint32_t* bounds, uint32_t* n_runs,
                                  cudaStream_t st, uint32_t* nl) {
  uint32_t P2 = 2;
  while (P2 < S) P2 <<= 1;
  const size_t smem = (size_t)P2 * 4;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_skew_partition,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  ++*nl;
  k_skew_partition<<<1, kSkewPartThreads, smem, st>>>(rids, n_out, n_src, K, S, P2, seed, bounds,
                                                      n_runs);
  return cudaGetLastError();
}

}  // namespace dpg
