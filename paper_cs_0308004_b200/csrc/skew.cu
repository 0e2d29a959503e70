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
