// micro.cu -- standalone microbenchmarks of record-granular random access on
// this GPU (not part of libdpg.so).  Separates the costs DPG trades between:
//   rd_rand : random record reads  (XOR-reduced, no record writes)
//   wr_rand : random record writes (constant data, no record reads)
//   gather  : random reads -> sequential writes (the direct retrieval)
//   scatter : sequential reads -> random writes (the fused DPG write side)
// each with high memory-level parallelism (every lane keeps U words in flight)
// and optional L2 eviction hints.  Build: nvcc -O3 -arch=sm_100a micro.cu -o micro
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint64_t pol_first() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint64_t pol_last() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint32_t ldh(const uint32_t* a, uint64_t p) { uint32_t v; asm volatile("ld.global.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(p)); return v; }
__device__ __forceinline__ void sth(uint32_t* a, uint32_t v, uint64_t p) { asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" :: "l"(a), "r"(v), "l"(p) : "memory"); }

// Records of R 4-byte words; lanes < R of a warp handle one record per step.
template <int U, int MODE, int LH, int SH>
__global__ void __launch_bounds__(256) k(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                                         const uint32_t* __restrict__ perm, uint32_t n, uint32_t R,
                                         uint32_t* sink) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint64_t lp = LH == 1 ? pol_first() : pol_last();
  const uint64_t sp = SH == 1 ? pol_first() : pol_last();
  uint32_t acc = 0;
  for (uint32_t g0 = gw * 32; g0 < n; g0 += nw * 32) {
    const uint32_t my = g0 + lane < n ? perm[g0 + lane] : 0;
    for (uint32_t k0 = 0; k0 < 32; k0 += U) {
      uint32_t v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t r = __shfl_sync(~0u, my, (k0 + u) & 31);
        const uint32_t row = g0 + k0 + u;
        v[u] = 0x5a5a5a5au ^ row;
        if (lane < (int)R && row < n) {
          const uint32_t* a = (MODE == 0 || MODE == 2) ? src + (uint64_t)r * R + lane
                                                       : src + (uint64_t)row * R + lane;
          if (MODE != 1) v[u] = LH ? ldh(a, lp) : __ldg(a);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t r = __shfl_sync(~0u, my, (k0 + u) & 31);
        const uint32_t row = g0 + k0 + u;
        if (lane < (int)R && row < n) {
          if (MODE == 0) { acc ^= v[u]; continue; }
          uint32_t* a = MODE == 2 ? dst + (uint64_t)row * R + lane : dst + (uint64_t)r * R + lane;
          if (SH) sth(a, v[u], sp); else *a = v[u];
        }
      }
    }
  }
  if (acc == 0x12345678u) *sink = acc;
}

template <int U, int MODE, int LH, int SH>
float run(const uint32_t* src, uint32_t* dst, const uint32_t* perm, uint32_t n, uint32_t R,
          uint32_t* sink, uint8_t* flush, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  std::vector<float> ts;
  for (int i = 0; i < reps + 1; ++i) {
    CK(cudaMemset(flush, i, 1u << 30));
    cudaEventRecord(a);
    k<U, MODE, LH, SH><<<148 * 8, 256>>>(src, dst, perm, n, R, sink);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (i) ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

int main(int argc, char** argv) {
  uint32_t total_mb = argc > 1 ? atoi(argv[1]) : 100;
  uint8_t* flush; CK(cudaMalloc(&flush, 1u << 30));
  uint32_t* sink; CK(cudaMalloc(&sink, 4));
  for (uint32_t rec : {100u, 128u}) {
    const uint32_t R = rec / 4;
    const uint32_t n = (uint32_t)(((uint64_t)total_mb << 20) / rec);
    uint32_t *src, *dst, *perm;
    CK(cudaMalloc(&src, (uint64_t)n * rec)); CK(cudaMalloc(&dst, (uint64_t)n * rec));
    CK(cudaMalloc(&perm, (uint64_t)n * 4));
    std::vector<uint32_t> h(n);
    for (uint32_t i = 0; i < n; ++i) h[i] = i;
    std::mt19937 g(1); std::shuffle(h.begin(), h.end(), g);
    CK(cudaMemcpy(perm, h.data(), (uint64_t)n * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(src, 1, (uint64_t)n * rec));
    const double rb = (double)n * rec;
    auto pr = [&](const char* name, float ms, double bytes) {
      printf("rec %3u n %8u %-28s %8.1f us %7.0f GB/s\n", rec, n, name, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
    };
    pr("rd_rand U8", run<8, 0, 0, 0>(src, dst, perm, n, R, sink, flush, 5), rb);
    pr("rd_rand U16", run<16, 0, 0, 0>(src, dst, perm, n, R, sink, flush, 5), rb);
    pr("rd_rand U32", run<32, 0, 0, 0>(src, dst, perm, n, R, sink, flush, 5), rb);
    pr("wr_rand U8", run<8, 1, 0, 0>(src, dst, perm, n, R, sink, flush, 5), rb);
    pr("wr_rand U8 st:last", run<8, 1, 0, 2>(src, dst, perm, n, R, sink, flush, 5), rb);
    pr("gather U8", run<8, 2, 0, 0>(src, dst, perm, n, R, sink, flush, 5), 2 * rb);
    pr("gather U16", run<16, 2, 0, 0>(src, dst, perm, n, R, sink, flush, 5), 2 * rb);
    pr("gather U32", run<32, 2, 0, 0>(src, dst, perm, n, R, sink, flush, 5), 2 * rb);
    pr("gather U16 st:first", run<16, 2, 0, 1>(src, dst, perm, n, R, sink, flush, 5), 2 * rb);
    pr("scatter U8", run<8, 3, 0, 0>(src, dst, perm, n, R, sink, flush, 5), 2 * rb);
    pr("scatter U16", run<16, 3, 0, 0>(src, dst, perm, n, R, sink, flush, 5), 2 * rb);
    pr("scatter U16 ld:first st:last", run<16, 3, 1, 2>(src, dst, perm, n, R, sink, flush, 5), 2 * rb);
    cudaFree(src); cudaFree(dst); cudaFree(perm);
  }
  return 0;
}
