// micro_dist.cu -- cost of the per-rid step of DPG Phase I on this GPU: find
// the run (r >> s) of every rid of a CTA's chunk and count per run, by
//   ballot : per-warp counters, equal keys grouped with one ballot per key bit
//   match  : per-warp counters, equal keys grouped with __match_any_sync
//   atoms  : shared-memory atomicAdd on per-CTA counters
//   atoms_w: shared-memory atomicAdd on per-warp counters (no cross-warp conflicts)
// rids staged in shared memory first (as the fused kernel does).  Not part of
// libdpg.so.   nvcc -O3 -arch=sm_100a micro_dist.cu -o micro_dist
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(const uint32_t* rids, uint32_t n, uint32_t s, uint32_t K,
                                         uint32_t* out) {
  extern __shared__ uint32_t sm[];
  uint32_t* rc = sm;                      // rid chunk
  uint16_t* hw = reinterpret_cast<uint16_t*>(sm + 8192);   // 16 x K u16 (K <= 4096)
  uint32_t* hc = sm + 8192 + 16 * 4096 / 2;                 // K u32
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const uint32_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk), span = hi > lo ? hi - lo : 0;
  for (uint32_t i = tid; i < span; i += 512) rc[i] = rids[lo + i];
  for (uint32_t i = tid; i < 16 * K; i += 512) hw[i] = 0;
  for (uint32_t i = tid; i < K; i += 512) hc[i] = 0;
  __syncthreads();
  long long t0 = clock64();
  const uint32_t sub = ((span + 15) / 16 + 31) & ~31u;
  const uint32_t wlo = min(span, warp * sub), whi = min(span, wlo + sub);
  uint16_t* myh = hw + warp * K;
  const uint32_t kbits = 32 - __clz(K);
  const uint32_t lt = (1u << lane) - 1u;
  if (MODE == 2) {
    for (uint32_t i = tid; i < span; i += 512) atomicAdd(&hc[rc[i] >> s], 1u);
  } else if (MODE == 3) {
    for (uint32_t i0 = wlo; i0 < whi; i0 += 32) {
      const uint32_t i = i0 + lane;
      if (i < whi) atomicAdd(reinterpret_cast<uint32_t*>(myh) + ((rc[i] >> s) >> 1), 1u << (16 * ((rc[i] >> s) & 1)));
    }
  } else {
    constexpr int U = 4;
    for (uint32_t i0 = wlo; i0 < whi; i0 += 32 * U) {
      uint32_t key[U], peers[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = i0 + u * 32 + lane;
        key[u] = i < whi ? rc[i] >> s : K;
      }
      if (MODE == 0) {
#pragma unroll
        for (int u = 0; u < U; ++u) peers[u] = 0xFFFFFFFFu;
        for (uint32_t j = 0; j < kbits; ++j) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t bit = (key[u] >> j) & 1u;
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, bit);
            peers[u] &= bit ? bal : ~bal;
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) peers[u] = __match_any_sync(0xFFFFFFFFu, key[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (key[u] < K && (peers[u] & lt) == 0) myh[key[u]] = (uint16_t)(myh[key[u]] + __popc(peers[u]));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = (uint32_t)(t1 - t0);
  if (tid < 16) out[gridDim.x + blockIdx.x] = hw[tid] + hc[tid];
}

int main() {
  const uint32_t n = 1 << 20, K = 2048, s = 9;
  std::vector<uint32_t> h(n);
  for (uint32_t i = 0; i < n; ++i) h[i] = i;
  std::mt19937 g(1); std::shuffle(h.begin(), h.end(), g);
  uint32_t *rids, *out;
  cudaMalloc(&rids, n * 4); cudaMalloc(&out, 4096 * 4);
  cudaMemcpy(rids, h.data(), n * 4, cudaMemcpyHostToDevice);
  const int smem = 8192 * 4 + 16 * 4096 * 2 + 4096 * 4;
  const char* names[] = {"ballot", "match", "atoms", "atoms_w"};
  for (int m = 0; m < 4; ++m) {
    auto fn = m == 0 ? k<0> : m == 1 ? k<1> : m == 2 ? k<2> : k<3>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      fn<<<148, 512, smem>>>(rids, n, s, K, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      std::vector<uint32_t> o(148);
      cudaMemcpy(o.data(), out, 148 * 4, cudaMemcpyDeviceToHost);
      std::sort(o.begin(), o.end());
      printf("%-8s kernel %7.1f us   count loop median %6u cycles (%.2f cyc/rid/SM)  %s\n", names[m],
             ms * 1e3, o[74], o[74] / (double)(n / 148), cudaGetErrorString(cudaGetLastError()));
    }
  }
}
