// micro3.cu -- what limits random row access on B200 when the rows are
// L2-resident?  (Design evidence for the gather of the L2-run DPG; not part of
// libdpg.so.)  A footprint of F MB is made L2-resident by a warm-up pass, then
// N random rows (hash of the item index) are read (XOR-reduced) or written.
//   ld4   : row-mapped, 4-byte lanes (rec/4 lanes per row)
//   ld16w : enclosing 16-byte-aligned window of the row, 16-byte lanes
//   tma   : each lane issues a cp.async.bulk of the row's 16-byte window into
//           shared memory (mbarrier per warp)
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a micro3.cu -o micro3
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// MODE 0: ld4 read; 1: ld16w read; 2: st4 write; 3: st16w write (window, only aligned interior of 16-B words)
template <int MODE, int U>
__global__ void __launch_bounds__(512) k_rows(uint8_t* buf, uint32_t nrows, uint32_t rec, uint32_t S,
                                              uint32_t n, uint32_t* sink) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  uint32_t acc = 0;
  if (MODE == 0 || MODE == 2) {
    const uint32_t R = rec / 4, RPI = R <= 32 ? 32 / R : 1, lr = lane / R, lw = lane % R;
    for (uint32_t i0 = gw * RPI * U; i0 < n; i0 += nw * RPI * U) {
      uint32_t v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t it = i0 + u * RPI + lr;
        const uint32_t r = hsh(it) % nrows;
        uint32_t* p = reinterpret_cast<uint32_t*>(buf + (uint64_t)r * S) + lw;
        if (lr < RPI && it < n) {
          if (MODE == 0) v[u] = __ldcg(p); else *p = it;
        } else v[u] = 0;
      }
      if (MODE == 0) {
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u];
      }
    }
  } else {
    // window of 16-B words covering [r*S, r*S+rec): W16 words
    const uint32_t W16 = (rec + 12 + 15) / 16 + 0;   // max words a 4-B-aligned row can span
    const uint32_t RPI = 32 / W16, lr = lane / W16, lw = lane % W16;
    for (uint32_t i0 = gw * RPI * U; i0 < n; i0 += nw * RPI * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t it = i0 + u * RPI + lr;
        const uint32_t r = hsh(it) % nrows;
        const uint64_t a0 = (uint64_t)r * S, a1 = a0 + rec;
        const uint64_t w = (a0 & ~15ull) + 16ull * lw;
        v[u] = make_uint4(0, 0, 0, 0);
        if (lr < RPI && it < n && w < a1) {
          if (MODE == 1) v[u] = __ldcg(reinterpret_cast<const uint4*>(buf + w));
          else if (w >= a0 && w + 16 <= a1) *reinterpret_cast<uint4*>(buf + w) = make_uint4(it, 1, 2, 3);
        }
      }
      if (MODE == 1) {
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
      }
    }
  }
  if (acc == 0x12345678u) *sink = acc;
}

// TMA: each lane bulk-copies one row window (112 B for 100-B rows) to smem.
__global__ void __launch_bounds__(512) k_tma(const uint8_t* buf, uint32_t nrows, uint32_t rec, uint32_t S,
                                             uint32_t n, uint32_t* sink, int per_lane) {
  extern __shared__ __align__(128) uint8_t dyn[];
  uint8_t (*sm)[2][32 * 128] = reinterpret_cast<uint8_t (*)[2][32 * 128]>(dyn + 256);
  uint64_t (*bar)[2] = reinterpret_cast<uint64_t (*)[2]>(dyn);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  if (lane == 0) {
    for (int k = 0; k < 2; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[warp][k])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t acc = 0;
  uint32_t ph[2] = {0, 0};
  uint32_t k = 0;
  for (uint32_t i0 = gw * 32; i0 < n; i0 += nw * 32, k ^= 1) {
    // wait for the copies issued two iterations ago into this buffer
    uint64_t* b = &bar[warp][k];
    const uint32_t it = i0 + lane;
    const uint32_t r = hsh(it) % nrows;
    const uint64_t a0 = (uint64_t)r * S;
    const uint64_t w0 = a0 & ~15ull, w1 = (a0 + rec + 15) & ~15ull;
    const uint32_t bytes = (uint32_t)(w1 - w0);
    const uint32_t tot = __reduce_add_sync(0xffffffffu, it < n ? bytes : 0u);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tot) : "memory");
    __syncwarp();
    if (it < n)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(&sm[warp][k][lane * 128])), "l"(buf + w0), "r"(bytes), "r"(smem_u32(b)) : "memory");
    // wait
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(b)), "r"(ph[k]) : "memory");
    }
    ph[k] ^= 1;
    acc ^= *reinterpret_cast<const uint32_t*>(&sm[warp][k][lane * 128 + 16]);
  }
  if (acc == 0x12345678u) *sink = acc;
}

template <typename F>
float timeit(F f, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  std::vector<float> ts;
  for (int i = 0; i < reps + 1; ++i) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (i) ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

int main(int argc, char** argv) {
  const uint64_t foot_mb = argc > 1 ? atoi(argv[1]) : 26;
  const uint32_t n = argc > 2 ? atoi(argv[2]) : (16u << 20);
  uint8_t* buf; uint32_t* sink;
  CK(cudaMalloc(&buf, (foot_mb << 20) + 4096));
  CK(cudaMemset(buf, 1, (foot_mb << 20) + 4096));
  CK(cudaMalloc(&sink, 4));
  const int G = 148 * 4;
  CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 + 16 * 2 * 32 * 128));
  auto pr = [&](const char* what, uint32_t rec, uint32_t S, float ms) {
    printf("foot %4lluMB %-8s rec %4u S %4u n %9u %8.1f us %6.2f Grow/s %7.0f GB/s\n",
           (unsigned long long)foot_mb, what, rec, S, n, ms * 1e3, n / (ms * 1e-3) / 1e9,
           (double)n * rec / (ms * 1e-3) / 1e9);
  };
  for (auto rs : std::vector<std::pair<uint32_t, uint32_t>>{{100, 100}, {128, 128}, {64, 64}, {96, 128}, {100, 128}, {32, 32}}) {
    const uint32_t rec = rs.first, S = rs.second;
    const uint32_t nrows = (uint32_t)((foot_mb << 20) / S);
    // warm
    k_rows<0, 8><<<G, 512>>>(buf, nrows, rec, S, nrows * 4, sink);
    pr("ld4", rec, S, timeit([&] { k_rows<0, 8><<<G, 512>>>(buf, nrows, rec, S, n, sink); }));
    pr("ld4u16", rec, S, timeit([&] { k_rows<0, 16><<<G, 512>>>(buf, nrows, rec, S, n, sink); }));
    pr("ld16w", rec, S, timeit([&] { k_rows<1, 8><<<G, 512>>>(buf, nrows, rec, S, n, sink); }));
    pr("st4", rec, S, timeit([&] { k_rows<2, 8><<<G, 512>>>(buf, nrows, rec, S, n, sink); }));
    pr("st16w", rec, S, timeit([&] { k_rows<3, 8><<<G, 512>>>(buf, nrows, rec, S, n, sink); }));
    if (rec <= 128)
      pr("tma", rec, S, timeit([&] { k_tma<<<148, 512, 256 + 16 * 2 * 32 * 128>>>(buf, nrows, rec, S, n, sink, 1); }));
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
