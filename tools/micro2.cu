// micro2.cu -- what does a random record access cost on B200, by granularity,
// alignment, L2 residency and temporal locality?  (Design evidence for the
// DPG write side; not part of libdpg.so.)
//
// Item i touches bytes [perm[i]*S + off, perm[i]*S + off + C) of a buffer
// (read: XOR-reduced; write: constant data).  C, S, off multiples of 4; lanes
// move 4 bytes (or 16 when C, S, off are multiples of 16).
//   full aligned chunks      : S = C, off = 0
//   100-byte rows            : S = C = 100
//   100 B in 128-B slots     : S = 128, C = 100
//   interior sectors only    : 'int' mode: [roundup32(p*100), rounddown32(p*100+100))
// perm: uniform permutation, or "blocked" (blocks of B consecutive rows, block
// order random, order inside a block random) to model temporal locality.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a micro2.cu -o micro2
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <numeric>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int WB, bool WRITE, bool INTERIOR>
__global__ void __launch_bounds__(256) k(uint8_t* buf, const uint32_t* __restrict__ perm, uint32_t n,
                                         uint32_t C, uint32_t S, uint32_t off, uint32_t* sink) {
  using T = typename std::conditional<WB == 16, uint4, uint32_t>::type;
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t R = INTERIOR ? 3 * 32 / WB : C / WB;   // words per item (interior: <= 96 B)
  const uint32_t RPI = R <= 32 ? 32 / R : 1;
  const uint32_t lr = lane / R, lw = lane % R;
  uint32_t acc = 0;
  constexpr int U = 8;
  for (uint32_t g0 = gw * 32; g0 < n; g0 += nw * 32) {
    const uint32_t my = g0 + lane < n ? perm[g0 + lane] : 0;
    for (uint32_t k0 = 0; k0 < 32; k0 += U * RPI) {
      T v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t rr = k0 + u * RPI + lr;
        const uint32_t p = __shfl_sync(~0u, my, rr & 31);
        uint64_t a0 = (uint64_t)p * S + off, a1 = a0 + C;
        if (INTERIOR) { a0 = (a0 + 31) & ~31ull; a1 &= ~31ull; }
        const uint64_t a = a0 + (uint64_t)lw * WB;
        const bool on = lr < RPI && rr < 32 && g0 + rr < n && a < a1;
        if constexpr (WB == 16) v[u] = make_uint4(p, lane, 1, 2); else v[u] = p ^ lane;
        if (on) {
          if (WRITE) *reinterpret_cast<T*>(buf + a) = v[u];
          else v[u] = __ldcg(reinterpret_cast<const T*>(buf + a));
        }
      }
      if (!WRITE) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if constexpr (WB == 16) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w; else acc ^= v[u];
        }
      }
    }
  }
  if (acc == 0x12345678u) *sink = acc;
}

__global__ void k_flush(uint4* f, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    f[i] = make_uint4(i, 1, 2, 3);
}

struct Ctx { uint8_t* flush; size_t flush_bytes; uint32_t* sink; };

template <int WB, bool WRITE, bool INTERIOR>
float run(Ctx& c, uint8_t* buf, const uint32_t* perm, uint32_t n, uint32_t C, uint32_t S, uint32_t off,
          bool warm, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  std::vector<float> ts;
  for (int i = 0; i < reps + 1; ++i) {
    if (!warm) k_flush<<<148 * 4, 512>>>((uint4*)c.flush, c.flush_bytes / 16);
    else k<WB, WRITE, INTERIOR><<<148 * 8, 256>>>(buf, perm, n, C, S, off, c.sink);
    cudaEventRecord(a);
    k<WB, WRITE, INTERIOR><<<148 * 8, 256>>>(buf, perm, n, C, S, off, c.sink);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (i) ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

static std::vector<uint32_t> make_perm(uint32_t n, uint32_t B, uint32_t seed) {
  std::mt19937 g(seed);
  std::vector<uint32_t> h(n);
  if (B <= 1) {
    std::iota(h.begin(), h.end(), 0u);
    std::shuffle(h.begin(), h.end(), g);
    return h;
  }
  const uint32_t nb = (n + B - 1) / B;
  std::vector<uint32_t> bo(nb);
  std::iota(bo.begin(), bo.end(), 0u);
  std::shuffle(bo.begin(), bo.end(), g);
  uint32_t k = 0;
  for (uint32_t q = 0; q < nb; ++q) {
    const uint32_t b0 = bo[q] * B, b1 = std::min(n, b0 + B);
    const uint32_t k0 = k;
    for (uint32_t j = b0; j < b1; ++j) h[k++] = j;
    std::shuffle(h.begin() + k0, h.begin() + k, g);
  }
  return h;
}

int main(int argc, char** argv) {
  const uint64_t foot_mb = argc > 1 ? atoi(argv[1]) : 1600;
  Ctx c;
  c.flush_bytes = 512ull << 20;
  CK(cudaMalloc(&c.flush, c.flush_bytes));
  CK(cudaMalloc(&c.sink, 4));
  const uint64_t foot = foot_mb << 20;
  uint8_t* buf;
  CK(cudaMalloc(&buf, foot + 4096));
  CK(cudaMemset(buf, 1, foot + 4096));
  uint32_t* perm;
  const uint32_t nmax = (uint32_t)(foot / 32);
  CK(cudaMalloc(&perm, (uint64_t)nmax * 4));
  auto pr = [&](const char* what, uint32_t C, uint32_t S, uint32_t B, bool warm, uint32_t n, float ms,
                double bytes) {
    printf("foot %5lluMB %-10s C %4u S %4u blk %5u %s n %9u %9.1f us %7.0f GB/s %6.2f Gitem/s\n",
           (unsigned long long)foot_mb, what, C, S, B, warm ? "warm" : "cold", n, ms * 1e3,
           bytes / (ms * 1e-3) / 1e9, n / (ms * 1e-3) / 1e9);
  };
  auto load = [&](uint32_t n, uint32_t B) {
    auto h = make_perm(n, B, 7);
    CK(cudaMemcpy(perm, h.data(), (uint64_t)n * 4, cudaMemcpyHostToDevice));
  };
  // 1. full aligned chunks: read and write rate vs granularity
  for (uint32_t C : {32u, 64u, 128u, 256u, 512u}) {
    const uint32_t n = (uint32_t)(foot / C);
    load(n, 1);
    pr("rd_full", C, C, 1, false, n, run<16, false, false>(c, buf, perm, n, C, C, 0, false), (double)n * C);
    pr("wr_full", C, C, 1, false, n, run<16, true, false>(c, buf, perm, n, C, C, 0, false), (double)n * C);
    if (foot_mb <= 128)
      pr("wr_full", C, C, 1, true, n, run<16, true, false>(c, buf, perm, n, C, C, 0, true), (double)n * C);
  }
  // 2. 100-byte rows: whole rows, rows in 128-B slots, interior sectors only; blocked locality
  for (uint32_t B : {1u, 8u, 64u, 1024u}) {
    const uint32_t n = (uint32_t)(foot / 128);
    load(n, B);
    pr("rd_row", 100, 100, B, false, n, run<4, false, false>(c, buf, perm, n, 100, 100, 0, false), n * 100.0);
    pr("wr_row", 100, 100, B, false, n, run<4, true, false>(c, buf, perm, n, 100, 100, 0, false), n * 100.0);
    if (foot_mb <= 128)
      pr("wr_row", 100, 100, B, true, n, run<4, true, false>(c, buf, perm, n, 100, 100, 0, true), n * 100.0);
    if (B == 1) {
      pr("wr_slot", 100, 128, B, false, n, run<4, true, false>(c, buf, perm, n, 100, 128, 0, false), n * 100.0);
      pr("wr_int", 100, 100, B, false, n, run<4, true, true>(c, buf, perm, n, 100, 100, 0, false), n * 100.0);
      pr("rd_slot", 100, 128, B, false, n, run<4, false, false>(c, buf, perm, n, 100, 128, 0, false), n * 100.0);
      pr("wr_slot16", 96, 128, B, false, n, run<16, true, false>(c, buf, perm, n, 96, 128, 0, false), n * 96.0);
    }
  }
  return 0;
}
