// datagen/gen_cuda.cu -- the same counter-based input generators as gen.c,
// evaluated on the GPU for inputs too large to build on the host (the
// multi-GPU configuration: 2^30 records).  Holds none of the method's
// arithmetic.  Bit-identical to gen.c (tests/test_gpu_datagen.py).
#include <cstdint>
#include <cuda_runtime.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL

__host__ __device__ static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static inline uint64_t stream_key(uint64_t seed, uint64_t sid) {
  return mix64(seed * GOLDEN ^ mix64(sid + 0x5851F42D4C957F2DULL));
}

// out[j] = byte (off + j) of stream key; off % 8 == 0, n % 8 == 0
__global__ void k_bytes(uint64_t key, uint64_t w0, uint64_t nw, uint64_t* out) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nw;
       t += (uint64_t)gridDim.x * blockDim.x)
    out[t] = mix64(key + (w0 + t + 1) * GOLDEN);
}

__device__ static inline uint64_t feistel_once(uint64_t key, unsigned half, unsigned rounds,
                                               uint64_t x) {
  const uint64_t mask = (1ULL << half) - 1;
  uint64_t l = x >> half, r = x & mask;
  for (unsigned i = 0; i < rounds; ++i) {
    uint64_t f = mix64(key ^ (r * GOLDEN) ^ ((uint64_t)(i + 1) << 56)) & mask;
    uint64_t nl = r, nr = l ^ f;
    l = nl;
    r = nr;
  }
  return (l << half) | r;
}

__global__ void k_feistel(uint64_t key, unsigned half, unsigned rounds, uint64_t n, uint64_t first,
                          uint64_t count, uint64_t* out) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count;
       j += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t x = feistel_once(key, half, rounds, first + j);
    while (x >= n) x = feistel_once(key, half, rounds, x);
    out[j] = x;
  }
}

extern "C" {

// bytes [off, off + n) of stream (seed, sid) into device buffer out (n, off multiples of 8)
int gen_bytes_cuda(uint64_t seed, uint64_t sid, uint64_t off, uint64_t n, void* out, void* stream) {
  if ((off | n) & 7) return 1;
  const uint64_t nw = n / 8;
  if (!nw) return 0;
  const unsigned grid = (unsigned)((nw + 255) / 256 < 148 * 32 ? (nw + 255) / 256 : 148 * 32);
  k_bytes<<<grid, 256, 0, (cudaStream_t)stream>>>(stream_key(seed, sid), off / 8, nw, (uint64_t*)out);
  return cudaGetLastError() != cudaSuccess;
}

int gen_feistel_cuda(uint64_t seed, uint64_t sid, unsigned bits, unsigned rounds, uint64_t n,
                     uint64_t first, uint64_t count, void* out, void* stream) {
  if (!count) return 0;
  const unsigned grid = (unsigned)((count + 255) / 256 < 148 * 32 ? (count + 255) / 256 : 148 * 32);
  k_feistel<<<grid, 256, 0, (cudaStream_t)stream>>>(stream_key(seed, sid), bits / 2, rounds, n,
                                                    first, count, (uint64_t*)out);
  return cudaGetLastError() != cudaSuccess;
}

}  // extern "C"
