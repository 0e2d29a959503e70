// direct.cu -- the standard retrieval the paper measures DPG against
// (P:73-77): "accesses the records of the source data file directly according
// to the sequence of the rids", i.e. dst[i] = src[rid[i]] with one random
// access per record.  Built as the measured GPU comparison (the "naive
// direct-gather" kernel), tuned honestly: each warp owns 32 consecutive
// output rows, lanes cover the words of a row, and a batch of independent
// row loads is issued before any store so many random reads are in flight.
//
// Also the owner-side reply scatter of the multi-GPU path (dst[pos[k]] =
// rows[k]), the same lane layout with the random side on the write.
#include "dpg_internal.cuh"

namespace dpg {

static constexpr int kDirectThreads = 256;

// HINT 0: plain loads and stores.
// HINT 1: both sides are touched exactly once (the INTERNAL -> dst gather of
//         the three-phase DPG): loads and stores carry an L2 evict_first hint.
// HINT 2: the source is an L2-resident run (the single-run DPG, whose run is
//         the whole source, staged into L2): loads evict_last, stores
//         evict_first so the output stream does not evict the run.
template <int W, int HINT>
__global__ void __launch_bounds__(kDirectThreads, 5) k_direct(const uint8_t* __restrict__ src,
                                                              uint64_t n_src, uint32_t rec,
                                                              const uint32_t* __restrict__ rids,
                                                              uint64_t n_out,
                                                              uint8_t* __restrict__ dst,
                                                              unsigned long long* status) {
  using T = typename Word<W>::T;
  const bool STREAM = HINT != 0;
  const uint64_t pol = HINT ? policy_evict_first() : 0;
  const uint64_t lpol = HINT == 2 ? policy_evict_last() : pol;
  // rows in flight per lane per batch: up to 128 bytes of loads per lane, so a
  // warp keeps a whole 32-row group (3.2 KB at 100-B rows) in flight
  constexpr int B = W >= 16 ? 2 : W == 8 ? 4 : 8;
  constexpr int B2 = W >= 16 ? 2 : 4;  // words in flight per lane for rows wider than a warp
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t R = rec / W;
  const uint32_t RPI = R <= 32 ? 32 / R : 1;
  const uint32_t lr = R <= 32 ? lane / R : 0;
  const uint32_t lw = R <= 32 ? lane % R : 0;
  const bool lane_on = R <= 32 ? (uint32_t)lane < RPI * R : true;

  for (uint64_t g0 = gw * 32; g0 < n_out; g0 += nw * 32) {
    const uint64_t i = g0 + lane;
    uint32_t my_r = 0;
    uint32_t my_ok = 0;
    if (i < n_out) {
      my_r = __ldg(rids + i);
      if (my_r < n_src) my_ok = 1;
      else report_bad(status, i);
    }
    const uint32_t cnt = (uint32_t)min_u64(32, n_out - g0);
    if (R <= 32) {
      // bit rr of okm: row g0+rr exists and its rid is valid (lanes >= cnt have my_ok = 0)
      const uint32_t okm = __ballot_sync(0xffffffffu, my_ok) & (lane_on ? 0xffffffffu : 0u);
      const uint8_t* s_lw = src + lw * W;
      uint8_t* d_row = dst + (g0 + lr) * rec + lw * W;
      for (uint32_t k0 = 0; k0 < cnt; k0 += RPI * B) {
        T v[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
          const uint32_t rr = k0 + u * RPI + lr;
          const uint32_t r = __shfl_sync(0xffffffffu, my_r, rr & 31);
          if ((okm >> (rr & 31)) & (rr < 32)) {
            const uint8_t* p = s_lw + (uint64_t)r * rec;
            v[u] = STREAM ? HintIO<W>::ld(p, lpol) : __ldg(reinterpret_cast<const T*>(p));
          }
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
          const uint32_t rr = k0 + u * RPI + lr;
          if ((okm >> (rr & 31)) & (rr < 32)) {
            uint8_t* p = d_row + (uint64_t)(k0 + u * RPI) * rec;
            if (STREAM) HintIO<W>::st(p, v[u], pol);
            else *reinterpret_cast<T*>(p) = v[u];
          }
        }
      }
    } else {
      for (uint32_t rr = 0; rr < cnt; ++rr) {
        const uint32_t r = __shfl_sync(0xffffffffu, my_r, rr);
        const uint32_t o = __shfl_sync(0xffffffffu, my_ok, rr);
        if (!o) continue;
        const uint8_t* s = src + (uint64_t)r * rec;
        uint8_t* d = dst + (g0 + rr) * rec;
        for (uint32_t w0 = 0; w0 < R; w0 += 32 * B2) {
          T v[B2];
#pragma unroll
          for (int u = 0; u < B2; ++u) {
            const uint32_t w = w0 + u * 32 + lane;
            if (w < R) v[u] = __ldg(reinterpret_cast<const T*>(s + w * W));
          }
#pragma unroll
          for (int u = 0; u < B2; ++u) {
            const uint32_t w = w0 + u * 32 + lane;
            if (w < R) *reinterpret_cast<T*>(d + w * W) = v[u];
          }
        }
      }
    }
  }
}

// dst[pos[k]] = rows[k]
template <int W>
__global__ void __launch_bounds__(kDirectThreads) k_scatter_rows(const uint8_t* __restrict__ rows,
                                                                 uint32_t rec,
                                                                 const uint32_t* __restrict__ pos,
                                                                 uint64_t n, uint8_t* __restrict__ dst,
                                                                 uint64_t n_dst) {
  using T = typename Word<W>::T;
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t R = rec / W;
  const uint32_t RPI = R <= 32 ? 32 / R : 1;
  const uint32_t lr = R <= 32 ? lane / R : 0;
  const uint32_t lw = R <= 32 ? lane % R : 0;
  const bool lane_on = R <= 32 ? (uint32_t)lane < RPI * R : true;
  for (uint64_t g0 = gw * 32; g0 < n; g0 += nw * 32) {
    const uint64_t k = g0 + lane;
    const uint32_t my_p = k < n ? __ldg(pos + k) : 0xffffffffu;
    const uint32_t cnt = (uint32_t)min_u64(32, n - g0);
    if (R <= 32) {
#pragma unroll 4
      for (uint32_t k0 = 0; k0 < 32; k0 += RPI) {
        const uint32_t rr = k0 + lr;
        const uint32_t p = __shfl_sync(0xffffffffu, my_p, rr & 31);
        if (lane_on && rr < cnt && p < n_dst)
          *reinterpret_cast<T*>(dst + (uint64_t)p * rec + lw * W) =
              __ldg(reinterpret_cast<const T*>(rows + (g0 + rr) * rec + lw * W));
      }
    } else {
      for (uint32_t rr = 0; rr < cnt; ++rr) {
        const uint32_t p = __shfl_sync(0xffffffffu, my_p, rr);
        if (p >= n_dst) continue;
        for (uint32_t w = lane; w < R; w += 32)
          *reinterpret_cast<T*>(dst + (uint64_t)p * rec + w * W) =
              __ldg(reinterpret_cast<const T*>(rows + (g0 + rr) * rec + w * W));
      }
    }
  }
}

static uint32_t grid_for(uint64_t n_rows, int sm_count) {
  uint64_t warps = (n_rows + 31) / 32;
  uint64_t blocks = (warps + (kDirectThreads / 32) - 1) / (kDirectThreads / 32);
  uint64_t cap = (uint64_t)sm_count * 5;  // 5 x 256 threads = 40 warps per SM (launch bounds)
  return (uint32_t)max_u64(1, min_u64(blocks, cap));
}

template <int STREAM>
static void direct_w(const uint8_t* src, uint64_t n_src, uint32_t rec, const uint32_t* rids,
                     uint64_t n_out, uint8_t* dst, uint32_t W, uint32_t grid,
                     unsigned long long* status, cudaStream_t st) {
  switch (W) {
    case 16: k_direct<16, STREAM><<<grid, kDirectThreads, 0, st>>>(src, n_src, rec, rids, n_out, dst, status); break;
    case 8: k_direct<8, STREAM><<<grid, kDirectThreads, 0, st>>>(src, n_src, rec, rids, n_out, dst, status); break;
    case 4: k_direct<4, STREAM><<<grid, kDirectThreads, 0, st>>>(src, n_src, rec, rids, n_out, dst, status); break;
    case 2: k_direct<2, STREAM><<<grid, kDirectThreads, 0, st>>>(src, n_src, rec, rids, n_out, dst, status); break;
    default: k_direct<1, STREAM><<<grid, kDirectThreads, 0, st>>>(src, n_src, rec, rids, n_out, dst, status); break;
  }
}

cudaError_t launch_direct(const uint8_t* src, uint64_t n_src, uint32_t rec, const uint32_t* rids,
                          uint64_t n_out, uint8_t* dst, uint32_t W, int sm_count,
                          unsigned long long* status, cudaStream_t st, uint32_t* nl,
                          int hint) {
  uint32_t grid = grid_for(n_out, sm_count);
  ++*nl;
  if (hint == 1) direct_w<1>(src, n_src, rec, rids, n_out, dst, W, grid, status, st);
  else if (hint == 2) direct_w<2>(src, n_src, rec, rids, n_out, dst, W, grid, status, st);
  else direct_w<0>(src, n_src, rec, rids, n_out, dst, W, grid, status, st);
  return cudaGetLastError();
}

// Stage [p, p+bytes) into L2 with evict_last priority: 64 KB bulk prefetches
// spread over the grid (cp.async.bulk.prefetch.L2; no completion signal).
__global__ void k_l2_prefetch(const uint8_t* p, uint64_t bytes) {
  const uint64_t pol = policy_evict_last();
  const uint8_t* a0 = reinterpret_cast<const uint8_t*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
  const uint8_t* a1 = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(p + bytes) & ~uintptr_t(15));
  constexpr uint64_t kChunk = 64 << 10;
  const uint64_t n = a1 > a0 ? (uint64_t)(a1 - a0) : 0;
  for (uint64_t off = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * kChunk; off < n;
       off += (uint64_t)gridDim.x * blockDim.x * kChunk)
    bulk_prefetch_l2(a0 + off, (uint32_t)min_u64(kChunk, n - off), pol);
}

cudaError_t launch_l2_prefetch(const void* p, uint64_t bytes, int sm_count, cudaStream_t st,
                               uint32_t* nl) {
  const uint64_t chunks = (bytes + (64 << 10) - 1) / (64 << 10);
  const uint32_t grid = (uint32_t)max_u64(1, min_u64((chunks + 127) / 128, (uint64_t)sm_count));
  ++*nl;
  k_l2_prefetch<<<grid, 128, 0, st>>>(reinterpret_cast<const uint8_t*>(p), bytes);
  return cudaGetLastError();
}

// DPG-Move join, last step: "join the temporary file with the remaining
// relation" -- out row i = a[i] (a_bytes) ++ b[i] (b_bytes), all
// three streams sequential.  Lanes cover the words of consecutive rows.
template <int W>
__global__ void __launch_bounds__(256) k_zip_rows(const uint8_t* __restrict__ a, uint32_t a_bytes,
                                                  const uint8_t* __restrict__ b, uint32_t b_bytes,
                                                  uint64_t n, uint8_t* __restrict__ out,
                                                  const uint32_t* __restrict__ key, uint64_t key_limit) {
  using T = typename Word<W>::T;
  const uint32_t AW = a_bytes / W, R = (a_bytes + b_bytes) / W;
  const uint64_t words = n * R;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < words; k += stride) {
    const uint64_t row = k / R;
    const uint32_t w = (uint32_t)(k - row * R);
    // a row whose key failed the integrity check has no b part: left unwritten
    if (key && (uint64_t)__ldg(key + row) >= key_limit) continue;
    const T v = w < AW ? __ldg(reinterpret_cast<const T*>(a + row * a_bytes) + w)
                       : __ldg(reinterpret_cast<const T*>(b + row * b_bytes) + (w - AW));
    reinterpret_cast<T*>(out)[k] = v;
  }
}

cudaError_t launch_zip_rows(const uint8_t* a, uint32_t a_bytes, const uint8_t* b, uint32_t b_bytes,
                            uint64_t n, uint8_t* out, uint32_t W, int sm_count, cudaStream_t st,
                            uint32_t* nl, const uint32_t* key, uint64_t key_limit) {
  const uint64_t words = n * ((a_bytes + b_bytes) / W);
  const uint32_t grid = (uint32_t)max_u64(1, min_u64((words + 255) / 256, (uint64_t)sm_count * 8));
  ++*nl;
  switch (W) {
    case 16: k_zip_rows<16><<<grid, 256, 0, st>>>(a, a_bytes, b, b_bytes, n, out, key, key_limit); break;
    case 8: k_zip_rows<8><<<grid, 256, 0, st>>>(a, a_bytes, b, b_bytes, n, out, key, key_limit); break;
    case 4: k_zip_rows<4><<<grid, 256, 0, st>>>(a, a_bytes, b, b_bytes, n, out, key, key_limit); break;
    case 2: k_zip_rows<2><<<grid, 256, 0, st>>>(a, a_bytes, b, b_bytes, n, out, key, key_limit); break;
    default: k_zip_rows<1><<<grid, 256, 0, st>>>(a, a_bytes, b, b_bytes, n, out, key, key_limit); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_scatter_rows(const uint8_t* rows, uint32_t rec, const uint32_t* pos, uint64_t n,
                                uint8_t* dst, uint64_t n_dst, uint32_t W, int sm_count,
                                cudaStream_t st, uint32_t* nl) {
  uint32_t grid = grid_for(n, sm_count);
  ++*nl;
  switch (W) {
    case 16: k_scatter_rows<16><<<grid, kDirectThreads, 0, st>>>(rows, rec, pos, n, dst, n_dst); break;
    case 8: k_scatter_rows<8><<<grid, kDirectThreads, 0, st>>>(rows, rec, pos, n, dst, n_dst); break;
    case 4: k_scatter_rows<4><<<grid, kDirectThreads, 0, st>>>(rows, rec, pos, n, dst, n_dst); break;
    case 2: k_scatter_rows<2><<<grid, kDirectThreads, 0, st>>>(rows, rec, pos, n, dst, n_dst); break;
    default: k_scatter_rows<1><<<grid, kDirectThreads, 0, st>>>(rows, rec, pos, n, dst, n_dst); break;
  }
  return cudaGetLastError();
}

}  // namespace dpg
