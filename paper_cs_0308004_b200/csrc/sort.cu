// sort.cu -- three-phase key-pointer sorting with DPG as phase 3 (section 3,
// P:481-490; "DPG acts as an accelerator for ... main memory sorting
// algorithms"; the Datamation shape).
//
//   phase 1  k_sort_extract: the key-pointer pairs -- each record's key
//            (key_bytes <= 12 unsigned bytes at key_off) as a big-endian
//            (hi: bytes 0..7, lo: bytes 8..11) pair and its rid.
//   phase 2  k_sort_pass x key_bytes: a stable LSD radix sort, one byte of the
//            key per pass from the last to the first (a counting sort per
//            byte: "count the number of elements destined for each bucket,
//            set bucket boundaries, distribute").  One cooperative
//            kernel per pass: per-CTA digit counts, a grid barrier, every CTA
//            derives its bucket bases, then the CTA's chunk is distributed
//            in order, 512 elements (one row) at a time: a rank inside the
//            warp (match_any), the warps' counts before it, the CTA's
//            running count of the digit -- so equal digits keep their order
//            (stable), which makes the LSD sort correct.
//   phase 3  dpg_retrieve of the records in the sorted rid order (api.cu).
#include "dpg_internal.cuh"

namespace dpg {

static constexpr int kSThreads = 512;
static constexpr int kSWarps = kSThreads / 32;

__global__ void k_sort_extract(const uint8_t* __restrict__ src, uint32_t rec, uint64_t n,
                               uint32_t key_off, uint32_t key_bytes, uint64_t* __restrict__ khi,
                               uint32_t* __restrict__ klo, uint32_t* __restrict__ rid,
                               const uint32_t* __restrict__ keys_u32, uint64_t key_limit,
                               unsigned long long* status) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (keys_u32) {
      // numeric 32-bit keys: the value's bytes, most significant first (a key
      // >= key_limit is reported at its position: referential integrity)
      const uint32_t kv = __ldcs(keys_u32 + i);
      if (kv >= key_limit) report_bad(status, i);
      khi[i] = (uint64_t)kv << 32;
      rid[i] = (uint32_t)i;
      continue;
    }
    const uint8_t* k = src + i * rec + key_off;
    uint64_t hi = 0;
    uint32_t lo = 0;
#pragma unroll
    for (uint32_t b = 0; b < 8; ++b) hi = (hi << 8) | (b < key_bytes ? k[b] : 0u);
#pragma unroll
    for (uint32_t b = 8; b < 12; ++b) lo = (lo << 8) | (b < key_bytes ? k[b] : 0u);
    khi[i] = hi;
    if (key_bytes > 8) klo[i] = lo;
    rid[i] = (uint32_t)i;
  }
}

struct SortPassArgs {
  const uint64_t* khi_in;
  const uint32_t* klo_in;
  const uint32_t* rid_in;
  uint64_t* khi_out;
  uint32_t* klo_out;
  uint32_t* rid_out;
  uint64_t n;
  uint64_t chunk;        // elements per CTA (multiple of kSThreads)
  uint32_t byte;         // key byte of this pass (0 = most significant)
  uint32_t with_lo;      // key_bytes > 8: carry the low word
  uint32_t* counts;      // [256 * grid]
  uint32_t* gbar;        // monotonic grid barrier words
  uint32_t cache;        // 1: each tile is staged in shared memory, written out as bucket runs
  uint32_t tile;         // elements per tile (staging capacity)
};

__device__ __forceinline__ uint32_t digit_of(uint64_t hi, uint32_t lo, uint32_t byte) {
  return byte < 8 ? (uint32_t)(hi >> (8 * (7 - byte))) & 255u : (lo >> (8 * (11 - byte))) & 255u;
}

__global__ void __launch_bounds__(kSThreads, 1) k_sort_pass(SortPassArgs a) {
  // with a.cache: [chunk] khi, [chunk] klo, [chunk] rid of the chunk in bucket
  // order (staged, then written out as one contiguous run per bucket)
  extern __shared__ __align__(16) uint8_t sdyn[];
  __shared__ uint32_t hist[256];       // CTA counts
  __shared__ uint32_t gbase[256];      // first global slot of this CTA's block of digit d
  __shared__ uint32_t run[256];        // elements of digit d placed so far (this CTA)
  __shared__ uint32_t wcnt[kSWarps][256];   // (row tag << 16 | count) per warp and digit
  __shared__ uint32_t wsum[kSWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t c = blockIdx.x, G = gridDim.x;
  const uint64_t lo = min_u64(a.n, (uint64_t)c * a.chunk);
  const uint64_t hi = min_u64(a.n, lo + a.chunk);
  for (uint32_t d = tid; d < 256; d += kSThreads) { hist[d] = 0; run[d] = 0; }
  for (uint32_t k = tid; k < kSWarps * 256; k += kSThreads) (&wcnt[0][0])[k] = 0xFFFF0000u;
  __syncthreads();
  // ---- count ----
  for (uint64_t i0 = lo + tid; i0 < hi; i0 += 4 * kSThreads) {
    uint64_t kh[4];
    uint32_t kl[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t i = i0 + u * kSThreads;
      kh[u] = 0; kl[u] = 0;
      if (i < hi) {
        kh[u] = __ldcg(a.khi_in + i);
        if (a.with_lo) kl[u] = __ldcg(a.klo_in + i);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + u * kSThreads < hi) atomicAdd(&hist[digit_of(kh[u], kl[u], a.byte)], 1u);
  }
  __syncthreads();
  for (uint32_t d = tid; d < 256; d += kSThreads) a.counts[c * 256 + d] = hist[d];
  grid_barrier_mono(a.gbar, G);
  // ---- bases: global (smaller digits, then earlier CTAs) and local; the
  // CTA rows of counts are read coalesced, 8 independent loads in flight ----
  if (tid < 256) {
    uint32_t tot = 0, pre = 0;
    uint32_t q = 0;
    for (; q + 8 <= G; q += 8) {
      uint32_t x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = __ldcg(a.counts + (q + u) * 256 + tid);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        tot += x[u];
        if (q + u < c) pre += x[u];
      }
    }
    for (; q < G; ++q) {
      const uint32_t x = __ldcg(a.counts + q * 256 + tid);
      tot += x;
      if (q < c) pre += x;
    }
    uint32_t y = tot;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, y, d);
      if (lane >= d) y += t;
    }
    if (lane == 31) wsum[warp] = y;
    gbase[tid] = y - tot + pre;
  }
  __syncthreads();
  if (tid < 256) {
    uint32_t off = 0;
    for (int w = 0; w < warp; ++w) off += wsum[w];
    gbase[tid] += off;
  }
  __syncthreads();
  uint64_t* sk = reinterpret_cast<uint64_t*>(sdyn);
  uint32_t* sl = reinterpret_cast<uint32_t*>(sdyn + 8 * a.tile);
  uint32_t* sr = sl + a.tile;
  __shared__ uint32_t th[256];         // digit counts of the current tile
  __shared__ uint32_t tl[256];         // their exclusive scan (tile staging bases)
  uint32_t tag = 0;
  // the CTA's chunk in tiles of a.tile elements (staged in shared memory and
  // written out as one contiguous run per digit); rows of 512 in order
  for (uint64_t t0 = lo; t0 < hi; t0 += a.tile) {
    const uint64_t t1 = min_u64(hi, t0 + a.tile);
    if (a.cache) {
      // tile histogram and its scan
      for (uint32_t d = tid; d < 256; d += kSThreads) th[d] = 0;
      __syncthreads();
      for (uint64_t i = t0 + tid; i < t1; i += kSThreads)
        atomicAdd(&th[digit_of(__ldcg(a.khi_in + i), a.with_lo ? __ldcg(a.klo_in + i) : 0u, a.byte)], 1u);
      __syncthreads();
      if (tid < 256) {
        const uint32_t x = th[tid];
        uint32_t y = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t t = __shfl_up_sync(0xffffffffu, y, d);
          if (lane >= d) y += t;
        }
        if (lane == 31) wsum[warp] = y;
        tl[tid] = y - x;
      }
      __syncthreads();
      if (tid < 256) {
        uint32_t off = 0;
        for (int w = 0; w < warp; ++w) off += wsum[w];
        tl[tid] += off;
      }
      __syncthreads();
    }
    // elements of this tile placed so far, per digit (the CTA's running count
    // run[] holds the tiles before)
    __shared__ uint32_t trun[256];
    for (uint32_t d = tid; d < 256; d += kSThreads) trun[d] = 0;
    __syncthreads();
    auto load_row = [&](uint64_t r0, uint64_t& kh, uint32_t& kl, uint32_t& rd) {
      const uint64_t i = r0 + tid;
      kh = 0; kl = 0; rd = 0;
      if (r0 < t1 && i < t1) {
        kh = __ldcs(a.khi_in + i);
        if (a.with_lo) kl = __ldcs(a.klo_in + i);
        rd = __ldcs(a.rid_in + i);
      }
    };
    uint64_t nh0, nh1;
    uint32_t nl0, nl1, nr0, nr1;
    load_row(t0, nh0, nl0, nr0);
    load_row(t0 + kSThreads, nh1, nl1, nr1);
    for (uint64_t r0 = t0; r0 < t1; r0 += kSThreads, ++tag) {
      const uint64_t i = r0 + tid;
      const bool on = i < t1;
      const uint64_t kh = nh0;
      const uint32_t kl = nl0, rd = nr0;
      nh0 = nh1; nl0 = nl1; nr0 = nr1;
      load_row(r0 + 2 * kSThreads, nh1, nl1, nr1);
      const uint32_t d = on ? digit_of(kh, kl, a.byte) : 256u + lane;   // off lanes: unique dummies
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      const uint32_t rank = __popc(peers & lanemask_lt());
      const uint32_t t16 = (tag & 0xFFFFu) << 16;
      if (on && rank == 0) wcnt[warp][d] = t16 | __popc(peers);
      __syncthreads();
      if (on) {
        uint32_t before = 0;
        for (int w = 0; w < warp; ++w) {
          const uint32_t x = wcnt[w][d];
          before += (x & 0xFFFF0000u) == t16 ? (x & 0xFFFFu) : 0u;
        }
        const uint32_t k = trun[d] + before + rank;   // stable rank of the element in the tile
        if (a.cache) {
          const uint32_t p = tl[d] + k;
          sk[p] = kh;
          sl[p] = kl;
          sr[p] = rd;
        } else {
          const uint32_t slot = gbase[d] + run[d] + k;
          a.khi_out[slot] = kh;
          if (a.with_lo) a.klo_out[slot] = kl;
          a.rid_out[slot] = rd;
        }
      }
      __syncthreads();
      if (tid < 256) {
        uint32_t add = 0;
        for (int w = 0; w < kSWarps; ++w) {
          const uint32_t x = wcnt[w][tid];
          add += (x & 0xFFFF0000u) == t16 ? (x & 0xFFFFu) : 0u;
        }
        trun[tid] += add;
      }
      __syncthreads();
    }
    if (a.cache) {
      // ---- write out: staged slot p of digit d goes to gbase[d] + run[d] +
      // p - tl[d]: consecutive threads, consecutive slots of one bucket run ----
      const uint32_t cnt = (uint32_t)(t1 - t0);
      for (uint32_t p = tid; p < cnt; p += kSThreads) {
        const uint64_t kh = sk[p];
        const uint32_t kl = sl[p];
        const uint32_t d = digit_of(kh, kl, a.byte);
        const uint32_t slot = gbase[d] + run[d] + (p - tl[d]);
        a.khi_out[slot] = kh;
        if (a.with_lo) a.klo_out[slot] = kl;
        a.rid_out[slot] = sr[p];
      }
      __syncthreads();
    }
    for (uint32_t d = tid; d < 256; d += kSThreads) run[d] += trun[d];
    __syncthreads();
  }
}

__global__ void k_keys_u32(const uint64_t* __restrict__ khi, uint64_t n, uint32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)(__ldcs(khi + i) >> 32);
}

cudaError_t launch_sort_rids(const uint8_t* src, uint32_t rec, uint64_t n, uint32_t key_off,
                             uint32_t key_bytes, uint8_t* ws, uint32_t* rids_out, uint32_t* gbar,
                             int sm, cudaStream_t st, uint32_t* nl, const uint32_t* keys_u32,
                             uint32_t* keys_out, uint64_t key_limit, unsigned long long* status) {
  // ws: [khi 0 | khi 1 | klo 0 | klo 1 | rid 0 | counts], 256-byte aligned pieces
  auto al = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
  uint64_t* khi[2] = {reinterpret_cast<uint64_t*>(ws), reinterpret_cast<uint64_t*>(ws + al(8 * n))};
  uint8_t* p = ws + 2 * al(8 * n);
  uint32_t* klo[2] = {reinterpret_cast<uint32_t*>(p), reinterpret_cast<uint32_t*>(p + al(4 * n))};
  p += 2 * al(4 * n);
  uint32_t* rid0 = reinterpret_cast<uint32_t*>(p);
  p += al(4 * n);
  uint32_t* counts = reinterpret_cast<uint32_t*>(p);
  uint32_t* rid[2] = {rid0, rids_out};
  // the passes alternate buffers; start so that the last pass lands in rids_out
  if (key_bytes % 2 == 0) {
    uint32_t* t = rid[0];
    rid[0] = rid[1];
    rid[1] = t;
  }
  ++*nl;
  const uint32_t g = (uint32_t)max_u64(1, min_u64((n + 255) / 256, (uint64_t)sm * 8));
  k_sort_extract<<<g, 256, 0, st>>>(src, rec, n, key_off, key_bytes, khi[0], klo[0], rid[0],
                                    keys_u32, key_limit, status);
  cudaError_t e = cudaGetLastError();
  const uint64_t chunk = ((n + sm - 1) / sm + kSThreads - 1) / kSThreads * kSThreads;
  // staging of one tile (16 B per element): 8192 elements = 128 KB
  const uint32_t tile = 8192;
  uint32_t dyn = 16 * tile;
  {
    static int set_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (set_dev != dev) {
      if (cudaFuncSetAttribute(k_sort_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn) !=
          cudaSuccess) {
        cudaGetLastError();
        dyn = 0;
      } else {
        set_dev = dev;
      }
    }
  }
  uint32_t in = 0;
  for (int byte = (int)key_bytes - 1; byte >= 0 && e == cudaSuccess; --byte, in ^= 1) {
    SortPassArgs s;
    s.khi_in = khi[in];
    s.klo_in = klo[in];
    s.rid_in = rid[in];
    s.khi_out = khi[in ^ 1];
    s.klo_out = klo[in ^ 1];
    s.rid_out = rid[in ^ 1];
    s.n = n;
    s.chunk = chunk;
    s.byte = (uint32_t)byte;
    s.with_lo = key_bytes > 8;
    s.counts = counts;
    s.gbar = gbar;
    s.cache = dyn ? 1 : 0;
    s.tile = dyn ? tile : kSThreads;
    void* params[] = {&s};
    ++*nl;
    e = cudaLaunchCooperativeKernel((const void*)k_sort_pass, dim3(sm), dim3(kSThreads), params, dyn,
                                    st);
  }
  if (e == cudaSuccess && keys_out) {
    // the sorted keys (numeric mode): the last pass's key buffer
    ++*nl;
    k_keys_u32<<<g, 256, 0, st>>>(khi[key_bytes % 2], n, keys_out);
    e = cudaGetLastError();
  }
  return e;
}

uint64_t sort_ws_bytes(uint64_t n, int sm) {
  auto al = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
  return 2 * al(8 * n) + 2 * al(4 * n) + al(4 * n) + al(256ull * 4 * sm) + 256;
}

// DPG-Sort join, last step: out row j = a[j] (a_bytes, the moved
// R records, sequential) ++ b[idx[j]] (b_bytes, F read in rid_F order:
// non-decreasing idx, so F streams through once).  W-byte words, flat over
// the output (coalesced stores); rows with idx >= n_b stay unwritten.
template <int W>
__global__ void __launch_bounds__(256) k_zip_gather(const uint8_t* __restrict__ a, uint32_t a_bytes,
                                                    const uint8_t* __restrict__ b, uint32_t b_bytes,
                                                    uint64_t n_b, const uint32_t* __restrict__ idx,
                                                    uint64_t n, uint8_t* __restrict__ out) {
  using T = typename Word<W>::T;
  const uint32_t AW = a_bytes / W, R = (a_bytes + b_bytes) / W;
  const uint64_t words = n * R;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < words; k += stride) {
    const uint64_t row = k / R;
    const uint32_t w = (uint32_t)(k - row * R);
    const uint32_t f = __ldg(idx + row);
    if (f >= n_b) continue;
    const T v = w < AW ? __ldcs(reinterpret_cast<const T*>(a + row * a_bytes) + w)
                       : __ldg(reinterpret_cast<const T*>(b + (uint64_t)f * b_bytes) + (w - AW));
    __stcs(reinterpret_cast<T*>(out) + k, v);
  }
}

cudaError_t launch_zip_gather(const uint8_t* a, uint32_t a_bytes, const uint8_t* b, uint32_t b_bytes,
                              uint64_t n_b, const uint32_t* idx, uint64_t n, uint8_t* out, uint32_t W,
                              int sm, cudaStream_t st, uint32_t* nl) {
  const uint64_t words = n * ((a_bytes + b_bytes) / W);
  const uint32_t grid = (uint32_t)max_u64(1, min_u64((words + 255) / 256, (uint64_t)sm * 8));
  ++*nl;
  switch (W) {
    case 16: k_zip_gather<16><<<grid, 256, 0, st>>>(a, a_bytes, b, b_bytes, n_b, idx, n, out); break;
    case 8: k_zip_gather<8><<<grid, 256, 0, st>>>(a, a_bytes, b, b_bytes, n_b, idx, n, out); break;
    case 4: k_zip_gather<4><<<grid, 256, 0, st>>>(a, a_bytes, b, b_bytes, n_b, idx, n, out); break;
    case 2: k_zip_gather<2><<<grid, 256, 0, st>>>(a, a_bytes, b, b_bytes, n_b, idx, n, out); break;
    default: k_zip_gather<1><<<grid, 256, 0, st>>>(a, a_bytes, b, b_bytes, n_b, idx, n, out); break;
  }
  return cudaGetLastError();
}

}  // namespace dpg
