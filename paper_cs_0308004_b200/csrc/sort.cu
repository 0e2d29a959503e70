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
#include <cstring>
#include <utility>

#include "dpg_internal.cuh"

namespace dpg {

static constexpr int kSThreads = 512;
static constexpr int kSWarps = kSThreads / 32;

__global__ void k_sort_extract(const uint8_t* __restrict__ src, uint32_t rec, uint64_t n,
                               uint32_t key_off, uint32_t key_bytes, uint64_t* __restrict__ khi,
                               uint32_t* __restrict__ klo, uint32_t* __restrict__ rid,
                               const uint32_t* __restrict__ keys_u32, uint64_t key_limit,
                               unsigned long long* status, const uint32_t* cond = nullptr) {
  pdl_wait();                                                 // (launched with PDL: launch_pdl)
  if (cond && *(volatile const uint32_t*)cond == 0) return;   // (the fallback, not needed)
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (keys_u32) {
      // numeric 32-bit keys: the value's bytes, most significant first (a key
      // >= key_limit is reported at its position: referential integrity)
      const uint32_t kv = __ldcs(keys_u32 + i);
      if (kv >= key_limit) report_bad(status, i);
      khi[i] = (uint64_t)kv << 32 | (uint32_t)i;      // the rid rides in the low half
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
  uint64_t chunk;        // elements per CTA (multiple of the tile)
  uint32_t byte;         // key byte of this pass (0 = most significant)
  uint32_t* counts;      // [grid * 256 + 256]
  uint32_t* gbar;        // monotonic grid barrier words
  // Phase I as radix passes (launch_radix_distribute, template SH): the digit
  // is (key word >> shift) & 255 instead of key byte `byte`; SRC passes
  // read the rid list and form the key word (rid << 32) | position, a rid
  // >= n_src becoming 0xFFFFFFFF (reported at its position).
  int32_t shift;
  const uint32_t* rids_in;
  uint64_t n_src;
  unsigned long long* status;
  const uint32_t* cond;   // non-null: the pass runs only if *cond != 0 (the key sort's fallback)
  uint32_t npasses;       // passes in this launch (0 = 1): bytes byte, byte - 1, ...
  // RB passes: run_start[K+1] of the runs (rid >> rb_s, rb_bits digits) of the output
  uint32_t* run_start;
  uint32_t rb_s, rb_bits, rb_K;
};

// Elements per lane of a tile and CTAs per SM.  The key sorts (dpg_sort_rids,
// the DPG-Sort join): 16 per lane (8192-element tiles), one CTA per SM.  Path
// 2's Phase I passes (launch_radix_distribute): 4 per lane, three CTAs of 512
// threads per SM (<= 42 registers, ~55 KB of shared memory each), so one
// CTA's barriers and digit scans overlap the others' memory traffic -- 1.3-1.5x
// faster there, 1.5x slower for the 1 Mi-key sort of config 2, whose CTAs
// hold about one tile each (profiles/r02_radix_occupancy.md).
static constexpr int kSKpt = 16;
static constexpr uint32_t kSTile = kSThreads * kSKpt;
static constexpr int kRKpt = 4, kRCtas = 3;
static constexpr uint32_t kRTile = kSThreads * kRKpt;

__device__ __forceinline__ uint32_t digit_of(uint64_t hi, uint32_t lo, uint32_t byte) {
  return byte < 8 ? (uint32_t)(hi >> (8 * (7 - byte))) & 255u : (lo >> (8 * (11 - byte))) & 255u;
}

// The lanes of `on` (a warp ballot) whose digit d (< 256) equals this
// lane's: eight ballots (cheaper than match.any, whose issue rate is low).
__device__ __forceinline__ uint32_t match_digit(uint32_t d, uint32_t on) {
  uint32_t m = on;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const uint32_t bit = (d >> b) & 1u;
    const uint32_t v = __ballot_sync(0xffffffffu, bit);
    m &= ~(v ^ (0u - bit));                // v if the bit is set, ~v if not
  }
  return m;
}

// One counting-sort pass over key byte a.byte.  LO: the key has a
// low word (key bytes 8..11); RID: the rid travels in its own array (else it
// is packed in the low half of the key word, numeric keys <= 4 bytes).  SRC /
// SH: path 2's radix Phase I (the first pass reads the rid list; the digit is
// a shifted byte of the rid); MP: several passes in one launch; RB: the last
// radix pass also writes the run boundaries.
//   count   the CTA's digit counts, a grid barrier, the bucket bases by a
//           column scan per digit and a second barrier (smaller digits first,
//           then earlier CTAs);
//   place   the chunk in tiles of 512 KPT: warp w takes the tile's elements
//           [32 KPT w, 32 KPT (w + 1)) into registers (KPT per lane, index order =
//           (k, lane)), counts them per digit (warp-private counters), the
//           16 x 256 counters become per-warp offsets into a
//           shared-memory staging area in digit order, and every element goes
//           to its stable position there (rank among equal digits of the same
//           32 elements from ballots); the staged tile then leaves as one
//           contiguous run per digit.  Four CTA barriers per tile.
template <bool LO, bool RID, bool SRC, int KPT = kSKpt, int MINB = 1, bool SH = SRC, bool MP = false,
          bool RB = false>
__global__ void __launch_bounds__(kSThreads, MINB) k_sort_pass(SortPassArgs a0) {
  constexpr uint32_t kTile = kSThreads * KPT;
  pdl_wait();                                                        // (sort_coop_launch)
  if (a0.cond && *(volatile const uint32_t*)a0.cond == 0) return;   // every CTA alike
  extern __shared__ __align__(16) uint8_t sdyn[];
  uint64_t* sk = reinterpret_cast<uint64_t*>(sdyn);                // [kTile]
  uint32_t* sl = reinterpret_cast<uint32_t*>(sdyn + 8 * kTile);    // [kTile] (LO)
  uint32_t* sr = sl + (LO ? kTile : 0);                            // [kTile] (RID)
  __shared__ uint32_t hist[256];       // CTA counts
  __shared__ uint32_t gbase[256];      // first global slot of this CTA's block of digit d
  __shared__ uint32_t run[256];        // elements of digit d written so far (this CTA)
  __shared__ uint32_t woff[kSWarps][256];   // per warp: counts, then staging offsets
  __shared__ uint32_t tl[256];         // staging base of digit d in the current tile
  __shared__ uint32_t tt[256];         // elements of digit d in the current tile
  __shared__ uint32_t delta[256];      // gbase + run - tl: staged position -> global slot
  __shared__ uint32_t wsum[kSWarps];
  // RB (the last radix pass of path 2's Phase I): run boundaries while writing
  __shared__ uint32_t lastb[RB ? 256 : 1];     // run of the last element of digit d written
  __shared__ uint32_t dslot[RB ? 256 : 1], drun[RB ? 256 : 1], ndef;   // deferred firsts
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t c = blockIdx.x, G = gridDim.x;
  // MP (npasses > 1): consecutive passes in one launch (key bytes byte,
  // byte - 1, ...), the buffers swapping after each, a grid barrier between
  // passes.  (Only the key sort's fallback uses it: the per-pass argument copy
  // costs registers, ~20 % per pass on the DPG-Sort join's 64 Mi keys.)
  const uint32_t np = MP ? max(1u, a0.npasses) : 1u;
  for (uint32_t ps = 0; ps < np; ++ps) {
    SortPassArgs a = a0;
    if (ps & 1) {
      a.khi_in = a0.khi_out;
      a.klo_in = a0.klo_out;
      a.rid_in = a0.rid_out;
      a.khi_out = const_cast<uint64_t*>(a0.khi_in);
      a.klo_out = const_cast<uint32_t*>(a0.klo_in);
      a.rid_out = const_cast<uint32_t*>(a0.rid_in);
    }
    a.byte = a0.byte - ps;
    a.shift = a0.shift + 8 * (int32_t)ps;
    if (ps) grid_barrier_mono(a.gbar, G);   // the previous pass's rows, from every CTA
    const uint64_t lo = min_u64(a.n, (uint64_t)c * a.chunk);
    const uint64_t hi = min_u64(a.n, lo + a.chunk);
    const uint32_t byte = a.byte;
    const int32_t shift = a.shift;
    // (SH, a compile-time choice: the key sorts' inner loops keep byte digits)
    auto dig = [&](uint64_t kh, uint32_t kl) -> uint32_t {
      return SH ? (uint32_t)(kh >> shift) & 255u : digit_of(kh, kl, byte);
    };
    // SRC: the key word of element i (rid << 32 | i; 0xFFFFFFFF for a bad rid)
    auto src_word = [&](uint64_t i, uint32_t r) -> uint64_t {
      return (uint64_t)(r < a.n_src ? r : 0xFFFFFFFFu) << 32 | (uint32_t)i;
    };
    for (uint32_t d = tid; d < 256; d += kSThreads) { hist[d] = 0; run[d] = 0; }
    if (RB && tid == 0) ndef = 0;
    // (RB) the run of an element: its truncated run digits, capped at K
    auto run_of = [&](uint64_t k) -> uint32_t {
      uint32_t b = (uint32_t)(k >> 32) >> a.rb_s;
      if (a.rb_bits < 32) b &= (1u << a.rb_bits) - 1u;
      return min(b, a.rb_K);
    };
    __syncthreads();
    // ---- count (only the key word that holds the digit is read) ----
    for (uint64_t i0 = lo + tid; i0 < hi; i0 += 16 * kSThreads) {
      uint32_t dg[16];
  #pragma unroll
      for (int u = 0; u < 16; ++u) {
        const uint64_t i = i0 + u * kSThreads;
        dg[u] = 256;
        if (SRC) {
          if (i < hi) {
            const uint32_t r = __ldcg(a.rids_in + i);
            if (r >= a.n_src) report_bad(a.status, i);
            dg[u] = dig(src_word(i, r), 0u);
          }
        } else if (i < hi) {
          dg[u] = (!LO || byte < 8) ? dig(__ldcg(a.khi_in + i), 0u)
                                    : digit_of(0ull, __ldcg(a.klo_in + i), byte);
        }
      }
  #pragma unroll
      for (int u = 0; u < 16; ++u)
        if (dg[u] < 256) atomicAdd(&hist[dg[u]], 1u);
    }
    __syncthreads();
    for (uint32_t d = tid; d < 256; d += kSThreads) a.counts[c * 256 + d] = hist[d];
    grid_barrier_mono(a.gbar, G);
    // ---- bases, in two steps.  (1) CTA c scans the CTA counts of digits c,
    // c + G, ... (a column prefix over the CTAs, written in place) and writes
    // the digit's total; (2) after a second barrier every CTA reads its own row
    // of column prefixes and the 256 totals.  (Each CTA summing all G rows
    // itself read G^2 * 256 words per pass: 50 M at G = 444.) ----
    uint32_t* tot_w = a.counts + (uint64_t)G * 256;   // [256] digit totals
    for (uint32_t d = c; d < 256; d += G) {
      uint32_t carry = 0;
      for (uint32_t q0 = 0; q0 < G; q0 += kSThreads) {
        const uint32_t q = q0 + tid;
        const uint32_t v = q < G ? __ldcg(a.counts + (uint64_t)q * 256 + d) : 0u;
        uint32_t x = v;
  #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += t;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        uint32_t off = carry;
        for (int w = 0; w < warp; ++w) off += wsum[w];
        if (q < G) a.counts[(uint64_t)q * 256 + d] = off + x - v;
        for (int w = 0; w < kSWarps; ++w) carry += wsum[w];
        __syncthreads();
      }
      if (tid == 0) tot_w[d] = carry;
    }
    grid_barrier_mono(a.gbar, G);
    if (tid < 256) {
      const uint32_t tot = __ldcg(tot_w + tid);
      const uint32_t pre = __ldcg(a.counts + (uint64_t)c * 256 + tid);
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

    const uint32_t wb = warp * 32 * KPT;
    uint64_t kh[KPT];
    uint32_t kl[KPT], rd[KPT];
    // the warp's 512 elements of the tile at t0 into registers (index order =
    // (k, lane)); issued for the next tile before the current one is written out
    auto load_tile = [&](uint64_t t0) {
      const uint32_t cnt = (uint32_t)min_u64(kTile, hi > t0 ? hi - t0 : 0);
  #pragma unroll
      for (int k = 0; k < KPT; ++k) {
        const uint32_t e = wb + k * 32 + lane;
        kh[k] = 0;
        kl[k] = 0;
        rd[k] = 0;
        if (SRC && e < cnt) {
          kh[k] = src_word(t0 + e, __ldcs(a.rids_in + t0 + e));
        } else if (e < cnt) {
          kh[k] = __ldcs(a.khi_in + t0 + e);
          if (LO) kl[k] = __ldcs(a.klo_in + t0 + e);
          if (RID) rd[k] = __ldcs(a.rid_in + t0 + e);
        }
      }
    };
    load_tile(lo);
    for (uint64_t t0 = lo; t0 < hi; t0 += kTile) {
      const uint32_t cnt = (uint32_t)min_u64(kTile, hi - t0);
      // ---- count the warp's elements per digit ----
      uint32_t* wo = woff[warp];
  #pragma unroll
      for (int k = 0; k < 8; ++k) wo[k * 32 + lane] = 0;
      __syncwarp();
  #pragma unroll
      for (int k = 0; k < KPT; ++k)
        if (wb + k * 32 + lane < cnt) atomicAdd(&wo[dig(kh[k], kl[k])], 1u);
      __syncthreads();
      // ---- per-digit tile totals, their scan (staging bases), per-warp offsets ----
      if (tid < 256) {
        uint32_t s2 = 0;
  #pragma unroll
        for (int w = 0; w < kSWarps; ++w) {
          const uint32_t x = woff[w][tid];
          woff[w][tid] = s2;
          s2 += x;
        }
        tt[tid] = s2;
        uint32_t y = s2;
  #pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t t = __shfl_up_sync(0xffffffffu, y, d);
          if (lane >= d) y += t;
        }
        if (lane == 31) wsum[warp] = y;
        tl[tid] = y - s2;
      }
      __syncthreads();
      if (tid < 256) {
        uint32_t off = 0;
        for (int w = 0; w < warp; ++w) off += wsum[w];
        tl[tid] += off;
        delta[tid] = gbase[tid] + run[tid] - tl[tid];
      }
      __syncthreads();
      // ---- place every element at its stable staging position ----
      const uint32_t lt = lanemask_lt();
  #pragma unroll
      for (int k = 0; k < KPT; ++k) {
        const bool on = wb + k * 32 + lane < cnt;
        const uint32_t d = dig(kh[k], kl[k]);
        const uint32_t pm = match_digit(d, __ballot_sync(0xffffffffu, on));
        if (on) {
          const uint32_t pos = tl[d] + wo[d] + __popc(pm & lt);
          sk[pos] = kh[k];
          if (LO) sl[pos] = kl[k];
          if (RID) sr[pos] = rd[k];
        }
        __syncwarp();
        if (on && (pm & lt) == 0) wo[d] += __popc(pm);
        __syncwarp();
      }
      load_tile(t0 + kTile);     // in flight during the write-out
      __syncthreads();
      // ---- write out: staged slot p of digit d goes to gbase[d] + run[d] +
      // p - tl[d]: consecutive threads, consecutive slots of one digit run ----
      for (uint32_t p = tid; p < cnt; p += kSThreads) {
        const uint64_t k = sk[p];
        const uint32_t l = LO ? sl[p] : 0u;
        const uint32_t d = dig(k, l);
        const uint32_t slot = delta[d] + p;
        __stcg(a.khi_out + slot, k);
        if (LO) __stcg(a.klo_out + slot, l);
        if (RID) __stcg(a.rid_out + slot, sr[p]);
        if (RB) {
          // run_start[b'] = slot for the runs b' in (run of the previous
          // element, b]; the previous element is the staged one before, or
          // this CTA's last of digit d; the CTA's first of digit d waits for
          // the end of the pass (its predecessor is another CTA's)
          const uint32_t b = run_of(k);
          uint32_t bp = 0;
          bool known = true;
          if (p > tl[d]) {
            bp = run_of(sk[p - 1]);
          } else if (run[d] > 0) {
            bp = lastb[d];
          } else {
            known = false;
            const uint32_t q = atomicAdd(&ndef, 1u);
            dslot[q] = slot;
            drun[q] = b;
          }
          if (known)
            for (uint32_t bb = bp + 1; bb <= b; ++bb) a.run_start[bb] = slot;
          if (slot + 1 == a.n)
            for (uint32_t bb = b + 1; bb <= a.rb_K; ++bb) a.run_start[bb] = (uint32_t)a.n;
        }
      }
      __syncthreads();
      if (tid < 256) {
        if (RB && tt[tid]) lastb[tid] = run_of(sk[tl[tid] + tt[tid] - 1]);
        run[tid] += tt[tid];
      }
      // (the next tile's first barrier orders this update before the next write-out)
    }
    if (RB) {
      // the deferred firsts: their predecessors, written by other CTAs
      grid_barrier_mono(a.gbar, G);
      for (uint32_t q = tid; q < ndef; q += kSThreads) {
        const uint32_t slot = dslot[q], b = drun[q];
        const uint32_t b0 = slot ? run_of(__ldcg(a.khi_out + slot - 1)) + 1 : 0u;
        for (uint32_t bb = b0; bb <= b; ++bb) a.run_start[bb] = slot;
      }
    }
  }   // passes
}

__global__ void k_keys_u32(const uint64_t* __restrict__ khi, uint64_t n, uint32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)(__ldcs(khi + i) >> 32);
}

__global__ void k_unpack(const uint64_t* __restrict__ khi, uint64_t n, uint32_t* __restrict__ rids,
                         uint32_t* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = __ldcs(khi + i);
    rids[i] = (uint32_t)x;
    if (keys) keys[i] = (uint32_t)(x >> 32);
  }
}

// The key sort's prefix step: after stable passes over the first four key
// bytes, elements with equal 4-byte prefixes are adjacent and in rid order;
// each group of up to kFixMax elements is ordered by the remaining key bytes
// (ties keep rid order) by the thread at its start, and rids_out receives the
// sorted rids.  A longer group sets *overflow: the full sort then runs.
constexpr uint32_t kFixMax = 32;
__global__ void k_sort_fixup(const uint64_t* __restrict__ khi, const uint32_t* __restrict__ klo,
                             const uint32_t* __restrict__ rid, uint64_t n, bool lo_w,
                             uint32_t* __restrict__ rids_out, uint32_t* __restrict__ overflow) {
  pdl_wait();
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t kj = khi[j];
    const uint32_t pj = (uint32_t)(kj >> 32);
    if (j > 0 && (uint32_t)(khi[j - 1] >> 32) == pj) continue;       // not a group start
    uint32_t g = 1;
    while (j + g < n && g <= kFixMax && (uint32_t)(khi[j + g] >> 32) == pj) ++g;
    if (g == 1) {
      rids_out[j] = rid[j];
      continue;
    }
    if (g > kFixMax) {
      atomicOr(overflow, 1u);
      continue;
    }
    uint64_t k[kFixMax];
    uint32_t l[kFixMax], r[kFixMax];
    for (uint32_t e = 0; e < g; ++e) {
      k[e] = khi[j + e];
      l[e] = lo_w ? klo[j + e] : 0u;
      r[e] = rid[j + e];
    }
    for (uint32_t e = 1; e < g; ++e) {      // insertion sort: stable, g <= 32
      const uint64_t ke = k[e];
      const uint32_t le = l[e], re = r[e];
      uint32_t f = e;
      while (f > 0 && (k[f - 1] > ke || (k[f - 1] == ke && l[f - 1] > le))) {
        k[f] = k[f - 1];
        l[f] = l[f - 1];
        r[f] = r[f - 1];
        --f;
      }
      k[f] = ke;
      l[f] = le;
      r[f] = re;
    }
    for (uint32_t e = 0; e < g; ++e) rids_out[j + e] = r[e];
  }
}

template <bool LO, bool RID, bool SRC = false, int KPT = kSKpt, int MINB = 1, bool SH = SRC,
          bool MP = false, bool RB = false>
static cudaError_t set_pass_smem() {
  static int set_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (set_dev == dev) return cudaSuccess;
  const int dyn = (8 + (LO ? 4 : 0) + (RID ? 4 : 0)) * kSThreads * KPT;
  const cudaError_t e = cudaFuncSetAttribute(k_sort_pass<LO, RID, SRC, KPT, MINB, SH, MP, RB>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
  if (e == cudaSuccess) set_dev = dev;
  return e;
}

extern uint32_t g_debug_flags;

// A sort pass: a cooperative launch (grid barriers), with PDL after the
// previous kernel of the sort (pdl_wait) unless the tuning flag 0x40000 asks
// for plain launches (A/B: profiles/r02_pdl.md)
static bool sort_pdl() { return !(g_debug_flags & 0x40000u); }
static cudaError_t sort_coop_launch(const void* fn, int grid, void** params, uint32_t dyn,
                                    cudaStream_t st, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[2];
  unsigned na = 0;
  at[na].id = cudaLaunchAttributeCooperative;
  at[na].val.cooperative = 1;
  ++na;
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kSThreads);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelExC(&cfg, fn, params);
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
  uint32_t* overflow = reinterpret_cast<uint32_t*>(p + al(256ull * 4 * sm + 1024));
  // numeric keys (<= 4 bytes): the rid rides in the low half of the key word;
  // only the key bytes a key below key_limit can have nonzero are sorted on
  const bool packed = keys_u32 != nullptr;
  uint32_t first = 0;
  if (packed && key_limit != ~0ull) {
    uint32_t kb = 0;
    for (uint64_t m = key_limit > 0 ? key_limit - 1 : 0; m; m >>= 8) ++kb;
    first = 4 - max(kb, 1u);
  }
  const bool lo_w = key_bytes > 8;
  const uint32_t g = (uint32_t)max_u64(1, min_u64((n + 255) / 256, (uint64_t)sm * 8));
  const int grid = sm;
  const uint64_t chunk = ((n + grid - 1) / grid + kSTile - 1) / kSTile * kSTile;
  const uint32_t dyn = (8 + (lo_w ? 4 : 0) + (packed ? 0 : 4)) * kSTile;
  const void* fn = packed ? (const void*)k_sort_pass<false, false, false>
                          : lo_w ? (const void*)k_sort_pass<true, true, false>
                                 : (const void*)k_sort_pass<false, true, false>;
  const void* fn_mp = lo_w ? (const void*)k_sort_pass<true, true, false, kSKpt, 1, false, true>
                           : (const void*)k_sort_pass<false, true, false, kSKpt, 1, false, true>;
  cudaError_t e = packed ? set_pass_smem<false, false>()
                         : lo_w ? set_pass_smem<true, true>() : set_pass_smem<false, true>();
  if (e == cudaSuccess && !packed)
    e = lo_w ? set_pass_smem<true, true, false, kSKpt, 1, false, true>()
             : set_pass_smem<false, true, false, kSKpt, 1, false, true>();
  // the passes over key bytes [lo_byte, hi_byte) in LSD order, in one
  // launch, the buffers ping-ponging: the last pass lands in index (passes odd)
  // (one launch per pass; one launch for all of them with `one_launch`)
  auto run_passes = [&](uint32_t lo_byte, uint32_t hi_byte, uint32_t* const rid[2],
                        const uint32_t* cond, bool one_launch) {
    uint32_t in = 0;
    for (uint32_t byte = hi_byte; byte > lo_byte && e == cudaSuccess; --byte, in ^= 1) {
      SortPassArgs sa;
      std::memset(&sa, 0, sizeof(sa));
      sa.khi_in = khi[in];
      sa.klo_in = klo[in];
      sa.rid_in = rid[in];
      sa.khi_out = khi[in ^ 1];
      sa.klo_out = klo[in ^ 1];
      sa.rid_out = rid[in ^ 1];
      sa.n = n;
      sa.chunk = chunk;
      sa.byte = byte - 1;
      sa.counts = counts;
      sa.gbar = gbar;
      sa.shift = -1;
      sa.cond = cond;
      sa.npasses = one_launch ? hi_byte - lo_byte : 1;
      void* params[] = {&sa};
      ++*nl;
      e = sort_coop_launch(one_launch ? fn_mp : fn, grid, params, dyn, st, sort_pdl());
      if (one_launch) break;
    }
  };
  // Keys longer than 4 bytes (the Datamation 10-byte keys): four
  // passes sort by the 4-byte prefix, the short groups of equal prefixes are
  // finished by k_sort_fixup; only if some group is longer (few distinct
  // prefixes) do the extraction and all key_bytes passes run (launched
  // always, each returning at once unless the fixup set the flag).
  if (!packed && key_bytes > 4 && e == cudaSuccess) {
    uint32_t* rid_p[2] = {rid0, rids_out};          // 4 passes: the result in rid0
    // (the flag is cleared first, so that the kernels follow one another:
    // PDL links kernel to kernel)
    if (e == cudaSuccess) e = cudaMemsetAsync(overflow, 0, 4, st);
    ++*nl;
    if (e == cudaSuccess) {
      k_sort_extract<<<g, 256, 0, st>>>(src, rec, n, key_off, key_bytes, khi[0], klo[0], rid_p[0],
                                        nullptr, 0, status);
      e = cudaGetLastError();
    }
    run_passes(0, 4, rid_p, nullptr, false);
    if (e == cudaSuccess) {
      ++*nl;
      e = launch_pdl(k_sort_fixup, dim3(g), dim3(256), 0, st, sort_pdl(), 1,
                     (const uint64_t*)khi[0], (const uint32_t*)klo[0], (const uint32_t*)rid_p[0],
                     n, lo_w, rids_out, overflow);
    }
    uint32_t* rid_f[2] = {rid0, rids_out};
    if (key_bytes % 2 == 0) std::swap(rid_f[0], rid_f[1]);   // the last pass lands in rids_out
    if (e == cudaSuccess) {
      ++*nl;
      e = launch_pdl(k_sort_extract, dim3(g), dim3(256), 0, st, sort_pdl(), 1, src, rec, n,
                     key_off, key_bytes, khi[0], klo[0], rid_f[0], (const uint32_t*)nullptr,
                     (uint64_t)0, status, (const uint32_t*)overflow);
    }
    run_passes(0, key_bytes, rid_f, overflow, true);
    if (e == cudaSuccess && keys_out) {
      // (keys_out is only requested with packed numeric keys)
      e = cudaErrorInvalidValue;
    }
    return e;
  }
  const uint32_t passes = key_bytes - first;
  uint32_t* rid[2] = {rid0, rids_out};
  // the passes alternate buffers; start so that the last pass lands in rids_out
  if (passes % 2 == 0) std::swap(rid[0], rid[1]);
  ++*nl;
  k_sort_extract<<<g, 256, 0, st>>>(src, rec, n, key_off, key_bytes, khi[0], klo[0], rid[0],
                                    keys_u32, key_limit, status);
  if (e == cudaSuccess) e = cudaGetLastError();
  run_passes(first, key_bytes, rid, nullptr, false);
  if (e == cudaSuccess && packed) {
    // the sorted (key, rid) words of the last pass: rids (and keys) out
    ++*nl;
    k_unpack<<<g, 256, 0, st>>>(khi[passes % 2], n, rids_out, keys_out);
    e = cudaGetLastError();
  } else if (e == cudaSuccess && keys_out) {
    ++*nl;
    k_keys_u32<<<g, 256, 0, st>>>(khi[passes % 2], n, keys_out);
    e = cudaGetLastError();
  }
  return e;
}

// Phase I of the multi-kernel plan as stable radix passes over the run index
// b = rid >> s (Fig. 1's "Append r to RID_RUN[run_num]", as a
// counting sort; reading A24): P = ceil(bits(K-1) / 8) passes of
// 8 bits, the first reading the rid list, each writing every element as one
// contiguous run per digit from a shared-memory staged tile.  out[n] (8-byte
// elements (rid << 32) | position, by run, positions ascending inside a run;
// a rid >= n_src is 0xFFFFFFFF and sorts last, into run K-1 at the latest),
// tmp[n] a ping-pong buffer (P >= 2), counts[256 * 3 * sm + 256]; the last
// pass also writes run_start[K+1] from the boundaries of the sorted runs (RB).
uint32_t radix_passes(uint64_t K) {
  uint32_t bits = 0;
  for (uint64_t m = K > 1 ? K - 1 : 0; m; m >>= 1) ++bits;
  return bits ? (bits + 7) / 8 : 1;
}

cudaError_t launch_radix_distribute(const uint32_t* rids, uint64_t n, uint64_t n_src, uint32_t s,
                                    uint32_t K, uint64_t* tmp, uint64_t* out, uint32_t* counts,
                                    uint32_t* gbar, uint32_t* run_start, int sm, cudaStream_t st,
                                    uint32_t* nl, unsigned long long* status) {
  const uint32_t P = radix_passes(K);
  if (n == 0) return cudaMemsetAsync(run_start, 0, ((uint64_t)K + 1) * 4, st);
  const int grid = kRCtas * sm;
  // the pass kinds: first (reads the rids) / later, and the last one also
  // writes the run boundaries (RB)
  const void* f_first = P == 1
      ? (const void*)k_sort_pass<false, false, true, kRKpt, kRCtas, true, false, true>
      : (const void*)k_sort_pass<false, false, true, kRKpt, kRCtas, true, false, false>;
  const void* f_mid = (const void*)k_sort_pass<false, false, false, kRKpt, kRCtas, true, false, false>;
  const void* f_last = (const void*)k_sort_pass<false, false, false, kRKpt, kRCtas, true, false, true>;
  cudaError_t e = set_pass_smem<false, false, true, kRKpt, kRCtas, true, false, true>();
  if (e == cudaSuccess) e = set_pass_smem<false, false, true, kRKpt, kRCtas, true, false, false>();
  if (e == cudaSuccess) e = set_pass_smem<false, false, false, kRKpt, kRCtas, true, false, false>();
  if (e == cudaSuccess) e = set_pass_smem<false, false, false, kRKpt, kRCtas, true, false, true>();
  const uint64_t chunk = ((n + grid - 1) / grid + kRTile - 1) / kRTile * kRTile;
  const uint32_t dyn = 8 * kRTile;
  const uint64_t* in = nullptr;
  for (uint32_t k = 0; k < P && e == cudaSuccess; ++k) {
    uint64_t* o = ((P - 1 - k) % 2 == 0) ? out : tmp;
    SortPassArgs a;
    std::memset(&a, 0, sizeof(a));
    a.khi_in = in;
    a.khi_out = o;
    a.n = n;
    a.chunk = chunk;
    a.counts = counts;
    a.gbar = gbar;
    a.shift = (int32_t)(32 + s + 8 * k);
    a.rids_in = rids;
    a.n_src = n_src;
    a.status = status;
    a.run_start = run_start;
    a.rb_s = s;
    a.rb_bits = 8 * P;
    a.rb_K = K;
    void* params[] = {&a};
    ++*nl;
    const void* fn = k == 0 ? f_first : k + 1 == P ? f_last : f_mid;
    e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kSThreads), params, dyn, st);
    in = o;
  }
  return e;
}

// Test helper (dpg_distribute): radix elements -> (local | pos << 32) with
// local = rid & (L - 1) (0xFFFFFFFF for a bad rid), run_start -> uint64.
__global__ void k_radix_unpack(const uint64_t* __restrict__ e, uint64_t n, uint32_t s,
                               const uint32_t* __restrict__ rs, uint32_t K,
                               uint64_t* __restrict__ out, uint64_t* __restrict__ rs_out) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = t; j < n; j += stride) {
    const uint32_t r = (uint32_t)(e[j] >> 32);
    const uint64_t local = r == 0xFFFFFFFFu ? 0xFFFFFFFFull : (r & ((1ull << s) - 1));
    out[j] = local | (e[j] << 32);
  }
  for (uint64_t b = t; b <= K; b += stride) rs_out[b] = rs[b];
}

cudaError_t launch_radix_unpack(const uint64_t* e, uint64_t n, uint32_t s, const uint32_t* rs,
                                uint32_t K, uint64_t* out, uint64_t* rs_out, cudaStream_t st,
                                uint32_t* nl) {
  ++*nl;
  const uint32_t g = (uint32_t)min_u64(4096, (max_u64(n, K + 1) + 255) / 256);
  k_radix_unpack<<<g, 256, 0, st>>>(e, n, s, rs, K, out, rs_out);
  return cudaGetLastError();
}

uint64_t sort_ws_bytes(uint64_t n, int sm) {
  auto al = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
  return 2 * al(8 * n) + 2 * al(4 * n) + al(4 * n) + al(256ull * 4 * sm + 1024) + 256;
}

// DPG-Sort join, last step: out row j = a[j] (a_bytes, the moved
// R records, sequential) ++ b[idx[j]] (b_bytes, F read in rid_F order:
// non-decreasing idx, so F streams through once).  W-byte words, flat over
// the output (coalesced stores); rows with idx >= n_b stay unwritten.
template <int W>
__global__ void __launch_bounds__(256) k_zip_gather(const uint8_t* __restrict__ a, uint32_t a_bytes,
                                                    const uint8_t* __restrict__ b, uint32_t b_bytes,
                                                    uint64_t n_b, const uint32_t* __restrict__ idx,
                                                    uint64_t n, uint8_t* __restrict__ out,
                                                    unsigned long long* status) {
  using T = typename Word<W>::T;
  const uint32_t AW = a_bytes / W, R = (a_bytes + b_bytes) / W;
  const uint64_t words = n * R;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < words; k += stride) {
    const uint64_t row = k / R;
    const uint32_t w = (uint32_t)(k - row * R);
    const uint32_t f = __ldg(idx + row);
    if (f >= n_b) {
      if (status && w == 0) report_bad(status, row);
      continue;
    }
    const T v = w < AW ? __ldcs(reinterpret_cast<const T*>(a + row * a_bytes) + w)
                       : __ldg(reinterpret_cast<const T*>(b + (uint64_t)f * b_bytes) + (w - AW));
    __stcs(reinterpret_cast<T*>(out) + k, v);
  }
}

cudaError_t launch_zip_gather(const uint8_t* a, uint32_t a_bytes, const uint8_t* b, uint32_t b_bytes,
                              uint64_t n_b, const uint32_t* idx, uint64_t n, uint8_t* out, uint32_t W,
                              int sm, cudaStream_t st, uint32_t* nl, unsigned long long* status) {
  const uint64_t words = n * ((a_bytes + b_bytes) / W);
  const uint32_t grid = (uint32_t)max_u64(1, min_u64((words + 255) / 256, (uint64_t)sm * 8));
  ++*nl;
  switch (W) {
    case 16: k_zip_gather<16><<<grid, 256, 0, st>>>(a, a_bytes, b, b_bytes, n_b, idx, n, out, status); break;
    case 8: k_zip_gather<8><<<grid, 256, 0, st>>>(a, a_bytes, b, b_bytes, n_b, idx, n, out, status); break;
    case 4: k_zip_gather<4><<<grid, 256, 0, st>>>(a, a_bytes, b, b_bytes, n_b, idx, n, out, status); break;
    case 2: k_zip_gather<2><<<grid, 256, 0, st>>>(a, a_bytes, b, b_bytes, n_b, idx, n, out, status); break;
    default: k_zip_gather<1><<<grid, 256, 0, st>>>(a, a_bytes, b, b_bytes, n_b, idx, n, out, status); break;
  }
  return cudaGetLastError();
}

}  // namespace dpg
