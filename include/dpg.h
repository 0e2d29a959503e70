/*
 * dpg.h -- C ABI of the B200-native DPG record-retrieval library (libdpg.so).
 *
 * The paper: "distribute-probe-gather" (DPG), arXiv cs/0308004.  Citations:
 * P:n = line n of the paper's LaTeX body, in the section named.
 *
 * The record-retrieval problem (section 2): given a data file R of
 * fixed-size records and a sequence of record ids S_rid, fill a destination
 * file D with
 *         for each i,  D[i] = R[S_rid[i]]
 * The rid sequence may be a permutation (sort phase 3, section 3)
 * or repeat rids (joins).  DPG computes exactly this result in
 * three phases (section 2.1, Fig. 1): Distribute the rids
 * into runs by their high bits, Probe each cache-resident run of the input,
 * Gather the probed records back into rid order.  On B200 the "cache" is
 * the L2 or shared memory: a source within the L2 budget is one
 * run, staged into the L2 by TMA bulk copies and probed in output order
 * (path 3); larger sources are cut into shared-memory runs whose probe
 * writes each record straight to its destination (paths 1/2; path 2 also
 * after a skew sample), into K L2-sized runs with an INTERNAL file (path 5:
 * records in 4-byte words of 36..116 bytes, and very large sources), or --
 * small records -- into three sequential passes
 * (path 6).  dpg_plan_t.path below lists the plans.
 *
 * Conventions (all entry points):
 *  - Pointers named src/rids/dst/fact/fk_col/dim/out are DEVICE pointers
 *    owned by the caller; the library never frees or retains them.  Records
 *    are laid out back to back: record j occupies bytes [j*rec, (j+1)*rec).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Calls are asynchronous w.r.t. the host and stream-ordered; the
 *    inputs must stay valid until the stream reaches the call.  Scratch space
 *    is library-owned and stream-ordered (cudaMallocAsync/cudaFreeAsync on
 *    `stream`), so calls on different streams may run concurrently.
 *  - Host-detected errors return immediately and enqueue nothing:
 *    DPG_ERR_INVALID_ARG for a NULL pointer with a nonzero count, rec == 0,
 *    n_src == 0 with n_out > 0, byte-size overflow, or dst overlapping an
 *    input (the paper always copies into a separate destination);
 *    DPG_ERR_UNSUPPORTED for n_out >= 2^32.
 *  - Scratch comes from a private stream-ordered memory pool per device (the
 *    process's default pool is not touched); the plans' persistent workspaces
 *    are cached per (device, stream), at most 8 of them (least recently used
 *    idle ones are freed).  A call holds its stream's workspace until its
 *    kernels are enqueued, so two host threads may drive the same stream.
 *    dpg_release_cache() frees every cached buffer and trims the pool.
 *  - n_out == 0 is a no-op returning DPG_OK.
 *  - Device-detected errors: a rid >= n_src (an fk >= n_dim) is skipped, its
 *    destination row is left unwritten, and the smallest offending position
 *    is recorded in a per-device status word.  dpg_sync_status() reports it.
 *  - Any rec >= 1 and any pointer alignment is supported; 16-byte aligned
 *    pointers with rec % 16 == 0 (or % 4 == 0) take the widest vector path.
 */
#ifndef DPG_H
#define DPG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DPG_OK = 0,
    DPG_ERR_INVALID_ARG = 1,
    DPG_ERR_RID_RANGE = 2,
    DPG_ERR_UNSUPPORTED = 3,
    DPG_ERR_OOM = 4,
    DPG_ERR_CUDA = 5,
    DPG_ERR_NCCL = 6
} dpg_status_t;

typedef void *dpg_stream_t; /* a cudaStream_t */

/* Execution plan chosen for one call (host-side; no GPU needed; the skew
 * sample of dpg_retrieve may still switch path 1 to path 2 at run time,
 * dpg_last_path).  Run length L = 2^log2_run records (runs sized
 * to the cache, power of two, identified by the high-order bits of the
 * rid): the whole source for path 3, one shared-memory stage for paths 1/2,
 * one L2 run budget for path 5. */
typedef struct {
    uint32_t log2_run;      /* s: run of rid r is r >> s (reading A1)           */
    uint32_t pair_bytes;    /* 4 = packed (pos << s | local), 8 = (local, pos)  */
    uint64_t run_len;       /* L = 2^s                                          */
    uint64_t num_runs;      /* K = ceil(n_src / L)                              */
    uint32_t word_bytes;    /* vector width of the record copy (1..16)          */
    uint32_t slot_pairs;    /* pairs staged per shared-memory stage             */
    uint32_t smem_bytes;    /* dynamic shared memory of the probe-gather kernel */
    uint32_t grid_distribute; /* CTAs of the distribute kernels (chunks)        */
    uint32_t grid_probe;    /* CTAs of the persistent probe-gather kernel       */
    uint32_t hist_in_smem;  /* 1: per-CTA run histogram in shared memory        */
    uint32_t pay_bytes;     /* payload bytes carried per pair (join: fact row)  */
    uint32_t path;          /* 1 = one persistent cooperative kernel (fused.cu)
                               2 = distribute kernels (counting, or stable
                                   radix passes: dist_radix) + probe-gather
                                   kernel over work items (run, chunk)
                               3 = one L2-resident run (l2run.cu): the source
                                   fits the L2 budget, K = 1; Phase II loads it
                                   into L2, Phase III probes it in rid order
                                   writing dst sequentially
                               4 = two L2 runs (l2pair.cu): Phase I compaction,
                                   run 0 probed into INTERNAL, run 1 fused with
                                   Phase III (one cooperative kernel)
                               5 = K L2 runs (l2k.cu): Phase I distribute
                                   kernel, K staged probes into INTERNAL,
                                   Phase III gather
                               6 = three sequential passes (seq3.cu), small
                                   records: tile-sorted RID_RUN, run probes
                                   into a tile-major INTERNAL, tile gathers
                               7 = two levels: owner super-runs, path 6 in
                                   each, one gather back                       */
    uint32_t nstages;       /* shared-memory stages of the probe-gather pipeline */
    uint32_t stage_bytes;   /* bytes per stage                                  */
    uint32_t gather;        /* 1 = probe writes rows straight to dst (rows are
                               whole 32-B sectors); 2 = INTERNAL file + gather
                               (Fig. 1 literally; rows straddle sectors)       */
    uint32_t npre;          /* source runs prefetched before Phase I (fused)    */
    uint32_t rid_cache;     /* 1: each CTA's rid chunk is staged in smem (fused) */
    uint32_t hist_warps;    /* warps owning private 16-bit run counters (fused) */
    uint32_t tile;          /* rids per Phase I tile of a CTA (fused, path 6)   */
    uint32_t cluster;       /* path 6: CTAs (SMs) whose shared memory holds one
                               run together (thread-block cluster, DSMEM)      */
    uint32_t dist_radix;    /* path 2: Phase I as this many stable 8-bit radix
                               passes over the run index (0 = counting
                               distribute with atomics)                        */
} dpg_plan_t;

/* Optional overrides for tests and tuning (zero = automatic).  The output
 * of every call is independent of all of them (a property test checks it). */
typedef struct {
    uint32_t log2_run;      /* force s (tiny inputs then span many runs)        */
    uint32_t grid_distribute;
    uint32_t grid_probe;
    uint32_t pair_bytes;    /* force 8-byte pairs                               */
    uint32_t hist_mode;     /* 0 auto, 1 force shared-memory, 2 force global,
                               3 force radix passes (path 2, no payload)       */
    uint32_t path;          /* 0 auto, 1 force fused kernel, 2 force multi-kernel,
                               3 force the L2-run kernel (any source size),
                               4 two L2 runs (rec % 4 == 0, 8..116 bytes),
                               5 K L2 runs (log2_run, if set, fixes the run
                                 length)                                        */
    uint32_t gather;        /* 0 auto, 1 force direct-to-dst, 2 force INTERNAL  */
    uint32_t cluster;       /* path 6: CTAs holding one run together (1, 2, 4,
                               8; 0 = automatic)                                */
} dpg_options_t;

/* Build the plan the library would use (host only; sm_count <= 0 queries the
 * current device, or uses 148 when no device is present). */
dpg_status_t dpg_plan(size_t rec_bytes, uint64_t n_src, uint64_t n_out,
                      size_t pay_bytes, const dpg_options_t *opt, int sm_count,
                      dpg_plan_t *plan);

/* DPG record retrieval: dst[i] = src[rids[i]] for i in [0, n_out) (P:196-201,
 * Fig. 1).  src: n_src records of rec_bytes; rids: n_out uint32 in
 * [0, n_src); dst: n_out records, must not overlap src or rids. */
dpg_status_t dpg_retrieve(const void *src, size_t rec_bytes, uint64_t n_src,
                          const uint32_t *rids, uint64_t n_out, void *dst,
                          dpg_stream_t stream);

/* dpg_retrieve with overrides (opt may be NULL). */
dpg_status_t dpg_retrieve_ex(const void *src, size_t rec_bytes, uint64_t n_src,
                             const uint32_t *rids, uint64_t n_out, void *dst,
                             dpg_stream_t stream, const dpg_options_t *opt);

/* The standard approach the paper compares against: access
 * src[rids[i]] directly, one random access per record.  Same arguments and
 * result as dpg_retrieve; one kernel.  The measured comparison. */
dpg_status_t dpg_retrieve_direct(const void *src, size_t rec_bytes, uint64_t n_src,
                                 const uint32_t *rids, uint64_t n_out, void *dst,
                                 dpg_stream_t stream);

/* dpg_retrieve_direct with L2 eviction hints: hint 0 plain, 1 loads and
 * stores evict_first, 2 loads evict_last + stores evict_first (source staged
 * in L2 beforehand, e.g. by dpg_l2_prefetch); hint 3 the same direct
 * retrieval on the L2-run kernel's gather (16-byte window loads realigned in
 * shared memory, coalesced 16-byte output stores; path 3 without staging). */
dpg_status_t dpg_retrieve_direct_ex(const void *src, size_t rec_bytes, uint64_t n_src,
                                    const uint32_t *rids, uint64_t n_out, void *dst,
                                    dpg_stream_t stream, int hint);

/* Stage [ptr, ptr+bytes) into L2 with evict_last priority (bulk L2
 * prefetches; asynchronous, no completion signal). */
dpg_status_t dpg_l2_prefetch(const void *ptr, uint64_t bytes, dpg_stream_t stream);

/* DPG-Move foreign-key join (section 4.2.1).  The fact
 * relation R is scanned in file order, so its join triples (k, rid_R, rid_F)
 * come in rid_R order; the foreign key names the dimension record
 * directly (dense key), so rid_F = fk_col[i].  The records of F (dim) are
 * moved into R's order by DPG and joined with R ("join the temporary file
 * with the remaining relation"):
 *     out row i = fact[i] (fact_bytes) ++ dim[fk_col[i]] (rec_bytes)
 * out: n_fact rows of fact_bytes + rec_bytes, in fact order.  An fk_col entry
 * >= n_dim is a referential-integrity error (row left unwritten). */
dpg_status_t dpg_fk_join(const void *fact, size_t fact_bytes, uint64_t n_fact,
                         const uint32_t *fk_col, const void *dim, size_t rec_bytes,
                         uint64_t n_dim, void *out, dpg_stream_t stream);

/* The standard join the paper compares against, the measured
 * comparison for dpg_fk_join: the same rows, each built with one random
 * access to dim[fk_col[i]].  Same arguments and errors as dpg_fk_join. */
dpg_status_t dpg_fk_join_direct(const void *fact, size_t fact_bytes, uint64_t n_fact,
                                const uint32_t *fk_col, const void *dim, size_t rec_bytes,
                                uint64_t n_dim, void *out, dpg_stream_t stream);

dpg_status_t dpg_fk_join_ex(const void *fact, size_t fact_bytes, uint64_t n_fact,
                            const uint32_t *fk_col, const void *dim, size_t rec_bytes,
                            uint64_t n_dim, void *out, dpg_stream_t stream,
                            const dpg_options_t *opt);

/* Phase I alone (Distribute, Fig. 1), for tests: the
 * rids are distributed into runs r >> log2_run.  pairs_out[j] (uint64) =
 * local | (pos << 32) where local = rid - run*L and pos = the rid's position
 * in `rids`; the entries of run b occupy [run_start[b], run_start[b+1]).
 * Within a run the order of entries is unspecified (the GPU distributes in
 * parallel); the set of entries of each run is unique.  run_start_out has
 * num_runs + 1 uint64 entries. */
dpg_status_t dpg_distribute(const uint32_t *rids, uint64_t n_out, uint64_t n_src,
                            uint32_t log2_run, uint64_t *pairs_out,
                            uint64_t *run_start_out, dpg_stream_t stream,
                            const dpg_options_t *opt);

/* ---- Data skew: runs from a sorted sample of the rids (section 2.3) ----
 * "If there is a great deal of data skew ... the N/L partitions of the input
 * sequence of rids must be chosen on some other basis than the high order
 * bits ... sample the rids from the rid sequence.  The sampled set of rids is
 * then sorted, and partitions of the rids are chosen so as to evenly
 * partition the sampled set" (reading A23).
 *
 * dpg_skew_partition: draws sample_size rids of rids[n_out] (device) at
 * uniform positions (with replacement; the SplitMix64 sequence started at
 * `seed`, so the result is a function of its arguments), sorts them, and
 * takes the cut candidates sample[i * sample_size / num_runs], i = 1 ..
 * num_runs - 1; a candidate is kept when it is below n_src and above the last
 * kept cut (at first: above the smallest sampled rid), so ties collapse.
 * bounds_out (HOST, room for num_runs + 1 uint32) receives 0, the cuts, n_src
 * -- strictly ascending; *n_runs_out (host) the number of runs (<= num_runs;
 * every run holds at least one sampled rid).  A sampled rid >= n_src counts as
 * n_src.  Synchronous (one stream synchronisation).  Errors: n_out == 0,
 * num_runs == 0 or sample_size < num_runs -> DPG_ERR_INVALID_ARG;
 * sample_size > 32768 or n_src >= 2^32 -> DPG_ERR_UNSUPPORTED. */
dpg_status_t dpg_skew_partition(const uint32_t *rids, uint64_t n_out, uint64_t n_src,
                                uint32_t num_runs, uint32_t sample_size, uint64_t seed,
                                uint32_t *bounds_out, uint32_t *n_runs_out,
                                dpg_stream_t stream);

/* dpg_retrieve with the runs given by boundaries: run k holds the rids in
 * [bounds[k], bounds[k+1]) (bounds: HOST, n_runs + 1 uint32, bounds[0] = 0,
 * bounds[n_runs] = n_src < 2^32, non-decreasing -- else DPG_ERR_INVALID_ARG).
 * Runs wider than a shared-memory stage are split at the multiples of the
 * plan's L = 2^s (constraint (1)); the multi-kernel plan (path 2)
 * runs them.  Result, device buffers and error rules as dpg_retrieve; records
 * too large for a shared-memory stage -> DPG_ERR_UNSUPPORTED.  The layout is
 * uploaded with a pageable copy (the call may wait for the stream). */
dpg_status_t dpg_retrieve_bounds(const void *src, size_t rec_bytes, uint64_t n_src,
                                 const uint32_t *rids, uint64_t n_out, const uint32_t *bounds,
                                 uint64_t n_runs, void *dst, dpg_stream_t stream);

/* Phase I alone over boundary runs (tests): the runs are the caller's bounds
 * (HOST, as dpg_retrieve_bounds) merged with the multiples of L = 2^log2_run,
 * a caller bound equal to a multiple of L leaving an empty run before it;
 * *num_runs_out (host) receives their number K = n_runs + ceil(n_src / L) - 1.
 * pairs_out[n_out] (device) = (rid - start of its run) | (pos << 32), the
 * entries of run b in [run_start_out[b], run_start_out[b+1]) (device, K + 1
 * uint64), unordered within a run as dpg_distribute.  run_start_out == NULL:
 * only *num_runs_out is set. */
dpg_status_t dpg_distribute_bounds(const uint32_t *rids, uint64_t n_out, uint64_t n_src,
                                   const uint32_t *bounds, uint64_t n_runs, uint32_t log2_run,
                                   uint64_t *pairs_out, uint64_t *run_start_out,
                                   uint64_t *num_runs_out, dpg_stream_t stream);

/* Multi-GPU Phase I by owner: rids (uint32 or uint64,
 * rid_bytes = 4 or 8, device) are distributed to owners r >> log2_span
 * (parts owners, each owning 2^log2_span consecutive source records of the
 * n_src_total).  Outputs (device): local_out[j] = rid - owner * 2^log2_span
 * and pos_out[j] = the rid's position, grouped by owner (owner 0 first; order
 * inside an owner unspecified); counts_out[parts] (uint64) = requests per
 * owner.  Invalid rids (>= n_src_total) are reported as in dpg_retrieve and
 * dropped.  Requires n_src_total <= parts << log2_span. */
dpg_status_t dpg_partition(const void *rids, uint32_t rid_bytes, uint64_t n, uint64_t n_src_total,
                           uint32_t log2_span, uint32_t parts, uint32_t *local_out,
                           uint32_t *pos_out, uint64_t *counts_out, dpg_stream_t stream);

/* Multi-GPU Phase I with Phase III's map: rids
 * (uint32 or uint64 by rid_bytes, n of them, device) are grouped by owner =
 * rid >> log2_span (parts owners, <= 512); local_out[m] (device, n entries)
 * receives the owner-local offsets (rid - owner << log2_span), owner by
 * owner, each row's in output order within its CTA block; inv_out[i]
 * (device, n) the position of row i's request in local_out (0xFFFFFFFF for a
 * rid >= n_src_total, which is also reported to dpg_sync_status);
 * counts_out[parts] (device, uint64) the requests per owner.  Asynchronous. */
dpg_status_t dpg_partition_inv(const void *rids, uint32_t rid_bytes, uint64_t n,
                               uint64_t n_src_total, uint32_t log2_span, uint32_t parts,
                               uint32_t *local_out, uint32_t *inv_out, uint64_t *counts_out,
                               dpg_stream_t stream);

/* Phase III over the replies: dst[i] = rows[inv[i]] for inv[i] < n_rows (rows
 * of rec_bytes, device; dst n rows, device; other rows left unwritten).
 * Output rows written in order (sequential stores).  Asynchronous. */
dpg_status_t dpg_gather_rows(const void *rows, size_t rec_bytes, uint64_t n_rows,
                             const uint32_t *inv, uint64_t n, void *dst, dpg_stream_t stream);

/* Owner-side helper of the multi-GPU path: dst[pos[k]] = rows[k] for k in
 * [0, n) (Phase III against received replies).  pos must be distinct. */
dpg_status_t dpg_scatter_rows(const void *rows, size_t rec_bytes, const uint32_t *pos,
                              uint64_t n, void *dst, uint64_t n_dst, dpg_stream_t stream);

/* End-to-end entry with HOST buffers: copies src and rids host->device,
 * runs dpg_retrieve, copies dst device->host and synchronises `stream`.
 * Host buffers should be pinned for full PCIe bandwidth.  Device buffers are
 * library-owned and cached across calls, per (device, stream), for the 8 most
 * recently used streams (an older entry is freed after a device
 * synchronisation; dpg_release_cache frees them all).  dpg_release_cache also frees the
 * per-stream workspaces and trims the library's memory pool (it synchronises
 * every device). */
dpg_status_t dpg_retrieve_host(const void *src_host, size_t rec_bytes, uint64_t n_src,
                               const uint32_t *rids_host, uint64_t n_out, void *dst_host,
                               dpg_stream_t stream);

/* dpg_retrieve_host without the final synchronisation: the copies and the
 * retrieval are enqueued on `stream` and dst_host is complete once the stream
 * reaches the call (the caller synchronises).  Host buffers must be pinned
 * and stay valid until then.  Calls on different streams use different
 * device buffers, so a caller alternating two streams overlaps one call's
 * device->host copy with the next call's host->device copy (PCIe is full
 * duplex). */
dpg_status_t dpg_retrieve_host_async(const void *src_host, size_t rec_bytes, uint64_t n_src,
                                     const uint32_t *rids_host, uint64_t n_out, void *dst_host,
                                     dpg_stream_t stream);
void dpg_release_cache(void);

/* Batch lookup of keys in a hash index (section 4).  The index
 * (device, built by the caller): `table` = 2^m_log2 primary slots and `pool`
 * = overflow entries, each 16 bytes {uint32 key, uint32 rid, uint32 next,
 * uint32 0}; key k is in slot h(k) = (k * 0x9E3779B1 mod 2^32) >> (32 -
 * m_log2) or in the chain of pool entries linked from that slot by `next`
 * (0xFFFFFFFF ends a chain); rid 0xFFFFFFFF marks an empty slot (whose next
 * is 0xFFFFFFFF).  Keys in the index are distinct.  out[i] (device, n) =
 * the rid of keys[i] (device, n), 0xFFFFFFFF when absent.  m_log2 in
 * [1, 31].
 * dpg_hash_lookup: DPG -- the keys distributed into runs by
 * partition of the hash array (partitions of at most the L2 run budget, or
 * 2^log2_run slots when log2_run > 0; at most 512), each partition staged
 * into the L2 and probed by its run's keys, the rids gathered back into query
 * order.  dpg_hash_lookup_direct: one random slot read per key.
 * Asynchronous; workspace library-owned. */
dpg_status_t dpg_hash_lookup(const void *table, uint32_t m_log2, const void *pool,
                             const uint32_t *keys, uint64_t n, uint32_t *out,
                             dpg_stream_t stream, uint32_t log2_run);
dpg_status_t dpg_hash_lookup_direct(const void *table, uint32_t m_log2, const void *pool,
                                    const uint32_t *keys, uint64_t n, uint32_t *out,
                                    dpg_stream_t stream);

/* Batch lookup of keys in an enhanced B+-tree (section 4).  The
 * index (device, built by the caller): levels[0] = the N indexed keys sorted
 * ascending (distinct), rids[j] (device) the rid of levels[0][j]; levels[t]
 * = every 16th entry of levels[t-1] (level_n[t] = ceil(level_n[t-1] / 16)),
 * up to a top level of <= 16 entries; n_levels <= 10; each level 64-byte
 * aligned and readable up to a multiple of 16 entries (host arrays `levels`
 * of device pointers and `level_n` of counts).  out[i] (device, n) = the
 * rid of keys[i] (device, n), 0xFFFFFFFF when absent.
 * dpg_btree_lookup: the two-pass DPG lookup -- the top of the
 * tree places every key in a run of consecutive subtrees (runs of 2^s
 * level-0 entries within the L2 run budget, or 2^log2_run when > 0; at most
 * 512 runs), each run's lower levels are staged into the L2 and its keys
 * complete their descent there, the rids gathered back into query order.
 * dpg_btree_lookup_direct: one full descent per key.  Asynchronous. */
dpg_status_t dpg_btree_lookup(const uint32_t *const *levels, const uint64_t *level_n,
                              uint32_t n_levels, const uint32_t *rids, const uint32_t *keys,
                              uint64_t n, uint32_t *out, dpg_stream_t stream, uint32_t log2_run);
dpg_status_t dpg_btree_lookup_direct(const uint32_t *const *levels, const uint64_t *level_n,
                                     uint32_t n_levels, const uint32_t *rids, const uint32_t *keys,
                                     uint64_t n, uint32_t *out, dpg_stream_t stream);

/* Multi-GPU retrieval (north_star config 5; not in the paper: reading A14,
 * DESIGN.md section 8).  One process per GPU.  dpg_get_unique_id: an NCCL
 * unique id (128 bytes) made on one rank and sent to the others by the
 * caller.  dpg_comm_create: the communicator of `nranks` (<= 8) processes on
 * the current device (blocking until all ranks join); dpg_comm_destroy frees
 * it and its receive windows.  dpg_retrieve_dist: the global retrieval
 * D[i] = R[rids[i]] over a source of n_src_total records range-partitioned
 * by rank (rank r owns records [r*S, (r+1)*S), S = the smallest power of two
 * with nranks * S >= n_src_total; src_shard holds this rank's records, device)
 * and an output block-partitioned by the caller: this rank passes the rids
 * (uint64, device) of its n_out_local output rows and receives their records
 * in dst (device, n_out_local * rec_bytes).  Collective: every rank calls it
 * (with its own block; 0 rows allowed).  Steps: owner partition, one NCCL
 * all-gather of the count matrix, grouped send/recv of the requests, the
 * owner's DPG writing each requester's rows straight into that requester's
 * receive window (CUDA IPC, NVLink), a stream-ordered all-reduce, Phase III
 * from the window.  NCCL is loaded at run time (DPG_ERR_NCCL if absent or on
 * an NCCL failure).  Invalid rids as dpg_retrieve.  Synchronises `stream`
 * (the counts size the exchange).  Failure handling: before each collective
 * the ranks agree on their local status (an all-reduce), so a rank that fails
 * locally (allocation, IPC mapping, a launch) makes every rank return the
 * error together; while waiting for the stream a rank polls NCCL's
 * asynchronous error state and aborts the communicator on an error or after
 * DPG_NCCL_TIMEOUT_S seconds (default 600) -- an aborted communicator then
 * returns DPG_ERR_NCCL on every call and must be destroyed. */
dpg_status_t dpg_get_unique_id(uint8_t id[128]);
dpg_status_t dpg_comm_create(const uint8_t id[128], int nranks, int rank, void **comm);
dpg_status_t dpg_retrieve_dist(void *comm, const void *src_shard, size_t rec_bytes,
                               uint64_t n_src_total, const uint64_t *rids, uint64_t n_out_local,
                               void *dst, dpg_stream_t stream);
dpg_status_t dpg_comm_destroy(void *comm);

/* The same global retrieval for P (<= 8) VIRTUAL ranks in one process on the
 * current GPU (testing and single-GPU measurement of the exchange): rank r's
 * source shard src_shards[r] (device; records [r*S, (r+1)*S) of the global
 * source, S as for dpg_retrieve_dist), its rids rids[r] (uint64, device,
 * n_out[r] of them) and its output dst[r] (device).  Host arrays of P
 * entries.  Every step is dpg_retrieve_dist's -- owner partition, the count
 * matrix, the owner-side offsets of the requests and of each requester's
 * window rows (the same code), the owner's segmented DPG writing into the
 * requesters' windows, Phase III from the window -- with NCCL replaced by a
 * host read of the counts and one device-to-device copy per (requester,
 * owner) pair.  Synchronises `stream` once.  Errors as dpg_retrieve_dist
 * (no DPG_ERR_NCCL: no NCCL is used). */
dpg_status_t dpg_retrieve_dist_loopback(int P, const void *const *src_shards, size_t rec_bytes,
                                        uint64_t n_src_total, const uint64_t *const *rids,
                                        const uint64_t *n_out, void *const *dst,
                                        dpg_stream_t stream);

/* The exchange's arithmetic (host only, no CUDA): for the P x (P + 1) count
 * matrix C (host, row-major; C[q][o] = rows of rank q whose rids rank o owns,
 * o < P; C[q][P] = rank q's rows), rank `me`'s plan -- roff[P+1]: where the
 * requests from each requester q start in me's receive buffer (requester
 * order); soff[P+1]: where me's requests to each owner start in its own
 * request list (owner order); win_row[P]: the row of requester q's window at
 * which me's replies to q start (q's window holds the replies owner by
 * owner); *n_req: the requests me receives; *cap: the largest rank's rows
 * (each window's capacity).  dpg_retrieve_dist and
 * dpg_retrieve_dist_loopback compute exactly this.  P in [1, 64], 0 <= me < P,
 * else DPG_ERR_INVALID_ARG. */
dpg_status_t dpg_exchange_plan(const uint64_t *counts, int P, int me, uint64_t *roff,
                               uint64_t *soff, uint64_t *win_row, uint64_t *n_req,
                               uint64_t *cap);

/* Receive windows for the fused multi-GPU exchange (one process per GPU on
 * one node).  dpg_ipc_alloc: a device buffer of `bytes` on the current device
 * (library-owned until dpg_ipc_free) and its 64-byte CUDA IPC handle, to be
 * sent to the peer processes.  dpg_ipc_open: maps a peer's buffer from its
 * handle into this process (peer access over NVLink enabled lazily); the
 * pointer is valid for kernels on this device until dpg_ipc_close.  A
 * process cannot open its own handle.  Errors: DPG_ERR_INVALID_ARG (NULL
 * arguments, zero bytes), DPG_ERR_OOM, DPG_ERR_CUDA (the driver's
 * refusal, e.g. no peer access).  Synchronous. */
dpg_status_t dpg_ipc_alloc(size_t bytes, void **ptr, uint8_t handle[64]);
dpg_status_t dpg_ipc_open(const uint8_t handle[64], void **ptr);
dpg_status_t dpg_ipc_close(void *ptr);
dpg_status_t dpg_ipc_free(void *ptr);

/* Retrieval into output segments: D[k] = R[rids[k]] as dpg_retrieve, with
 * output row k of segment q (rows seg_rows[0] + ... + seg_rows[q-1] up to the
 * next boundary) written to seg_dst[q] + (k - first row of q) * rec_bytes.
 * nseg in [1, 8]; seg_rows and seg_dst are HOST arrays of nseg entries (the
 * row counts must sum to n_out); each seg_dst[q] is a device pointer, and it
 * may be a peer GPU's memory mapped into this process (dpg_ipc_open): the
 * multi-GPU exchange uses this to write an owner's replies straight into each
 * requester's receive window over NVLink, with no reply buffer and no
 * separate collective for the records (north_star config 5; SV 8(f) #1).
 * The plan is dpg_retrieve's: shared-memory runs (both kernels) write each
 * staged record to its segment row; the L2 run and the K-run L2 plan's last
 * gather do the same per 32-row group (4-byte-multiple records of 8..116
 * bytes); a plan that cannot (another record in an L2 run) is replaced by
 * the shared-memory runs; only a record no plan takes falls back to one
 * direct gather per segment.  Errors as dpg_retrieve
 * (DPG_ERR_INVALID_ARG also for counts that do not sum to n_out, a NULL
 * segment with rows, or a segment overlapping src or rids).  Asynchronous. */
dpg_status_t dpg_retrieve_segments(const void *src, size_t rec_bytes, uint64_t n_src,
                                   const uint32_t *rids, uint64_t n_out, uint32_t nseg,
                                   const uint64_t *seg_rows, void *const *seg_dst,
                                   dpg_stream_t stream);

/* DPG-Sort join: the join pairs (rid_R = i, rid_F =
 * fk_col[i]) sorted by rid_F (stable), the fact rows (R) moved into a
 * temporary file in that order by DPG retrieval, then joined with dim (F)
 * read in rid_F order.  out (device, n_fact rows of fact_bytes + rec_bytes):
 * row j = fact[rid_R_j] ++ dim[rid_F_j], pairs in stable fk order -- the same
 * rows as dpg_fk_join, in fk order instead of fact order.  Only the key bytes
 * an fk below n_dim can have are sorted ("the lowest log N bits"),
 * so an fk >= n_dim is reported at its fact position (dpg_sync_status) and
 * leaves the content of out unspecified (reading A19).  Same argument rules
 * as dpg_fk_join.  Asynchronous. */
dpg_status_t dpg_fk_join_sort(const void *fact, size_t fact_bytes, uint64_t n_fact,
                              const uint32_t *fk_col, const void *dim, size_t rec_bytes,
                              uint64_t n_dim, void *out, dpg_stream_t stream);

/* Three-phase key-pointer sorting with DPG as the record-copy phase
 * (section 3; DPG sort).  Keys: key_bytes
 * (1..12) unsigned bytes at key_off inside each record, compared
 * lexicographically (the Datamation key: 10 bytes at offset 0);
 * the sort is stable (equal keys keep ascending rid, reading A10).
 * dpg_sort_rids: phases 1-2 only -- rids_out[n] (device) receives the rids in
 *   sorted order (key extraction + a stable LSD radix sort, one key byte per
 *   pass).  rids_out must not overlap src.
 * dpg_sort: phases 1-3 -- dst[n*rec] (device, not overlapping src) receives
 *   the records in sorted order (phase 3 = dpg_retrieve).
 * Errors: DPG_ERR_INVALID_ARG for a bad key range, NULL pointers with n > 0
 * or overlap; DPG_ERR_UNSUPPORTED for n >= 2^32.  Asynchronous on `stream`. */
dpg_status_t dpg_sort_rids(const void *src, size_t rec_bytes, uint64_t n, size_t key_off,
                           size_t key_bytes, uint32_t *rids_out, dpg_stream_t stream);
dpg_status_t dpg_sort(const void *src, size_t rec_bytes, uint64_t n, size_t key_off,
                      size_t key_bytes, void *dst, dpg_stream_t stream);

/* Synchronise `stream`, then report and clear the device status word:
 * DPG_ERR_RID_RANGE with *first_bad_index = smallest offending position
 * recorded since the last call, or DPG_OK.  The status word is per device,
 * shared by all streams. */
dpg_status_t dpg_sync_status(dpg_stream_t stream, uint64_t *first_bad_index);

const char *dpg_status_string(dpg_status_t status);

/* Number of kernel launches the most recent call on this host thread enqueued. */
uint32_t dpg_last_launch_count(void);

/* Plan path (dpg_plan_t.path) the most recent dpg_retrieve / dpg_fk_join on
 * this host thread ran.  With the automatic plan, an input of >= 4 Mi rids
 * planned on shared-memory runs (path 1) is first sampled for data skew
 * (section 2.3: 65,536 rids at evenly spaced positions, counted
 * per group of runs; one stream synchronisation); when the estimated rids
 * beyond the runs' fixed capacity exceed 2% of the input, the call runs the
 * multi-kernel plan (path 2) instead, whose run sizes are exact and whose
 * heavy runs are split into work items over all SMs.  (Not while the stream
 * is being captured into a CUDA graph: no sampling then.) */
uint32_t dpg_last_path(void);

/* Phase timing (bench.py's roofline): while enabled, every dpg_retrieve /
 * dpg_fk_join call records CUDA events on its own stream around Phase I
 * (distribute) and the fused probe-gather kernel.  dpg_phase_times
 * synchronises those events, returns the summed milliseconds and the number
 * of calls since the last read, and clears the record. */
void dpg_phase_timing(int enable);

/* Profiling only: when device_buf (>= grid*16 uint64) is non-NULL, the fused
 * kernel writes per-CTA %globaltimer stamps at its phase boundaries (start,
 * Phase I count done, barrier 1, scatter done, barrier 2, end).  NULL turns
 * it off. */
void dpg_debug_phase_stamps(void *device_buf);

/* Tuning experiments only (tools/): code-generation and launch variants (store
 * cache policies, reservation order, ring geometry, bit 18: plain launches
 * instead of programmatic dependent launch between a plan's kernels) and, for
 * timing experiments, bits that skip work and so change the result (bits 20
 * and 21 of the window gather).  0 is the default and what every other caller
 * gets. */
void dpg_debug_flags(uint32_t flags);
dpg_status_t dpg_phase_times(double *distribute_ms, double *probe_gather_ms, uint32_t *calls);
/* Same record split by phase: Phase I (distribute), Phase II (probe) and
 * Phase III (gather) of the three-kernel plan (path 6) are timed separately;
 * for the other plans *phase2_ms covers the probe-gather kernel(s) and
 * *phase3_ms is 0. */
dpg_status_t dpg_phase_times_ex(double *phase1_ms, double *phase2_ms, double *phase3_ms,
                                uint32_t *calls);

int dpg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DPG_H */
