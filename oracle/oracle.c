/*
 * oracle/oracle.c -- CPU ORACLE for DPG record retrieval (arXiv cs/0308004).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load, call or execute
 * anything under oracle/.  The product path (paper_cs_0308004_b200/) never
 * does, and shares no code, header, table or helper with this file.
 *
 * Everything here is plain, slow, single-threaded C with no blocking, fusion
 * or reordering beyond what the cited passage states.  Citations:
 *   P:n  = /root/reference/PAPER.md line n (LaTeX body of the paper)
 *   S:n  = /root/reference/SPEC.md line n   (interfaces / test ideas only)
 *
 * Pins (tests/test_oracle.py, run with -m "not gpu"): the Fig. 2 worked
 * example (golden fixture tests/golden/fig2_example.txt),
 * brute force over all permutations n<=6 via an independent inverse-scatter
 * formulation, all rid sequences of length <= 4 over n <= 3 against numpy
 * fancy indexing, identity / multiset / sorted-key invariants, the join's
 * nested-loop cross-check; the 64-bit-rid entries against numpy indexing, the
 * 32-bit entries and a no-truncation check (rids >= 2^32); the skew
 * partition (tests/test_oracle_skew.py) against SplitMix64's published
 * sequence, S:166-169's statistical examples and exhaustive tiny cases, and
 * the boundary-mode Fig. 1 against (2) on multiples of L and the Fig. 2
 * example.  No function here is "parity unpinned".
 *
 * Return convention (reading A6 of DESIGN.md): 0 on success; -1 on an invalid
 * argument; 1 if some rid >= n_src, in which case *bad_index receives the
 * SMALLEST offending position i and dst row i is left unwritten (every other
 * row is still written).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ *
 * (1) The record-retrieval problem, by definition:             *
 *         for each i,  D[i] = R[S_rid[i]]                                   *
 *     with records of rec bytes laid out back to back and rids    *
 *     dense, 0-based, in [0, n_src) (reading A2).                *
 * ------------------------------------------------------------------------ */
int oracle_retrieve(const uint8_t *src, uint64_t rec, uint64_t n_src,
                    const uint32_t *rids, uint64_t n_out, uint8_t *dst,
                    uint64_t *bad_index)
{
    int status = 0;
    if (rec == 0) return -1;
    for (uint64_t i = 0; i < n_out; ++i) {
        uint64_t r = rids[i];
        if (r >= n_src) {
            if (status == 0) { status = 1; if (bad_index) *bad_index = i; }
            continue;
        }
        memcpy(dst + i * rec, src + r * rec, rec);
    }
    return status;
}

/* Same definition with 64-bit rids (the multi-GPU configuration uses them). */
int oracle_retrieve_u64(const uint8_t *src, uint64_t rec, uint64_t n_src,
                        const uint64_t *rids, uint64_t n_out, uint8_t *dst,
                        uint64_t *bad_index)
{
    int status = 0;
    if (rec == 0) return -1;
    for (uint64_t i = 0; i < n_out; ++i) {
        uint64_t r = rids[i];
        if (r >= n_src) {
            if (status == 0) { status = 1; if (bad_index) *bad_index = i; }
            continue;
        }
        memcpy(dst + i * rec, src + r * rec, rec);
    }
    return status;
}

/* The same loop split into `nthreads` contiguous index ranges, each run by
 * oracle_retrieve on its own thread (the CPU baseline's all-cores timing,
 * BASELINE.md): no arithmetic of its own.  Return and bad_index as
 * oracle_retrieve (the smallest offending position over all ranges). */
struct oracle_range {
    const uint8_t *src; uint64_t rec, n_src; const uint32_t *rids; uint64_t n; uint8_t *dst;
    uint64_t bad; int status;
};
static void *oracle_range_run(void *p)
{
    struct oracle_range *a = p;
    a->status = oracle_retrieve(a->src, a->rec, a->n_src, a->rids, a->n, a->dst, &a->bad);
    return NULL;
}
int oracle_retrieve_threads(const uint8_t *src, uint64_t rec, uint64_t n_src,
                            const uint32_t *rids, uint64_t n_out, uint8_t *dst,
                            uint64_t *bad_index, int nthreads)
{
    if (rec == 0 || nthreads < 1 || nthreads > 1024) return -1;
    struct oracle_range *r = calloc((size_t)nthreads, sizeof(*r));
    pthread_t *th = calloc((size_t)nthreads, sizeof(*th));
    if (!r || !th) { free(r); free(th); return -1; }
    for (int t = 0; t < nthreads; ++t) {
        uint64_t lo = n_out * (uint64_t)t / (uint64_t)nthreads;
        uint64_t hi = n_out * (uint64_t)(t + 1) / (uint64_t)nthreads;
        r[t] = (struct oracle_range){src, rec, n_src, rids + lo, hi - lo, dst + lo * rec, 0, 0};
        if (pthread_create(&th[t], NULL, oracle_range_run, &r[t]) != 0) { r[t].status = -2; }
    }
    int status = 0;
    for (int t = 0; t < nthreads; ++t) {
        if (r[t].status != -2) pthread_join(th[t], NULL);
        uint64_t lo = n_out * (uint64_t)t / (uint64_t)nthreads;
        if (r[t].status == -2 || r[t].status == -1) { status = -1; continue; }
        if (r[t].status == 1 && status == 0) { status = 1; if (bad_index) *bad_index = lo + r[t].bad; }
    }
    free(r); free(th);
    return status;
}

/* ------------------------------------------------------------------------ *
 * (2) The DPG algorithm exactly as Fig. 1 writes it, in the     *
 *     paper's order and notation, with INTERNAL (RECORD_RUN) materialised.  *
 *     Used to pin the intermediates of the method (RID runs, INTERNAL runs) *
 *     and to show that the three phases reach the definition (1).           *
 *                                                                          *
 *     L      run length in records.  Fig. 1 sets L from the     *
 *            cache size; here it is a parameter (reading A3).      *
 *     run of rid r = floor(r / L) (0-based; Fig. 1 writes ceil(r/L) with    *
 *            1-based runs, reading A1).                             *
 *                                                                          *
 *   Optional outputs (any may be NULL):                                     *
 *     run_start[NUM_RUNS+1]  offsets of each RID run inside rid_runs        *
 *     rid_runs[n_out]        RID_RUN[0] ++ RID_RUN[1] ++ ...       *
 *     rid_pos[n_out]         for each entry of rid_runs, the position i in  *
 *                            RID it came from (the "i-th step" of P:313)    *
 *     record_runs[n_out*rec] RECORD_RUN[0] ++ ... = INTERNAL        *
 *   Sizes: NUM_RUNS = ceil(n_src / L).  INTERNAL holds n_out records        *
 *   (reading A4: "same size as the data file" only for permutations).      *
 * ------------------------------------------------------------------------ */
int oracle_dpg_fig1(const uint8_t *src, uint64_t rec, uint64_t n_src,
                    const uint32_t *rids, uint64_t n_out, uint64_t L,
                    uint8_t *dst, uint64_t *run_start_out,
                    uint32_t *rid_runs_out, uint64_t *rid_pos_out,
                    uint8_t *record_runs_out, uint64_t *bad_index)
{
    if (rec == 0 || L == 0) return -1;
    /* Range check first (reading A6): the paper assumes valid rids. */
    for (uint64_t i = 0; i < n_out; ++i) {
        if ((uint64_t)rids[i] >= n_src) { if (bad_index) *bad_index = i; return 1; }
    }
    uint64_t num_runs = (n_src + L - 1) / L;          /* NUM_RUNS <- N/L */
    uint64_t *run_len = calloc(num_runs + 1, sizeof(uint64_t));
    uint64_t *run_start = calloc(num_runs + 1, sizeof(uint64_t));
    uint64_t *cursor = calloc(num_runs + 1, sizeof(uint64_t));
    uint32_t *RID_RUN = malloc((n_out ? n_out : 1) * sizeof(uint32_t));
    uint64_t *RID_POS = malloc((n_out ? n_out : 1) * sizeof(uint64_t));
    uint8_t *RECORD_RUN = malloc((n_out ? n_out : 1) * rec);
    if (!run_len || !run_start || !cursor || !RID_RUN || !RID_POS || !RECORD_RUN) {
        free(run_len); free(run_start); free(cursor); free(RID_RUN); free(RID_POS); free(RECORD_RUN);
        return -1;
    }
    /* The runs are growable lists in Fig. 1 ("Append r to RID_RUN[run_num]");
     * they are stored back to back here, sized by a counting pass. */
    for (uint64_t i = 0; i < n_out; ++i) run_len[rids[i] / L] += 1;
    for (uint64_t b = 0; b < num_runs; ++b) run_start[b + 1] = run_start[b] + run_len[b];

    /* Phase I: Distribute RID array into runs. */
    for (uint64_t b = 0; b < num_runs; ++b) cursor[b] = run_start[b];
    for (uint64_t i = 0; i < n_out; ++i) {
        uint32_t r = rids[i];
        uint64_t run_num = r / L;                      /* run_num = ceil(r/L), 1-based */
        RID_RUN[cursor[run_num]] = r;                  /* Append r to RID_RUN[run_num] */
        RID_POS[cursor[run_num]] = i;
        cursor[run_num] += 1;
    }

    /* Phase II: Probe partitions of INPUT_REC.  Run i of INPUT is
     * records [(i-1)L+1, iL] in 1-based notation = [iL, (i+1)L) 0-based. */
    for (uint64_t i = 0; i < num_runs; ++i) {
        const uint8_t *input_run = src + i * L * rec;  /* "Read into memory all records" */
        uint64_t out = run_start[i];                   /* RECORD_RUN[i] */
        for (uint64_t j = run_start[i]; j < run_start[i + 1]; ++j) {
            uint32_t r = RID_RUN[j];                   /* For each rid r in RID_RUN[i] */
            memcpy(RECORD_RUN + out * rec,             /* Append INPUT_REC[r] to RECORD_RUN[i] */
                   input_run + (r - i * L) * rec, rec);
            out += 1;
        }
    }

    /* Phase III: Gather records from RECORD_RUN[] into OUTPUT_REC in the same
     * order as RID[]: read the NEXT record of run floor(r/L). */
    for (uint64_t b = 0; b < num_runs; ++b) cursor[b] = run_start[b];
    for (uint64_t i = 0; i < n_out; ++i) {
        uint32_t r = rids[i];
        uint64_t run_num = r / L;
        memcpy(dst + i * rec, RECORD_RUN + cursor[run_num] * rec, rec);
        cursor[run_num] += 1;
    }

    if (run_start_out) memcpy(run_start_out, run_start, (num_runs + 1) * sizeof(uint64_t));
    if (rid_runs_out) memcpy(rid_runs_out, RID_RUN, n_out * sizeof(uint32_t));
    if (rid_pos_out) memcpy(rid_pos_out, RID_POS, n_out * sizeof(uint64_t));
    if (record_runs_out) memcpy(record_runs_out, RECORD_RUN, n_out * rec);
    free(run_len); free(run_start); free(cursor); free(RID_RUN); free(RID_POS); free(RECORD_RUN);
    return 0;
}

/* ------------------------------------------------------------------------ *
 * (3) DPG-Move foreign-key join, with the join triple  *
 *     (k, rid_R, rid_F) of P:565-567.  The fact relation R is scanned in    *
 *     file order, so rid_R = i; the foreign key k names the     *
 *     dimension record directly (dense key, reading A11), so rid_F = fk[i]. *
 *     Output row i = R-part ++ F[rid_F] ("join the temporary file with the  *
 *     remaining relation"): fact payload (fact_bytes) followed   *
 *     by the dimension record (rec bytes), in fact order.                   *
 * ------------------------------------------------------------------------ */
int oracle_fk_join(const uint8_t *fact, uint64_t fact_bytes, uint64_t n_fact,
                   const uint32_t *fk, const uint8_t *dim, uint64_t rec,
                   uint64_t n_dim, uint8_t *out, uint64_t *bad_index)
{
    int status = 0;
    if (rec == 0) return -1;
    uint64_t row = fact_bytes + rec;
    for (uint64_t i = 0; i < n_fact; ++i) {
        uint64_t rid_F = fk[i];
        if (rid_F >= n_dim) {                          /* referential integrity */
            if (status == 0) { status = 1; if (bad_index) *bad_index = i; }
            continue;
        }
        memcpy(out + i * row, fact + i * fact_bytes, fact_bytes);
        memcpy(out + i * row + fact_bytes, dim + rid_F * rec, rec);
    }
    return status;
}

/* Sampled oracle: the definition evaluated at selected output positions only
 * (for parity at full sizes, where the whole output is large). out row j is
 * D[idx[j]]. */
int oracle_retrieve_at(const uint8_t *src, uint64_t rec, uint64_t n_src,
                       const uint32_t *rids, const uint64_t *idx, uint64_t n_idx,
                       uint8_t *out)
{
    for (uint64_t j = 0; j < n_idx; ++j) {
        uint64_t r = rids[idx[j]];
        if (r >= n_src) return 1;
        memcpy(out + j * rec, src + r * rec, rec);
    }
    return 0;
}

/* Same, 64-bit rids (the multi-GPU configuration's global rids). */
int oracle_retrieve_at_u64(const uint8_t *src, uint64_t rec, uint64_t n_src,
                           const uint64_t *rids, const uint64_t *idx, uint64_t n_idx,
                           uint8_t *out)
{
    for (uint64_t j = 0; j < n_idx; ++j) {
        uint64_t r = rids[idx[j]];
        if (r >= n_src) return 1;
        memcpy(out + j * rec, src + r * rec, rec);
    }
    return 0;
}

/* ------------------------------------------------------------------------ *
 * (4) Three-phase key-pointer sorting (section 3): "extract the  *
 *     key-pointer pairs, sort the pairs by key, then retrieve the records   *
 *     in the sorted order" -- the last step is record retrieval (1).        *
 *     Keys: key_bytes bytes at key_off inside each record, compared as      *
 *     unsigned bytes, lexicographically (the Datamation key;     *
 *     reading A10); the sort is stable, so equal keys keep ascending rids.  *
 *     Phase 2 here is a plain bottom-up merge sort of the rids (stable by   *
 *     construction).  out_rids[n] receives the sorted rid sequence.         *
 * ------------------------------------------------------------------------ */
static int key_less_eq(const uint8_t *src, uint64_t rec, uint64_t key_off, uint64_t key_bytes,
                       uint32_t a, uint32_t b)
{
    /* a's key <= b's key */
    return memcmp(src + (uint64_t)a * rec + key_off, src + (uint64_t)b * rec + key_off,
                  key_bytes) <= 0;
}

int oracle_sort_rids(const uint8_t *src, uint64_t rec, uint64_t n, uint64_t key_off,
                     uint64_t key_bytes, uint32_t *out_rids)
{
    if (rec == 0 || key_off + key_bytes > rec || n >= (1ull << 32)) return -1;
    uint32_t *a = malloc((n ? n : 1) * sizeof(uint32_t));
    uint32_t *b = malloc((n ? n : 1) * sizeof(uint32_t));
    if (!a || !b) { free(a); free(b); return -1; }
    /* Phase 1: the key-pointer pairs (the key stays in the record; the
     * pointer is the rid, i.e. the record's position). */
    for (uint64_t i = 0; i < n; ++i) a[i] = (uint32_t)i;
    /* Phase 2: stable merge sort of the pointers by key. */
    for (uint64_t w = 1; w < n; w *= 2) {
        for (uint64_t lo = 0; lo < n; lo += 2 * w) {
            uint64_t mid = lo + w < n ? lo + w : n;
            uint64_t hi = lo + 2 * w < n ? lo + 2 * w : n;
            uint64_t i = lo, j = mid, k = lo;
            while (i < mid && j < hi) {
                /* left element first when keys are equal: stability */
                if (key_less_eq(src, rec, key_off, key_bytes, a[i], a[j])) b[k++] = a[i++];
                else b[k++] = a[j++];
            }
            while (i < mid) b[k++] = a[i++];
            while (j < hi) b[k++] = a[j++];
        }
        uint32_t *t = a; a = b; b = t;
    }
    memcpy(out_rids, a, n * sizeof(uint32_t));
    free(a); free(b);
    return 0;
}

/* ------------------------------------------------------------------------ *
 * (5) DPG-Sort join: "sort the rid pairs (rid_R,      *
 *     rid_F) according to the order of rid_F", then "move the records of R *
 *     according to the ordering of rid_F in the sorted sequence"; joined   *
 *     with F read in rid_F order.  With the dense key of reading A11,       *
 *     rid_R = i and rid_F = fk[i].  Output row j = fact[rid_R_j] (fact      *
 *     bytes) ++ dim[rid_F_j] (rec bytes), the pairs in stable rid_F order   *
 *     (ties keep ascending rid_R).  Phase "sort" is a plain bottom-up merge *
 *     sort; an fk >= n_dim is an error at the smallest fact position.       *
 * ------------------------------------------------------------------------ */
int oracle_fk_join_sort(const uint8_t *fact, uint64_t fact_bytes, uint64_t n_fact,
                        const uint32_t *fk, const uint8_t *dim, uint64_t rec,
                        uint64_t n_dim, uint8_t *out, uint64_t *bad_index)
{
    if (rec == 0 || n_fact >= (1ull << 32)) return -1;
    for (uint64_t i = 0; i < n_fact; ++i)
        if (fk[i] >= n_dim) { if (bad_index) *bad_index = i; return 1; }
    uint32_t *a = malloc((n_fact ? n_fact : 1) * sizeof(uint32_t));
    uint32_t *b = malloc((n_fact ? n_fact : 1) * sizeof(uint32_t));
    if (!a || !b) { free(a); free(b); return -1; }
    for (uint64_t i = 0; i < n_fact; ++i) a[i] = (uint32_t)i;       /* the pairs (i, fk[i]) */
    for (uint64_t w = 1; w < n_fact; w *= 2) {                      /* stable sort by rid_F */
        for (uint64_t lo = 0; lo < n_fact; lo += 2 * w) {
            uint64_t mid = lo + w < n_fact ? lo + w : n_fact;
            uint64_t hi = lo + 2 * w < n_fact ? lo + 2 * w : n_fact;
            uint64_t i = lo, j = mid, k = lo;
            while (i < mid && j < hi) {
                if (fk[a[i]] <= fk[a[j]]) b[k++] = a[i++];
                else b[k++] = a[j++];
            }
            while (i < mid) b[k++] = a[i++];
            while (j < hi) b[k++] = a[j++];
        }
        uint32_t *t = a; a = b; b = t;
    }
    uint64_t row = fact_bytes + rec;
    for (uint64_t j = 0; j < n_fact; ++j) {                         /* move R, join with F */
        memcpy(out + j * row, fact + (uint64_t)a[j] * fact_bytes, fact_bytes);
        memcpy(out + j * row + fact_bytes, dim + (uint64_t)fk[a[j]] * rec, rec);
    }
    free(a); free(b);
    return 0;
}

/* ------------------------------------------------------------------------ *
 * Batch index lookup (section 4): for each query key q[i], the    *
 * rid of the indexed record with that key, or 0xFFFFFFFF when no record has *
 * it.  The index maps keys[j] -> rid j (distinct keys).  The plain          *
 * definition: the (key, rid) pairs sorted by key (library qsort), each       *
 * query found by binary search -- no hash index involved, so the result does *
 * not depend on any index layout.                                            *
 * ------------------------------------------------------------------------ */
static int cmp_pair(const void *a, const void *b)
{
    const uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return x < y ? -1 : x > y;
}

int oracle_batch_lookup(const uint32_t *keys, uint64_t n_keys, const uint32_t *q, uint64_t n_q,
                        uint32_t *out)
{
    if (n_keys >= (1ull << 32)) return -1;
    uint64_t *pairs = malloc((n_keys ? n_keys : 1) * sizeof(uint64_t));
    if (!pairs) return -1;
    for (uint64_t j = 0; j < n_keys; ++j) pairs[j] = ((uint64_t)keys[j] << 32) | j;
    qsort(pairs, n_keys, sizeof(uint64_t), cmp_pair);
    for (uint64_t i = 0; i < n_q; ++i) {
        uint64_t lo = 0, hi = n_keys;                /* first pair with key >= q[i] */
        while (lo < hi) {
            const uint64_t mid = lo + (hi - lo) / 2;
            if ((uint32_t)(pairs[mid] >> 32) < q[i]) lo = mid + 1; else hi = mid;
        }
        out[i] = (lo < n_keys && (uint32_t)(pairs[lo] >> 32) == q[i]) ? (uint32_t)pairs[lo]
                                                                       : 0xFFFFFFFFu;
    }
    free(pairs);
    return 0;
}

/* ------------------------------------------------------------------------ *
 * (8) Data skew (section 2.3): "sample the rids from the rid     *
 *     sequence.  The sampled set of rids is then sorted, and partitions of  *
 *     the rids are chosen so as to evenly partition the sampled set."       *
 *     The paper leaves the draw unspecified (reading A23): sample_size      *
 *     positions are drawn uniformly, with replacement, by the SplitMix64    *
 *     sequence started at `seed` (draw k = mix(seed + (k+1) * gamma), the   *
 *     position floor(draw * n_out / 2^64)).  A sampled rid >= n_src counts  *
 *     as n_src (it never becomes a cut).  The sorted sample s[0..S) gives   *
 *     the cut candidates s[floor(i * S / num_runs)], i = 1 .. num_runs-1    *
 *     (S:162-170); a candidate is kept when it is below n_src and larger   *
 *     than the last kept cut (at first: than the smallest sampled rid), so  *
 *     equal quantiles collapse, fewer runs may result, and every run holds  *
 *     at least one sampled rid.  bounds_out[0..n_runs] = 0, cuts..., n_src *
 *     (room for num_runs + 1 entries); run k = rids in                     *
 *     [bounds[k], bounds[k+1]).                                            *
 * ------------------------------------------------------------------------ */
static uint64_t splitmix64_draw(uint64_t seed, uint64_t k)
{
    uint64_t z = seed + (k + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t oracle_splitmix64(uint64_t seed, uint64_t k) { return splitmix64_draw(seed, k); }

static int cmp_u32(const void *a, const void *b)
{
    const uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    return x < y ? -1 : x > y;
}

int oracle_skew_partition(const uint32_t *rids, uint64_t n_out, uint64_t n_src,
                          uint64_t num_runs, uint64_t sample_size, uint64_t seed,
                          uint32_t *bounds_out, uint64_t *n_runs_out)
{
    if (n_out == 0 || n_src == 0 || n_src > 0xFFFFFFFFull || num_runs < 1 ||
        sample_size < num_runs)
        return -1;
    uint32_t *sample = malloc(sample_size * sizeof(uint32_t));
    if (!sample) return -1;
    for (uint64_t k = 0; k < sample_size; ++k) {           /* sample the rids */
        const uint64_t z = splitmix64_draw(seed, k);
        const uint64_t pos = (uint64_t)(((unsigned __int128)z * n_out) >> 64);
        const uint32_t r = rids[pos];
        sample[k] = r < n_src ? r : (uint32_t)n_src;
    }
    qsort(sample, sample_size, sizeof(uint32_t), cmp_u32);  /* the sampled set is sorted */
    uint64_t n = 0;
    uint32_t last = sample[0];                             /* run 0 holds the smallest sampled rid */
    bounds_out[n++] = 0;
    for (uint64_t i = 1; i < num_runs; ++i) {              /* evenly partition the sample */
        const uint32_t q = sample[i * sample_size / num_runs];
        if (q > last && q < n_src) bounds_out[n++] = last = q;
    }
    bounds_out[n] = (uint32_t)n_src;
    *n_runs_out = n;
    free(sample);
    return 0;
}

/* Fig. 1 (as in (2)) with the runs given by boundaries instead of the high-   *
 * order bits ("the N/L partitions of the input sequence of rids must be       *
 * chosen on some other basis"): run k = [bounds[k], bounds[k+1]),  *
 * bounds ascending from 0 to n_src (an empty run is allowed).  Phase I finds  *
 * each rid's run by binary search; Phase II reads run k's records            *
 * [bounds[k], bounds[k+1]); Phase III as in (2).  run_start_out[n_runs + 1]   *
 * (may be NULL) receives the RID runs' offsets; rid_pos_out[n_out] (may be    *
 * NULL) the positions of the entries of each run, in Phase I order.           */
int oracle_dpg_bounds(const uint8_t *src, uint64_t rec, uint64_t n_src,
                      const uint32_t *rids, uint64_t n_out, const uint32_t *bounds,
                      uint64_t n_runs, uint8_t *dst, uint64_t *run_start_out,
                      uint64_t *rid_pos_out, uint64_t *bad_index)
{
    if (rec == 0 || n_runs == 0 || bounds[0] != 0 || bounds[n_runs] != n_src) return -1;
    for (uint64_t k = 0; k < n_runs; ++k)
        if (bounds[k] > bounds[k + 1]) return -1;
    for (uint64_t i = 0; i < n_out; ++i)
        if ((uint64_t)rids[i] >= n_src) { if (bad_index) *bad_index = i; return 1; }
    uint64_t *run_of = malloc((n_out ? n_out : 1) * sizeof(uint64_t));
    uint64_t *run_start = calloc(n_runs + 1, sizeof(uint64_t));
    uint64_t *cursor = calloc(n_runs + 1, sizeof(uint64_t));
    uint32_t *RID_RUN = malloc((n_out ? n_out : 1) * sizeof(uint32_t));
    uint64_t *RID_POS = malloc((n_out ? n_out : 1) * sizeof(uint64_t));
    uint8_t *RECORD_RUN = malloc((n_out ? n_out : 1) * rec);
    if (!run_of || !run_start || !cursor || !RID_RUN || !RID_POS || !RECORD_RUN) {
        free(run_of); free(run_start); free(cursor); free(RID_RUN); free(RID_POS); free(RECORD_RUN);
        return -1;
    }
    for (uint64_t i = 0; i < n_out; ++i) {                 /* the run k with b_k <= r < b_k+1 */
        uint64_t lo = 0, hi = n_runs;                      /* (the last such k, if runs are empty) */
        while (hi - lo > 1) {
            const uint64_t mid = lo + (hi - lo) / 2;
            if (bounds[mid] <= rids[i]) lo = mid; else hi = mid;
        }
        run_of[i] = lo;
        run_start[lo + 1] += 1;
    }
    for (uint64_t k = 0; k < n_runs; ++k) run_start[k + 1] += run_start[k];
    /* Phase I: Append r to RID_RUN[run] */
    for (uint64_t k = 0; k < n_runs; ++k) cursor[k] = run_start[k];
    for (uint64_t i = 0; i < n_out; ++i) {
        RID_RUN[cursor[run_of[i]]] = rids[i];
        RID_POS[cursor[run_of[i]]] = i;
        cursor[run_of[i]] += 1;
    }
    /* Phase II: run k of INPUT = records [bounds[k], bounds[k+1]) */
    for (uint64_t k = 0; k < n_runs; ++k) {
        const uint8_t *input_run = src + (uint64_t)bounds[k] * rec;
        for (uint64_t j = run_start[k]; j < run_start[k + 1]; ++j)
            memcpy(RECORD_RUN + j * rec, input_run + (uint64_t)(RID_RUN[j] - bounds[k]) * rec, rec);
    }
    /* Phase III: the next record of the rid's run, in RID order */
    for (uint64_t k = 0; k < n_runs; ++k) cursor[k] = run_start[k];
    for (uint64_t i = 0; i < n_out; ++i) {
        memcpy(dst + i * rec, RECORD_RUN + cursor[run_of[i]] * rec, rec);
        cursor[run_of[i]] += 1;
    }
    if (run_start_out) memcpy(run_start_out, run_start, (n_runs + 1) * sizeof(uint64_t));
    if (rid_pos_out) memcpy(rid_pos_out, RID_POS, n_out * sizeof(uint64_t));
    free(run_of); free(run_start); free(cursor); free(RID_RUN); free(RID_POS); free(RECORD_RUN);
    return 0;
}
