/*
 * datagen/gen.c -- seeded, synthetic input generators shared by the oracle
 * side (tests, bench cpu_baseline) and the CUDA side (tests, bench, smoke).
 *
 * This module holds NONE of the method's arithmetic: it only produces the
 * inputs (record bytes, rid sequences, foreign keys).  Reading A12/A13 of
 * the paper draws its data with UNIX random(); here
 * every stream is a counter-based splitmix64 keyed by (seed, stream id), so
 * any element can be regenerated pointwise and in parallel.
 *
 *   word(seed, sid, k) = mix64(key(seed, sid) + (k + 1) * GOLDEN)
 *   key(seed, sid)     = mix64(seed * GOLDEN ^ mix64(sid + 0x5851F42D4C957F2D))
 *   byte j of a byte stream = little-endian byte (j % 8) of word(j / 8)
 *
 * Permutations: Fisher-Yates (Durstenfeld) with unbiased bounded draws
 * (Lemire's multiply-and-reject), consuming words 0,1,2,... of the stream.
 * With-replacement draws: word k -> unbiased bounded draw, rejection
 * resamples walk a second counter range (k + n + retry * n) so each element
 * stays pointwise computable.
 * Large permutations that must be evaluated pointwise (multi-GPU config 5)
 * use a keyed balanced Feistel network on 2^bits with cycle walking.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static inline uint64_t stream_key(uint64_t seed, uint64_t sid)
{
    return mix64(seed * GOLDEN ^ mix64(sid + 0x5851F42D4C957F2DULL));
}

static inline uint64_t word_at(uint64_t key, uint64_t k)
{
    return mix64(key + (k + 1) * GOLDEN);
}

uint64_t gen_word(uint64_t seed, uint64_t sid, uint64_t k)
{
    return word_at(stream_key(seed, sid), k);
}

/* n bytes of stream (seed, sid) starting at byte offset `off`. */
void gen_bytes(uint64_t seed, uint64_t sid, uint64_t off, uint64_t n, uint8_t *out)
{
    const uint64_t key = stream_key(seed, sid);
    uint64_t j = 0;
    /* head: unaligned bytes up to a word boundary */
    while (j < n && ((off + j) & 7)) {
        uint64_t w = word_at(key, (off + j) >> 3);
        out[j] = (uint8_t)(w >> (8 * ((off + j) & 7)));
        ++j;
    }
    uint64_t nw = (n - j) >> 3;
    uint64_t w0 = (off + j) >> 3;
    #pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < (int64_t)nw; ++t) {
        uint64_t w = word_at(key, w0 + (uint64_t)t);
        memcpy(out + j + 8 * (uint64_t)t, &w, 8);     /* little-endian host */
    }
    j += 8 * nw;
    while (j < n) {
        uint64_t w = word_at(key, (off + j) >> 3);
        out[j] = (uint8_t)(w >> (8 * ((off + j) & 7)));
        ++j;
    }
}

/* Lemire bounded draw in [0, range) from a sequence of words. */
static inline uint64_t bounded(uint64_t key, uint64_t *ctr, uint64_t range)
{
    uint64_t x = word_at(key, (*ctr)++);
    __uint128_t m = (__uint128_t)x * range;
    uint64_t l = (uint64_t)m;
    if (l < range) {
        uint64_t t = (0 - range) % range;
        while (l < t) {
            x = word_at(key, (*ctr)++);
            m = (__uint128_t)x * range;
            l = (uint64_t)m;
        }
    }
    return (uint64_t)(m >> 64);
}

/* Uniformly random permutation of [0, n) (Fisher-Yates), uint32 output. */
void gen_permutation_u32(uint64_t seed, uint64_t sid, uint64_t n, uint32_t *out)
{
    const uint64_t key = stream_key(seed, sid);
    uint64_t ctr = 0;
    for (uint64_t i = 0; i < n; ++i) out[i] = (uint32_t)i;
    for (uint64_t i = n; i > 1; --i) {
        uint64_t j = bounded(key, &ctr, i);        /* j in [0, i) */
        uint32_t t = out[i - 1]; out[i - 1] = out[j]; out[j] = t;
    }
}

/* n iid uniform draws in [0, bound), with replacement, uint32 output.
 * Element k uses word k; a rejected draw retries with word k + n*(1+retry). */
void gen_uniform_u32(uint64_t seed, uint64_t sid, uint64_t n, uint64_t bound, uint32_t *out)
{
    const uint64_t key = stream_key(seed, sid);
    const uint64_t t = (0 - bound) % bound;
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < (int64_t)n; ++k) {
        uint64_t retry = 0;
        for (;;) {
            uint64_t x = word_at(key, (uint64_t)k + n * retry);
            __uint128_t m = (__uint128_t)x * bound;
            if ((uint64_t)m >= t) { out[k] = (uint32_t)(m >> 64); break; }
            ++retry;
        }
    }
}

/* Keyed balanced Feistel permutation of [0, 2^bits) (bits even, >= 2),
 * `rounds` rounds, cycle-walked onto [0, n) for n <= 2^bits.  Pointwise:
 * out[j] = P(first + j). */
static inline uint64_t feistel_once(uint64_t key, unsigned half, unsigned rounds, uint64_t x)
{
    const uint64_t mask = (1ULL << half) - 1;
    uint64_t l = x >> half, r = x & mask;
    for (unsigned i = 0; i < rounds; ++i) {
        uint64_t f = mix64(key ^ (r * GOLDEN) ^ ((uint64_t)(i + 1) << 56)) & mask;
        uint64_t nl = r, nr = l ^ f;
        l = nl; r = nr;
    }
    return (l << half) | r;
}

void gen_feistel_u64(uint64_t seed, uint64_t sid, unsigned bits, unsigned rounds,
                     uint64_t n, uint64_t first, uint64_t count, uint64_t *out)
{
    const uint64_t key = stream_key(seed, sid);
    const unsigned half = bits / 2;
    #pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < (int64_t)count; ++j) {
        uint64_t x = feistel_once(key, half, rounds, first + (uint64_t)j);
        while (x >= n) x = feistel_once(key, half, rounds, x);
        out[j] = x;
    }
}

/* Hash index over (keys[j], rid j), j < n (the indexed relation F of the
 * batch lookup): a primary array of 2^m_log2 slots and an overflow
 * pool, 16-byte entries {key, rid, next, 0}; slot h(key) = (key * 0x9E3779B1)
 * >> (32 - m_log2) holds the first key that hashes there, later colliding
 * keys go to the pool, linked from the slot (newest first); rid 0xFFFFFFFF
 * marks an empty slot, next 0xFFFFFFFF the end of a chain.  The pool is
 * then laid out in slot order (reading A20: the overflow area is "a second
 * hash array").  Returns the pool entries used. */
uint64_t gen_hash_index(const uint32_t *keys, uint64_t n, unsigned m_log2, uint32_t *table,
                        uint32_t *pool)
{
    const uint64_t M = 1ULL << m_log2;
    for (uint64_t h = 0; h < M; ++h) {
        table[4 * h] = 0; table[4 * h + 1] = 0xFFFFFFFFu;
        table[4 * h + 2] = 0xFFFFFFFFu; table[4 * h + 3] = 0;
    }
    uint64_t np = 0;
    for (uint64_t j = 0; j < n; ++j) {
        const uint32_t k = keys[j];
        const uint64_t h = (uint32_t)(k * 0x9E3779B1u) >> (32 - m_log2);
        uint32_t *s = table + 4 * h;
        if (s[1] == 0xFFFFFFFFu) {
            s[0] = k; s[1] = (uint32_t)j;
        } else {
            uint32_t *p = pool + 4 * np;
            p[0] = k; p[1] = (uint32_t)j; p[2] = s[2]; p[3] = 0;
            s[2] = (uint32_t)np++;
        }
    }
    /* the overflow pool in slot order ("a second hash array"):
     * chain of slot 0 first, each chain's entries consecutive */
    if (np) {
        uint32_t *sorted = (uint32_t *)malloc(np * 16);
        if (!sorted) return np;
        uint64_t w = 0;
        for (uint64_t h = 0; h < M; ++h) {
            uint32_t nx = table[4 * h + 2];
            if (nx == 0xFFFFFFFFu) continue;
            table[4 * h + 2] = (uint32_t)w;
            while (nx != 0xFFFFFFFFu) {
                const uint32_t *p = pool + 4 * (uint64_t)nx;
                uint32_t *d = sorted + 4 * w;
                d[0] = p[0]; d[1] = p[1]; d[3] = 0;
                nx = p[2];
                d[2] = nx == 0xFFFFFFFFu ? 0xFFFFFFFFu : (uint32_t)(w + 1);
                ++w;
            }
        }
        memcpy(pool, sorted, np * 16);
        free(sorted);
    }
    return np;
}
