"""Pins for the CPU oracle (no GPU).  Each test ties the oracle to something
other than itself: the paper's worked example, brute force through an
independent formulation, a library routine, or an invariant the mathematics
fixes.  A dropped term, a wrong index or a transposed operand in
oracle/oracle.c fails at least one of these."""
import itertools

import numpy as np
import pytest

import datagen
import oracle
from conftest import read_golden


def _distinct_records(n, rec, seed=1):
    """Records whose bytes identify them (first 4 bytes = rid, rest random)."""
    rng = np.random.default_rng(seed)
    src = rng.integers(0, 256, size=(n, rec), dtype=np.uint8)
    ids = np.arange(n, dtype=np.uint32).view(np.uint8).reshape(n, 4)
    k = min(4, rec)
    src[:, :k] = ids[:, :k]
    return src


# --------------------------------------------------------------------------
# Fig. 2 worked example, golden fixture with citations.
# --------------------------------------------------------------------------
def _fig2():
    g = read_golden("fig2_example.txt")
    n_src = int(g["n_src"][0])
    L = int(g["L"][0])
    keys = g["key_of_rid"]
    assert len(keys) == n_src
    # record r = its one-letter key (1 byte) ++ the rid (3 bytes): 4-byte records
    src = np.zeros((n_src, 4), dtype=np.uint8)
    for r, k in enumerate(keys):
        src[r, 0] = ord(k)
        src[r, 1] = r
    rids = np.array([int(x) for x in g["rid_sequence"]], dtype=np.uint32)
    return g, src, rids, L


def test_fig2_output_in_key_order():
    g, src, rids, L = _fig2()
    out = oracle.retrieve(src, rids)
    assert [chr(c) for c in out[:, 0]] == g["output_keys"]


def test_fig2_phases_match_paper():
    g, src, rids, L = _fig2()
    res = oracle.dpg_fig1(src, rids, L)
    rs = res["run_start"].astype(int)
    runs = [list(res["rid_runs"][rs[b]:rs[b + 1]]) for b in range(len(rs) - 1)]
    assert len(runs) == 3
    # Phase I: first four rids go to runs 1, 1, 0, 2
    first = [int(x) for x in rids[:4]]
    assert [next(b for b, run in enumerate(runs) if r in run) for r in first] == \
        [int(x) for x in g["first_runs"]]
    assert runs[0] == [int(x) for x in g["rid_run_0"]]
    assert runs[1] == [int(x) for x in g["rid_run_1"]]
    assert runs[2] == [int(x) for x in g["rid_run_2"]]
    # Phase II: INTERNAL run 0 = c, f, i, l
    internal0 = res["record_runs"][rs[0]:rs[1], 0]
    assert [chr(c) for c in internal0] == g["internal_run_0"]
    # Phase III: output in key order
    assert [chr(c) for c in res["dst"][:, 0]] == g["output_keys"]


# --------------------------------------------------------------------------
# SPEC's trivial definitional cases.
# --------------------------------------------------------------------------
def test_spec_trivial_cases():
    A, B, C = b"AAAA", b"BBBB", b"CCCC"
    src = np.frombuffer(A + B + C, dtype=np.uint8).reshape(3, 4)
    out = oracle.retrieve(src, np.array([2, 0, 1], dtype=np.uint32))
    assert out.tobytes() == C + A + B
    out = oracle.retrieve(src[:2], np.array([1, 1, 0], dtype=np.uint32))
    assert out.tobytes() == B + B + A


def test_identity_and_single_run():
    src = datagen.records(1000, 7, datagen.STREAMS[("test", "src")])
    ident = np.arange(1000, dtype=np.uint32)
    assert np.array_equal(oracle.retrieve(src, ident), src)
    # a single run (L >= n) makes Phase III a plain copy of INTERNAL
    rids = datagen.permutation(1000, datagen.STREAMS[("test", "rids")])
    res = oracle.dpg_fig1(src, rids, 1024)
    assert np.array_equal(res["dst"], res["record_runs"][np.argsort(res["rid_pos"])])
    assert np.array_equal(res["dst"], src[rids.astype(np.int64)])


# --------------------------------------------------------------------------
# Brute force on tiny inputs.
# --------------------------------------------------------------------------
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6])
def test_all_permutations_inverse_scatter(n):
    """For a permutation, D[i] = R[perm[i]] equals the scatter D[inv[r]] = R[r]."""
    rec = 3
    src = _distinct_records(n, rec, seed=n)
    for perm in itertools.permutations(range(n)):
        inv = [0] * n
        for i, r in enumerate(perm):
            inv[r] = i
        expect = np.zeros_like(src)
        for r in range(n):                       # scatter formulation
            expect[inv[r]] = src[r]
        rids = np.array(perm, dtype=np.uint32)
        assert np.array_equal(oracle.retrieve(src, rids), expect)
        for L in (1, 2, 3, n):
            assert np.array_equal(oracle.dpg_fig1(src, rids, L)["dst"], expect)


@pytest.mark.parametrize("n", [1, 2, 3])
def test_all_short_sequences_with_replacement(n):
    """Every rid sequence of length <= 4 over n <= 3 (duplicates, subsets,
    m != n) against numpy fancy indexing."""
    src = _distinct_records(n, 5, seed=10 + n)
    for m in range(0, 5):
        for seq in itertools.product(range(n), repeat=m):
            rids = np.array(seq, dtype=np.uint32)
            expect = src[rids.astype(np.int64)] if m else np.zeros((0, 5), np.uint8)
            assert np.array_equal(oracle.retrieve(src, rids), expect)
            for L in (1, 2, 4):
                assert np.array_equal(oracle.dpg_fig1(src, rids, L)["dst"], expect)


def test_fig1_intermediates_random():
    """Phase I is a stable distribution: run b holds exactly
    the rids of [bL, (b+1)L) in input order, checked against a filter scan;
    Phase II's run j-th record is INPUT[RID_RUN[j]]."""
    n, rec, L = 4096, 9, 256
    src = datagen.records(n, rec, datagen.STREAMS[("test", "src")])
    for rids in (datagen.permutation(n, 77), datagen.uniform(3000, n, 78)):
        res = oracle.dpg_fig1(src, rids, L)
        rs = res["run_start"].astype(np.int64)
        for b in range(len(rs) - 1):
            want = rids[(rids >= b * L) & (rids < (b + 1) * L)]
            got = res["rid_runs"][rs[b]:rs[b + 1]]
            assert np.array_equal(got, want)
            pos = res["rid_pos"][rs[b]:rs[b + 1]].astype(np.int64)
            assert np.array_equal(rids[pos], got)
            assert np.all(np.diff(pos) > 0)
        assert np.array_equal(res["record_runs"], src[res["rid_runs"].astype(np.int64)])
        assert np.array_equal(res["dst"], src[rids.astype(np.int64)])


# --------------------------------------------------------------------------
# Invariants (BASELINE.json north_star).
# --------------------------------------------------------------------------
def test_permutation_preserves_record_multiset():
    w = datagen.make("c1", scale=16)
    out = oracle.retrieve(w["src"], w["rids"])
    key = lambda a: a[np.lexsort(a.T[::-1])]
    assert np.array_equal(key(out), key(w["src"]))
    assert not np.array_equal(out, w["src"])


def test_sort_derived_rids_give_nondecreasing_keys():
    w = datagen.make("c2", scale=64)
    out = oracle.retrieve(w["src"], w["rids"])
    k = out[:, :10]
    hi = k[:, :8].copy().view(">u8").ravel()
    lo = k[:, 8:].copy().view(">u2").ravel()
    ok = (hi[1:] > hi[:-1]) | ((hi[1:] == hi[:-1]) & (lo[1:] >= lo[:-1]))
    assert ok.all()


def test_sort_ties_keep_ascending_rid():
    """Small key space so ties happen (reading A10): equal keys keep rid order."""
    src = datagen.records(5000, 12, 0x777)
    src[:, 1:10] = 0
    src[:, 0] %= 7
    rids = datagen.stable_key_argsort(src, 10)
    out = oracle.retrieve(src, rids)
    keys = out[:, 0]
    assert np.all(np.diff(keys.astype(int)) >= 0)
    for k in range(7):
        r = rids[keys == k]
        assert np.all(np.diff(r.astype(np.int64)) > 0)


def test_join_rows_pair_fact_with_named_dim_record():
    w = datagen.make("c4", scale=4096)
    out = oracle.fk_join(w["fact"], w["fk"], w["dim"])
    assert out.shape == (w["fact"].shape[0], 80)
    assert np.array_equal(out[:, :16], w["fact"])
    index = {w["dim"][j].tobytes(): j for j in range(w["dim"].shape[0])}
    assert len(index) == w["dim"].shape[0]          # random 64-B records are unique
    back = np.array([index[out[i, 16:].tobytes()] for i in range(out.shape[0])])
    assert np.array_equal(back, w["fk"].astype(np.int64))


def test_join_against_nested_loop():
    rng = np.random.default_rng(5)
    n_dim, n_fact = 13, 40
    dim = rng.integers(0, 256, (n_dim, 6), dtype=np.uint8)
    fact = rng.integers(0, 256, (n_fact, 3), dtype=np.uint8)
    fk = rng.integers(0, n_dim, n_fact).astype(np.uint32)
    rows = []
    for i in range(n_fact):                 # nested-loop join
        for j in range(n_dim):
            if fk[i] == j:
                rows.append(np.concatenate([fact[i], dim[j]]))
    assert np.array_equal(oracle.fk_join(fact, fk, dim), np.array(rows))


# --------------------------------------------------------------------------
# Error behaviour and edge cases (readings A6, A7).
# --------------------------------------------------------------------------
def test_rid_range_error_reports_smallest_index():
    src = _distinct_records(10, 4)
    rids = np.array([1, 2, 10, 3, 99, 4], dtype=np.uint32)
    with pytest.raises(oracle.RidRangeError) as e:
        oracle.retrieve(src, rids)
    assert e.value.index == 2
    with pytest.raises(oracle.RidRangeError) as e:
        oracle.fk_join(src[:6, :2], rids, src)
    assert e.value.index == 2


def test_empty_inputs():
    src = _distinct_records(5, 4)
    assert oracle.retrieve(src, np.zeros(0, np.uint32)).shape == (0, 4)
    with pytest.raises(oracle.RidRangeError):
        oracle.retrieve(np.zeros((0, 4), np.uint8), np.array([0], np.uint32))


def test_sampled_oracle_matches_full():
    w = datagen.make("c1", scale=8)
    full = oracle.retrieve(w["src"], w["rids"])
    idx = np.array([0, 5, 100, w["rids"].size - 1], dtype=np.uint64)
    assert np.array_equal(oracle.retrieve_at(w["src"], w["rids"], idx), full[idx.astype(np.int64)])


# --------------------------------------------------------------------------
# The generators are deterministic and produce what they claim.
# --------------------------------------------------------------------------
def test_generators():
    a = datagen.permutation(100000, 5)
    assert np.array_equal(np.sort(a), np.arange(100000, dtype=np.uint32))
    assert np.array_equal(a, datagen.permutation(100000, 5))
    u = datagen.uniform(100000, 1000, 6)
    assert u.max() < 1000 and len(np.unique(u)) > 990
    b1 = datagen.random_bytes(1001, 9)
    b2 = datagen.random_bytes(500, 9, offset=501)
    assert np.array_equal(b1[501:], b2)
    f = datagen.feistel(1000, 0, 1000, 11)
    assert np.array_equal(np.sort(f), np.arange(1000, dtype=np.uint64))
    f2 = datagen.feistel(1000, 300, 50, 11)
    assert np.array_equal(f2, f[300:350])


# --------------------------------------------------------------------------
# Three-phase key-pointer sorting (section 3): the sort oracle.
# --------------------------------------------------------------------------
def test_sort_oracle_brute_force_tiny():
    """Every tiny input against Python's sorted() on (key bytes, rid) -- an
    independent stable ordering -- with alphabets small enough to force ties."""
    rng = np.random.default_rng(5)
    for n in range(0, 8):
        for trial in range(40):
            rec = int(rng.integers(1, 6))
            key_off = int(rng.integers(0, rec))
            key_bytes = int(rng.integers(1, rec - key_off + 1))
            src = rng.integers(0, 3, (n, rec), dtype=np.uint8)
            want = sorted(range(n), key=lambda i: (bytes(src[i, key_off:key_off + key_bytes]), i))
            got = oracle.sort_rids(src, key_off, key_bytes)
            assert got.tolist() == want
            assert np.array_equal(oracle.sort(src, key_off, key_bytes),
                                  src[np.array(want, dtype=np.int64)] if n else src[:0])


def test_sort_oracle_against_lexsort_and_invariants():
    rng = np.random.default_rng(6)
    for n, rec, off, kb, alpha in [(5000, 100, 0, 10, 256), (3000, 24, 7, 9, 4), (4096, 16, 2, 3, 2)]:
        src = rng.integers(0, alpha, (n, rec), dtype=np.uint8)
        got = oracle.sort_rids(src, off, kb)
        # library routine: numpy's stable lexsort (last key = primary)
        cols = [src[:, off + j] for j in reversed(range(kb))]
        assert np.array_equal(got, np.lexsort(cols).astype(np.uint32))
        # invariants: a permutation, keys non-decreasing, ties by ascending rid
        assert np.array_equal(np.sort(got), np.arange(n, dtype=np.uint32))
        keys = [bytes(src[r, off:off + kb]) for r in got]
        for a, b, ra, rb in zip(keys, keys[1:], got, got[1:]):
            assert a < b or (a == b and ra < rb)


def test_sort_oracle_matches_datamation_generator():
    """Config 2's rids (the generator's own stable argsort of the 10-byte keys)
    are the oracle's sorted rids."""
    w = datagen.make("c2", scale=16)
    assert np.array_equal(oracle.sort_rids(w["src"], 0, 10), w["rids"])


def test_fk_join_sort_oracle_is_the_move_join_in_fk_order():
    """DPG-Sort join: the same rows as the DPG-Move join, permuted
    into stable fk order (numpy's stable argsort, an independent ordering)."""
    rng = np.random.default_rng(8)
    for n_fact, n_dim, fb, rec in [(0, 3, 4, 8), (1, 1, 2, 3), (500, 40, 16, 64), (3000, 7, 5, 11)]:
        dim = rng.integers(0, 256, (n_dim, rec), dtype=np.uint8)
        fact = rng.integers(0, 256, (n_fact, fb), dtype=np.uint8)
        fk = rng.integers(0, n_dim, n_fact).astype(np.uint32)
        move = oracle.fk_join(fact, fk, dim)
        order = np.argsort(fk, kind="stable")
        assert np.array_equal(oracle.fk_join_sort(fact, fk, dim), move[order])
    fk[17 % max(1, fk.size)] = n_dim
    with pytest.raises(oracle.RidRangeError):
        oracle.fk_join_sort(fact, fk, dim)


def test_exponential_fk_generator_shape():
    """Reading A18: exp(c * (r >> 10)) with r < 2^31 and c = -1e-7
    lies in (e^{-0.2097152}, 1], so the keys fill [0.8108 n_dim, n_dim) with a
    density falling as 1/key."""
    n_dim = 1 << 16
    fk = datagen.exp_fk(200000, n_dim, datagen.STREAMS[("c4x", "fk")])
    assert fk.dtype == np.uint32 and fk.max() < n_dim
    assert fk.min() >= int(np.floor(n_dim * np.exp(-1e-7 * ((2 ** 31 - 1) >> 10))))
    h = np.histogram(fk, bins=4, range=(int(0.8109 * n_dim), n_dim))[0]
    assert np.all(np.diff(h) < 0)


def test_batch_lookup_against_dict():
    """Batch lookup pinned to a Python dict over the same pairs,
    with absent keys, repeated queries and the empty cases."""
    rng = np.random.default_rng(3)
    keys = rng.choice(1 << 32, 5000, replace=False).astype(np.uint32)
    d = {int(k): j for j, k in enumerate(keys)}
    q = np.concatenate([keys[rng.integers(0, 5000, 3000)],
                        rng.integers(0, 1 << 32, 2000, dtype=np.uint64).astype(np.uint32),
                        np.array([0, 0xFFFFFFFF], dtype=np.uint32)])
    want = np.array([d.get(int(x), oracle.NOT_FOUND) for x in q], dtype=np.uint32)
    assert np.array_equal(oracle.batch_lookup(keys, q), want)
    assert oracle.batch_lookup(keys, q[:0]).size == 0
    assert np.all(oracle.batch_lookup(keys[:0], q[:10]) == oracle.NOT_FOUND)
    # a key equal to 0xFFFFFFFF is still found (the sentinel is a rid, not a key)
    k2 = np.array([7, 0xFFFFFFFF, 3], dtype=np.uint32)
    assert list(oracle.batch_lookup(k2, np.array([0xFFFFFFFF, 3, 8], np.uint32))) == \
        [1, 2, oracle.NOT_FOUND]


def test_hash_index_generator_holds_every_key():
    """The batch-lookup input (datagen.hash_index): walking slot h(k) and its
    overflow chain finds every key with its rid; absent keys are not found;
    every entry is in exactly one place."""
    keys = datagen.feistel(1 << 32, 0, 3000, 0x611).astype(np.uint32)
    table, pool = datagen.hash_index(keys, 11)
    E = 0xFFFFFFFF

    def walk(k):
        h = (int(k) * 0x9E3779B1 & 0xFFFFFFFF) >> (32 - 11)
        s = table[h]
        if s[1] == E:
            return E
        if s[0] == k:
            return int(s[1])
        nx = int(s[2])
        while nx != E:
            if pool[nx][0] == k:
                return int(pool[nx][1])
            nx = int(pool[nx][2])
        return E
    assert [walk(k) for k in keys] == list(range(3000))
    absent = datagen.feistel(1 << 32, 3000, 200, 0x611).astype(np.uint32)
    assert all(walk(k) == E for k in absent)
    assert (table[:, 1] != E).sum() + len(pool) == 3000


def test_btree_generator_descent_finds_every_key():
    """The batch-lookup B+-tree input (datagen.btree_index): a descent from the
    top (largest entry <= key in each 16-entry node) ends at every key with
    its rid; absent keys end at a different key."""
    keys = datagen.feistel(1 << 32, 0, 5000, 0x611).astype(np.uint32)
    levels, rids = datagen.btree_index(keys)
    assert levels[-1].size <= 16 and levels[0].size == 5000

    def descend(q):
        top = levels[-1]
        c = int(np.sum(top <= q))
        if c == 0:
            return None
        j = c - 1
        for t in range(len(levels) - 2, -1, -1):
            node = levels[t][16 * j:16 * j + 16]
            j = 16 * j + int(np.sum(node <= q)) - 1
        return j if levels[0][j] == q else None
    assert all(rids[descend(k)] == i for i, k in enumerate(keys))
    absent = datagen.feistel(1 << 32, 5000, 300, 0x611).astype(np.uint32)
    assert all(descend(k) is None for k in absent)


# --------------------------------------------------------------------------
# 64-bit rids (config 5's global rids): oracle_retrieve_u64,
# oracle_retrieve_at_u64 and the generated-source definition.
# --------------------------------------------------------------------------
def test_u64_retrieve_matches_numpy_indexing():
    """D[i] = R[rid[i]] with uint64 rids against numpy fancy indexing (an
    independent definition), every length <= 3 sequence over n <= 3 plus a
    seeded large case."""
    for n in range(1, 4):
        src = _distinct_records(n, 5, seed=n)
        for k in range(0, 4):
            for seq in itertools.product(range(n), repeat=k):
                rids = np.array(seq, dtype=np.uint64)
                got = oracle.retrieve(src, rids)
                assert np.array_equal(got, src[rids.astype(np.int64)] if k else np.zeros((0, 5), np.uint8))
    rng = np.random.default_rng(9)
    src = rng.integers(0, 256, size=(5000, 100), dtype=np.uint8)
    rids = rng.integers(0, 5000, 20000).astype(np.uint64)
    assert np.array_equal(oracle.retrieve(src, rids), src[rids.astype(np.int64)])
    # the same bytes through the 32-bit entry (a different code path)
    assert np.array_equal(oracle.retrieve(src, rids), oracle.retrieve(src, rids.astype(np.uint32)))


def test_u64_rids_are_not_truncated():
    """A rid >= 2^32 is out of range for a small source; a 32-bit truncation
    would silently copy record rid mod 2^32 instead."""
    src = _distinct_records(10, 8)
    rids = np.array([1, 2, (1 << 32) + 3, 4, (1 << 33) + 1], dtype=np.uint64)
    with pytest.raises(oracle.RidRangeError) as e:
        oracle.retrieve(src, rids)
    assert e.value.index == 2
    with pytest.raises(oracle.RidRangeError):
        oracle.retrieve_at(src, rids, np.array([2], dtype=np.uint64))
    assert np.array_equal(oracle.retrieve_at(src, rids, np.array([0, 3], dtype=np.uint64)),
                          src[[1, 4]])


def test_u64_retrieve_at_samples_the_definition():
    rng = np.random.default_rng(3)
    src = rng.integers(0, 256, size=(3000, 12), dtype=np.uint8)
    rids = rng.integers(0, 3000, 7000).astype(np.uint64)
    idx = np.unique(rng.integers(0, 7000, 500)).astype(np.uint64)
    full = src[rids.astype(np.int64)]
    assert np.array_equal(oracle.retrieve_at(src, rids, idx), full[idx.astype(np.int64)])
    assert np.array_equal(oracle.retrieve_at(src, rids.astype(np.uint32), idx),
                          full[idx.astype(np.int64)])


def test_retrieve_generated_matches_materialised_source():
    """The generated-source definition (config 5's records made pointwise at
    their byte offsets) equals the retrieval from the materialised stream."""
    n, rec, sid = 4096, 100, datagen.STREAMS[("c5", "src")]
    src = datagen.records(n, rec, sid)
    rids = datagen.feistel(n, 0, n, datagen.STREAMS[("c5", "rids")])[:300]
    rids = np.concatenate([rids, rids[:7]])                 # repeats
    assert np.array_equal(oracle.retrieve_generated(rec, n, sid, rids), src[rids.astype(np.int64)])
    with pytest.raises(oracle.RidRangeError) as e:
        oracle.retrieve_generated(rec, n, sid, np.array([5, n, 1], dtype=np.uint64))
    assert e.value.index == 1


def test_threaded_retrieve_equals_single_thread():
    """The all-cores timing entry (index ranges, one thread each) computes the
    definition: equal to numpy indexing for every thread count, and the
    smallest bad position over all ranges is reported."""
    rng = np.random.default_rng(21)
    src = rng.integers(0, 256, size=(3001, 13), dtype=np.uint8)
    rids = rng.integers(0, 3001, 10007).astype(np.uint32)
    for t in (1, 2, 3, 8, 64):
        assert np.array_equal(oracle.retrieve_threads(src, rids, t), src[rids.astype(np.int64)])
    bad = rids.copy()
    bad[[9000, 4321]] = 3001
    with pytest.raises(oracle.RidRangeError) as e:
        oracle.retrieve_threads(src, bad, 7)
    assert e.value.index == 4321
