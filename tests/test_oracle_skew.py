"""Pins for the oracle's data-skew functions (section 2.3; no GPU):
the sample generator against SplitMix64's published sequence, the partition
against S:162-170's examples (uniform, identical and exponential rids) and an
exhaustive recount of the quantile rule on small inputs, and the
boundary-mode Fig. 1 against numpy indexing, against the high-bit Fig. 1 on
boundaries at multiples of L, and against the Fig. 2 worked example."""
import numpy as np
import pytest

import datagen
import oracle
from conftest import read_golden


def test_splitmix64_published_sequence():
    # SplitMix64 (Steele, Lea, Flood, OOPSLA 2014) seeded with 1234567: the
    # reference test vector of the generator (first five outputs).
    want = [6457827717110365317, 3203168211198807973, 9817491932198370423,
            4593380528125082431, 16408922859458223821]
    assert [oracle.splitmix64(1234567, k) for k in range(5)] == want


def _bucket_counts(rids, bounds):
    """Rids per run [bounds[k], bounds[k+1]) by a full scan (np.searchsorted)."""
    run = np.searchsorted(bounds, rids, side="right") - 1
    return np.bincount(run, minlength=bounds.size - 1)


def _check_layout(b, n_src, num_runs):
    assert b[0] == 0 and b[-1] == n_src
    assert np.all(np.diff(b.astype(np.int64)) > 0)          # strictly ascending
    assert 1 <= b.size - 1 <= num_runs


def test_uniform_rids_balanced():
    # uniform rids over [0, n), 16 runs, m = 10^5: every bucket within
    # 4 sqrt(m) of m / 16 (full-scan counts)
    m, n = 100_000, 1 << 20
    rids = datagen.uniform(m, n, sid=31)
    b = oracle.skew_partition(rids, n, 16, 4096, seed=7)
    _check_layout(b, n, 16)
    assert b.size == 17
    c = _bucket_counts(rids, b)
    assert np.all(np.abs(c - m / 16) <= 4 * np.sqrt(m)), c


def test_identical_rids_one_run():
    # all rids identical -> one run
    for v in (0, 5, 999):
        rids = np.full(1000, v, dtype=np.uint32)
        b = oracle.skew_partition(rids, 1000, 16, 256, seed=1)
        assert list(b) == [0, 1000]


def test_exponential_rids_balanced_where_high_bits_are_not():
    # the paper's exponential keys, 16 runs, m = 10^5: the
    # largest bucket <= 2 m / 16, while 16 equal-width runs put most rids in one
    m, n = 100_000, 1 << 20
    rids = datagen.exp_fk(m, n, sid=32)
    b = oracle.skew_partition(rids, n, 16, 8192, seed=3)
    _check_layout(b, n, 16)
    assert _bucket_counts(rids, b).max() <= 2 * m / 16
    equal = np.arange(17, dtype=np.int64) * (n // 16)
    assert _bucket_counts(rids, equal).max() > 4 * m / 16


def test_quantile_rule_recount():
    # The rule restated through independent steps: draw positions from the
    # pinned generator with Python integers, sort with sorted(), walk the
    # quantiles; over many small inputs, including invalid rids and heavy ties.
    rng = np.random.default_rng(5)
    for trial in range(300):
        n_src = int(rng.integers(1, 40))
        m = int(rng.integers(1, 30))
        rids = rng.integers(0, n_src + 3, size=m).astype(np.uint32)   # some >= n_src
        K = int(rng.integers(1, 12))
        S = K + int(rng.integers(0, 20))
        seed = int(rng.integers(0, 2**63))
        sample = []
        for k in range(S):
            pos = (oracle.splitmix64(seed, k) * m) >> 64
            sample.append(min(int(rids[pos]), n_src))
        sample = sorted(sample)
        cuts, last = [], sample[0]
        for i in range(1, K):
            q = sample[i * S // K]
            if last < q < n_src:
                cuts.append(q)
                last = q
        got = oracle.skew_partition(rids, n_src, K, S, seed)
        assert list(got) == [0] + cuts + [n_src], (trial, n_src, K, S)
        # every run holds at least one sampled rid
        runs = np.searchsorted(got, [s for s in sample if s < n_src], side="right") - 1
        assert set(runs) == set(range(got.size - 1)) or all(s >= n_src for s in sample)


def test_skew_partition_errors():
    rids = np.arange(10, dtype=np.uint32)
    with pytest.raises(ValueError):
        oracle.skew_partition(rids[:0], 10, 4, 16, 0)            # empty rid sequence
    with pytest.raises(ValueError):
        oracle.skew_partition(rids, 10, 0, 16, 0)                # num_runs >= 1
    with pytest.raises(ValueError):
        oracle.skew_partition(rids, 10, 8, 4, 0)                 # sample_size >= num_runs


def _records(n, rec, seed=2):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, 256, size=(n, rec), dtype=np.uint8)
    src[:, :4] = np.arange(n, dtype=np.uint32).view(np.uint8).reshape(n, 4)
    return src


def test_dpg_bounds_is_retrieval():
    rng = np.random.default_rng(9)
    for n_src, m, rec in [(1, 5, 4), (37, 100, 8), (500, 2000, 12), (4096, 4096, 16)]:
        src = _records(n_src, rec)
        rids = rng.integers(0, n_src, size=m).astype(np.uint32)
        cuts = np.unique(rng.integers(0, n_src, size=7))
        b = np.concatenate([[0], cuts, cuts[:2], [n_src]]).astype(np.uint32)   # with empty runs
        b.sort()
        res = oracle.dpg_bounds(src, rids, b)
        assert np.array_equal(res["dst"], src[rids])              # D[i] = R[S_rid[i]]
        assert np.array_equal(np.diff(res["run_start"].astype(np.int64)),
                              _bucket_counts(rids, b))            # (last of equal bounds)
        # each run's entries in Phase I order = ascending positions (stable)
        rs = res["run_start"].astype(int)
        for k in range(b.size - 1):
            pos = res["rid_pos"][rs[k]:rs[k + 1]]
            assert np.all(np.diff(pos.astype(np.int64)) > 0)
            assert np.all((rids[pos] >= b[k]) & (rids[pos] < b[k + 1]))


def test_dpg_bounds_on_multiples_of_L_is_fig1():
    # Boundaries at the multiples of L are Fig. 1's high-order-bit runs
    rng = np.random.default_rng(11)
    src = _records(1000, 8)
    rids = rng.permutation(1000).astype(np.uint32)
    for L in (1, 7, 64, 1000, 4096):
        b = np.minimum(np.arange((1000 + L - 1) // L + 1) * L, 1000).astype(np.uint32)
        got = oracle.dpg_bounds(src, rids, b)
        want = oracle.dpg_fig1(src, rids, L)
        assert np.array_equal(got["dst"], want["dst"])
        assert np.array_equal(got["run_start"], want["run_start"])
        assert np.array_equal(got["rid_pos"], want["rid_pos"])


def test_dpg_bounds_fig2_example():
    g = read_golden("fig2_example.txt")
    n_src, L = int(g["n_src"][0]), int(g["L"][0])
    src = np.zeros((n_src, 4), dtype=np.uint8)
    for r, k in enumerate(g["key_of_rid"]):
        src[r, 0] = ord(k)
        src[r, 1] = r
    rids = np.array([int(x) for x in g["rid_sequence"]], dtype=np.uint32)
    b = np.array([0, L, 2 * L, n_src], dtype=np.uint32)
    res = oracle.dpg_bounds(src, rids, b)
    rs = res["run_start"].astype(int)
    assert [int(x) for x in rids[res["rid_pos"][rs[0]:rs[1]]]] == [int(x) for x in g["rid_run_0"]]
    assert [chr(c) for c in res["dst"][:, 0]] == g["output_keys"]


def test_dpg_bounds_errors():
    src = _records(10, 4)
    with pytest.raises(ValueError):
        oracle.dpg_bounds(src, np.zeros(3, np.uint32), np.array([0, 5, 9], np.uint32))  # end != n_src
    with pytest.raises(ValueError):
        oracle.dpg_bounds(src, np.zeros(3, np.uint32), np.array([0, 6, 5, 10], np.uint32))
    with pytest.raises(oracle.RidRangeError) as e:
        oracle.dpg_bounds(src, np.array([1, 10, 2], np.uint32), np.array([0, 10], np.uint32))
    assert e.value.index == 1
