"""GPU parity of DPG under data skew (section 2.3): the run
boundaries from a sorted rid sample (dpg_skew_partition) bit-exact against
oracle.skew_partition, Phase I over boundary runs against the boundary-mode
Fig. 1 (oracle.dpg_bounds), and retrieval over boundary runs
(dpg_retrieve_bounds) against the oracle -- uniform, exponential,
all-equal and sorted rids, empty runs, runs wider than a stage, invalid rids,
odd record sizes.  Boundaries given to the GPU come from the oracle or from
the test itself, never from the CUDA path."""
import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dpg():
    import paper_cs_0308004_b200 as m
    return m


def dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _rids(kind, n_out, n_src, seed):
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        return rng.integers(0, n_src, n_out).astype(np.uint32)
    if kind == "perm":
        return rng.permutation(n_src)[:n_out].astype(np.uint32)
    if kind == "exp":
        return datagen.exp_fk(n_out, n_src, sid=seed)
    if kind == "equal":
        return np.full(n_out, rng.integers(0, n_src), dtype=np.uint32)
    if kind == "sorted":
        return np.sort(rng.integers(0, n_src, n_out)).astype(np.uint32)
    if kind == "hot":      # 90% of the rids on 1% of the records
        r = rng.integers(0, n_src, n_out).astype(np.uint32)
        hot = rng.random(n_out) < 0.9
        r[hot] = rng.integers(0, max(1, n_src // 100), int(hot.sum())).astype(np.uint32)
        return r
    raise KeyError(kind)


PART_CASES = [
    # kind, n_out, n_src, num_runs, sample_size, seed
    ("uniform", 100_000, 1 << 20, 16, 4096, 7),
    ("exp", 100_000, 1 << 20, 16, 8192, 3),
    ("exp", 1 << 20, 1 << 24, 1024, 32768, 11),
    ("hot", 500_000, 3_000_000, 300, 30000, 5),
    ("equal", 1000, 1000, 16, 256, 1),
    ("sorted", 77_777, 12345, 100, 1000, 2),
    ("perm", 5, 5, 5, 5, 9),
    ("uniform", 1, 1, 1, 1, 0),
    ("uniform", 3, 2**32 - 1, 3, 17, 123456789),
    ("uniform", 10_000, 50, 64, 64, 4),            # more runs asked than distinct rids
    ("uniform", 65_536, 1 << 16, 1, 32768, 8),     # one run
]


@pytest.mark.parametrize("kind,n_out,n_src,K,S,seed", PART_CASES)
def test_skew_partition_matches_oracle(dpg, kind, n_out, n_src, K, S, seed):
    rids = _rids(kind, n_out, min(n_src, 1 << 30), seed) if n_src < 2**32 - 1 else \
        np.array([0, 2**32 - 2, 77], dtype=np.uint32)
    want = oracle.skew_partition(rids, n_src, K, S, seed)
    got = dpg.dpg_skew_partition(dev(rids), n_src, K, sample_size=S, seed=seed)
    assert np.array_equal(got, want), (got[:8], want[:8])


def test_skew_partition_invalid_rids_count_as_n_src(dpg):
    rng = np.random.default_rng(3)
    n_src = 1000
    rids = rng.integers(0, 2 * n_src, 20000).astype(np.uint32)     # half invalid
    for S, K in [(1000, 10), (32768, 200)]:
        want = oracle.skew_partition(rids, n_src, K, S, 5)
        got = dpg.dpg_skew_partition(dev(rids), n_src, K, sample_size=S, seed=5)
        assert np.array_equal(got, want)
    dpg.dpg_sync_status()                      # sampling reports nothing


def test_skew_partition_errors(dpg):
    r = dev(np.arange(10, dtype=np.uint32))
    with pytest.raises(dpg.DPGError) as e:
        dpg.dpg_skew_partition(r, 10, 8, sample_size=4)
    assert e.value.status == dpg.DPG_ERR_INVALID_ARG
    with pytest.raises(dpg.DPGError) as e:
        dpg.dpg_skew_partition(r, 10, 8, sample_size=32769)
    assert e.value.status == dpg.DPG_ERR_UNSUPPORTED
    with pytest.raises(dpg.DPGError) as e:
        dpg.dpg_skew_partition(r[:0], 10, 1, sample_size=4)
    assert e.value.status == dpg.DPG_ERR_INVALID_ARG


def _merged(bounds, n_src, s):
    """The layout dpg_distribute_bounds documents, built here independently:
    the bounds and the multiples of L in one ascending list, a bound equal to a
    multiple of L first."""
    L = 1 << s
    grid = [j * L for j in range(1, (n_src + L - 1) // L)]
    items = [(int(b), 0) for b in bounds] + [(g, 1) for g in grid]
    return np.array([v for v, _ in sorted(items)], dtype=np.uint32)


@pytest.mark.parametrize("kind,n_out,n_src,K,s", [
    ("exp", 200_000, 1 << 18, 64, 10),
    ("hot", 100_000, 300_000, 40, 12),
    ("uniform", 12_345, 777, 9, 5),
    ("equal", 5000, 5000, 16, 8),
    ("sorted", 50_000, 40_000, 200, 9),
])
def test_distribute_bounds_matches_fig1_boundary_runs(dpg, kind, n_out, n_src, K, s):
    rids = _rids(kind, n_out, n_src, 17)
    bounds = oracle.skew_partition(rids, n_src, K, max(K, 4096), 1)
    M = _merged(bounds, n_src, s)
    pairs, rs = dpg.dpg_distribute_bounds(dev(rids), n_src, bounds, s)
    rs = host(rs).astype(np.int64)
    pairs = host(pairs).view(np.uint64)
    assert rs.size == M.size
    ref = oracle.dpg_bounds(np.zeros((n_src, 1), np.uint8), rids, M)
    assert np.array_equal(rs, ref["run_start"].astype(np.int64))
    local = (pairs & 0xFFFFFFFF).astype(np.int64)
    pos = (pairs >> 32).astype(np.int64)
    ref_pos = ref["rid_pos"].astype(np.int64)
    for b in np.flatnonzero(np.diff(rs)):
        seg = slice(rs[b], rs[b + 1])
        assert np.array_equal(np.sort(pos[seg]), ref_pos[seg])        # same set of entries
        assert np.array_equal(local[seg], rids[pos[seg]].astype(np.int64) - int(M[b]))


RETRIEVE_CASES = []
_rng = np.random.default_rng(88)
for _k in range(36):
    _rec = [1, 3, 4, 8, 12, 16, 24, 32, 64, 100, 128, 256][_k % 12]
    _kind = ["exp", "hot", "uniform", "perm", "equal", "sorted"][_k % 6]
    _n_src = int(_rng.integers(1, 300_000))
    _n_out = int(_rng.integers(1, 400_000)) if _kind != "perm" else int(_rng.integers(1, _n_src + 1))
    _K = int(_rng.integers(1, 600))
    RETRIEVE_CASES.append((_k, _rec, _kind, _n_src, _n_out, _K))


@pytest.mark.parametrize("k,rec,kind,n_src,n_out,K", RETRIEVE_CASES)
def test_retrieve_bounds_matches_oracle(dpg, k, rec, kind, n_src, n_out, K):
    rng = np.random.default_rng(1000 + k)
    src = rng.integers(0, 256, size=(n_src, rec), dtype=np.uint8)
    rids = _rids(kind, n_out, n_src, k)
    bounds = oracle.skew_partition(rids, n_src, K, max(K, 8192), k)
    got = host(dpg.dpg_retrieve_bounds(dev(src), dev(rids), bounds))
    assert np.array_equal(got, oracle.dpg_bounds(src, rids, bounds)["dst"])
    dpg.dpg_sync_status()


@pytest.mark.parametrize("bounds_kind", ["one", "every", "empty_runs", "multiples"])
def test_retrieve_bounds_layouts(dpg, bounds_kind):
    """Bounds chosen by the test: one run over the whole source (split into
    stages by the plan), a run per record, repeated bounds (empty runs), and
    bounds on multiples of a power of two (ties with the plan's cuts)."""
    rng = np.random.default_rng(4)
    n_src, rec, n = 70_001, 20, 150_000
    src = rng.integers(0, 256, size=(n_src, rec), dtype=np.uint8)
    rids = rng.integers(0, n_src, n).astype(np.uint32)
    if bounds_kind == "one":
        b = np.array([0, n_src], np.uint32)
    elif bounds_kind == "every":
        b = np.arange(n_src + 1, dtype=np.uint32)
    elif bounds_kind == "empty_runs":
        c = np.sort(rng.integers(1, n_src, 50)).astype(np.uint32)
        b = np.concatenate([[0, 0], c, c[::3], [n_src, n_src]]).astype(np.uint32)
        b.sort()
    else:
        b = np.concatenate([np.arange(0, n_src, 512), [n_src]]).astype(np.uint32)
    got = host(dpg.dpg_retrieve_bounds(dev(src), dev(rids), b))
    assert np.array_equal(got, oracle.dpg_bounds(src, rids, b)["dst"])


def test_retrieve_bounds_invalid_rids(dpg):
    n_src, rec, n = 40_000, 16, 90_000
    rng = np.random.default_rng(2)
    src = rng.integers(0, 256, size=(n_src, rec), dtype=np.uint8)
    rids = datagen.exp_fk(n, n_src, sid=9)
    bounds = oracle.skew_partition(rids, n_src, 50, 4096, 0)
    bad = np.array([5000, 123, 89999])
    rids[bad] = n_src + np.arange(bad.size, dtype=np.uint32)
    out = torch.full((n, rec), 0x5A, dtype=torch.uint8, device="cuda")
    dpg.dpg_retrieve_bounds(dev(src), dev(rids), bounds, dst=out)
    with pytest.raises(dpg.DPGError) as ei:
        dpg.dpg_sync_status()
    assert ei.value.index == 123
    got = host(out)
    good = np.setdiff1d(np.arange(n), bad)
    assert np.array_equal(got[good], oracle.retrieve(src, rids[good]))
    assert (got[bad] == 0x5A).all()


def test_retrieve_bounds_rejects_bad_layouts(dpg):
    src = dev(np.zeros((100, 8), np.uint8))
    rids = dev(np.arange(100, dtype=np.uint32))
    for b in ([0, 99], [1, 100], [0, 60, 50, 100], [0]):
        with pytest.raises((dpg.DPGError, ValueError)):
            dpg.dpg_retrieve_bounds(src, rids, np.array(b, np.uint32))


@pytest.mark.slow
def test_retrieve_bounds_full_size_exponential(dpg):
    """Config 4's dimension side under the paper's exponential keys
    (P:890-896): 64 Mi rids into 16 Mi x 64 B, runs from a 32 Ki sample;
    the whole output against the oracle, in chunks."""
    n_src, rec, n = 1 << 24, 64, 1 << 26
    src = torch.empty((n_src, rec), dtype=torch.uint8, device="cuda")
    datagen.random_bytes_cuda(src, sid=41)
    rids = datagen.exp_fk(n, n_src, sid=42)
    bounds = oracle.skew_partition(rids, n_src, 4096, 32768, 3)
    out = dpg.dpg_retrieve_bounds(src, dev(rids), bounds)
    dpg.dpg_sync_status()
    hsrc = host(src)
    for c0 in range(0, n, 1 << 23):
        c1 = min(n, c0 + (1 << 23))
        assert np.array_equal(host(out[c0:c1]), oracle.retrieve(hsrc, rids[c0:c1])), c0
