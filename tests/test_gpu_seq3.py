"""GPU parity of the three sequential passes over shared-memory runs (path 6,
csrc/seq3.cu) against the CPU oracle: bit-exact on every record layout the
plan takes, many runs and chunks with ragged tails, duplicates, invalid rids,
the join's payload rows, and the Phase I intermediates against Fig. 1's
Phase I."""
import numpy as np
import pytest

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


def _case(seed, n_src, rec, n_out, kind):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, 256, size=(n_src, rec), dtype=np.uint8)
    if kind == "perm":
        rids = rng.permutation(n_src)[:n_out].astype(np.uint32)
    elif kind == "repl":
        rids = rng.integers(0, n_src, n_out).astype(np.uint32)
    elif kind == "equal":
        rids = np.full(n_out, rng.integers(0, n_src), dtype=np.uint32)
    elif kind == "sorted":
        rids = np.sort(rng.integers(0, n_src, n_out)).astype(np.uint32)
    else:
        raise KeyError(kind)
    return src, rids


CASES = []
_rng = np.random.default_rng(66)
for _k in range(48):
    _rec = [4, 8, 12, 16, 20, 24, 32, 48, 64, 100, 128, 256][_k % 12]
    _kind = ["perm", "repl", "equal", "sorted"][_k % 4]
    _n_src = int(_rng.integers(1, 40000))
    _n_out = int(_rng.integers(1, _n_src + 1)) if _kind == "perm" else int(_rng.integers(1, 2 * _n_src + 2))
    # runs of 2^s records (several to hundreds of runs), chunks of Phase I
    _smin = max(0, int(np.ceil(np.log2(max(1, _n_src / 8192)))))
    _smin = max(_smin, {4: 2, 12: 2, 20: 2, 100: 2, 8: 1, 24: 1, 48: 0}.get(_rec, 0))  # L*rec % 16 == 0
    _s = int(_rng.integers(_smin, max(_smin, min(16, int(np.log2(120000 // _rec)))) + 1))
    _g = int(_rng.integers(1, 40)) if _k % 3 else 0
    CASES.append((_k, _n_src, _rec, _n_out, _kind, _s, _g))


@pytest.mark.parametrize("k,n_src,rec,n_out,kind,s,g", CASES)
def test_seq3_sweep(dpg, k, n_src, rec, n_out, kind, s, g):
    src, rids = _case(k, n_src, rec, n_out, kind)
    p = dpg.dpg_plan(rec, n_src, n_out, path=6, log2_run=s, grid_distribute=g)
    assert p["path"] == 6 and p["run_len"] == 1 << s
    out = torch.full((n_out, rec), 0xA5, dtype=torch.uint8, device="cuda")
    dpg.dpg_retrieve(dev(src), dev(rids), dst=out, path=6, log2_run=s, grid_distribute=g)
    assert dpg.last_path() == 6
    assert np.array_equal(host(out), oracle.retrieve(src, rids))
    dpg.dpg_sync_status()


def test_seq3_default_geometry_many_runs(dpg):
    """The automatic stage (L * rec <= 128 KB) on a source of hundreds of runs,
    the last one partial and not a multiple of 16 bytes."""
    n_src, rec = 5_000_003, 12
    rng = np.random.default_rng(3)
    src = rng.integers(0, 256, size=(n_src, rec), dtype=np.uint8)
    rids = rng.integers(0, n_src, 3_000_001).astype(np.uint32)
    p = dpg.dpg_plan(rec, n_src, rids.size, path=6)
    assert p["path"] == 6 and p["num_runs"] > 100
    got = host(dpg.dpg_retrieve(dev(src), dev(rids), path=6))
    assert np.array_equal(got, oracle.retrieve(src, rids))


@pytest.mark.parametrize("n_src,n_out,s,kind", [(300_000, 300_000, 9, "perm"), (1 << 20, 777_777, 11, "repl"),
                                                 (1 << 24, 1 << 24, 15, "perm")])
def test_seq3_phase1_shrunk_tile(dpg, n_src, n_out, s, kind):
    """4-byte records with hundreds of runs: the plan shrinks the tile so that
    two Phase I CTAs share an SM (profiles/r02_s3_p6dist.md); several tiles,
    the last one ragged; the last case is config 3's 4-byte permutation."""
    rec = 4
    src, rids = _case(n_src + s, n_src, rec, n_out, kind)
    p = dpg.dpg_plan(rec, n_src, n_out, path=6, log2_run=s)
    full = min(32768, (110 << 10) // (rec + 2)) & ~15
    nsub = -(-n_out // p["tile"])
    assert p["path"] == 6 and 0.8 * full <= p["tile"] < full and p["grid_distribute"] == min(nsub, 296)
    assert n_out % p["tile"] != 0 and n_out > p["tile"]
    out = torch.full((n_out, rec), 0xA5, dtype=torch.uint8, device="cuda")
    dpg.dpg_retrieve(dev(src), dev(rids), dst=out, path=6, log2_run=s)
    assert dpg.last_path() == 6
    assert np.array_equal(host(out), oracle.retrieve(src, rids))
    dpg.dpg_sync_status()


def test_seq3_invalid_rids(dpg):
    """rid >= n_src: the row is left unwritten (canary kept), every other row
    is right, and the smallest offending position is reported (reading A6)."""
    n_src, rec, n = 30000, 16, 50000
    src, rids = _case(7, n_src, rec, n, "repl")
    bad = np.array([4321, 777, 49999, 20000])
    rids[bad] = n_src + np.arange(bad.size, dtype=np.uint32)
    out = torch.full((n, rec), 0x5A, dtype=torch.uint8, device="cuda")
    dpg.dpg_retrieve(dev(src), dev(rids), dst=out, path=6, log2_run=10)
    with pytest.raises(dpg.DPGError) as ei:
        dpg.dpg_sync_status()
    assert ei.value.index == 777
    got = host(out)
    good = np.setdiff1d(np.arange(n), bad)
    assert np.array_equal(got[good], oracle.retrieve(src, rids[good]))
    assert (got[bad] == 0x5A).all()


def test_seq3_phase1_against_fig1(dpg):
    """Phase I: RID_RUN[b] holds exactly the rids of run b with
    their positions; the run boundaries equal Fig. 1's; inside a run the
    entries come tile by tile in tile order (the pieces (tile, run) are
    concatenated), and sorted by position they are Fig. 1's
    RID_RUN[b] in its order."""
    n_src, n = 50_000, 120_000
    src, rids = _case(11, n_src, 4, n, "repl")
    s, g = 10, 23
    T = dpg.dpg_plan(4, n_src, n, path=6, log2_run=s, grid_distribute=g)["tile"]
    assert T == g * 16
    pairs, rs = dpg.dpg_distribute(dev(rids), n_src, s, path=6, grid_distribute=g)
    pairs = host(pairs).astype(np.uint64)
    rs = host(rs).astype(np.uint64)
    ref = oracle.dpg_fig1(src, rids, 1 << s)
    assert np.array_equal(rs, ref["run_start"])
    for b in range(rs.size - 1):
        seg = pairs[rs[b]:rs[b + 1]]
        pos = (seg >> np.uint64(32)).astype(np.int64)
        cells = pos // T
        assert (np.diff(cells) >= 0).all()
        order = np.argsort(pos, kind="stable")
        assert np.array_equal(pos[order], ref["rid_pos"][rs[b]:rs[b + 1]].astype(np.int64))
        local = (seg & np.uint64(0xffffffff))[order]
        assert np.array_equal(local + np.uint64(b << s), ref["rid_runs"][rs[b]:rs[b + 1]])


@pytest.mark.parametrize("fact_bytes,rec", [(16, 64), (4, 8), (8, 16), (16, 4)])
def test_seq3_join_payload(dpg, fact_bytes, rec):
    """DPG-Move join on path 6: Phase III writes fact[i] ++ dim[fk[i]]
    (P:593-608); an fk >= n_dim leaves its row unwritten and is reported."""
    rng = np.random.default_rng(fact_bytes * 1000 + rec)
    n_dim, n_fact = 70_000, 200_001
    dim = rng.integers(0, 256, size=(n_dim, rec), dtype=np.uint8)
    fact = rng.integers(0, 256, size=(n_fact, fact_bytes), dtype=np.uint8)
    fk = rng.integers(0, n_dim, n_fact).astype(np.uint32)
    out = host(dpg.dpg_fk_join(dev(fact), dev(fk), dev(dim), path=6))
    assert np.array_equal(out, oracle.fk_join(fact, fk, dim))
    fk[[5, 100_000]] = n_dim
    o = torch.full((n_fact, fact_bytes + rec), 0x33, dtype=torch.uint8, device="cuda")
    dpg.dpg_fk_join(dev(fact), dev(fk), dev(dim), out=o, path=6)
    with pytest.raises(dpg.DPGError) as ei:
        dpg.dpg_sync_status()
    assert ei.value.index == 5
    got = host(o)
    assert (got[[5, 100_000]] == 0x33).all()
    keep = np.setdiff1d(np.arange(n_fact), [5, 100_000])
    assert np.array_equal(got[keep], oracle.fk_join(fact[keep], fk[keep], dim))


def test_seq3_unaligned_source_falls_back(dpg):
    """A source that is not 16-byte aligned cannot be staged by one bulk copy:
    the automatic plan takes another shared-memory plan, a forced path 6
    reports DPG_ERR_UNSUPPORTED."""
    n_src, rec = 20000, 8
    src, rids = _case(5, n_src, rec, 30000, "repl")
    buf = torch.zeros(n_src * rec + 8, dtype=torch.uint8, device="cuda")
    buf[8:] = dev(src.reshape(-1))
    s = buf[8:].view(n_src, rec)
    with pytest.raises(dpg.DPGError):
        dpg.dpg_retrieve(s, dev(rids), path=6)
    got = host(dpg.dpg_retrieve(s, dev(rids)))
    assert np.array_equal(got, oracle.retrieve(src, rids))


@pytest.mark.parametrize("cl", [2, 4, 8])
@pytest.mark.parametrize("rec,n_src,n_out,kind", [(8, 300_001, 250_000, "repl"), (16, 200_000, 200_000, "perm"),
                                                  (4, 50_000, 120_001, "sorted"), (32, 123_457, 99_999, "equal")])
def test_seq3_cluster_runs(dpg, cl, rec, n_src, n_out, kind):
    """Runs held by a thread-block cluster of cl CTAs (each a slice of the run
    in its shared memory, lookups across the cluster through distributed
    shared memory): bit-exact on duplicates, permutations, sorted and
    all-equal rids, with short runs (many runs per cluster) and the automatic
    slice length."""
    src, rids = _case(cl * 10 + rec, n_src, rec, n_out, kind)
    for s in (0, 10):
        try:
            p = dpg.dpg_plan(rec, n_src, n_out, path=6, cluster=cl, log2_run=s)
        except dpg.DPGError:
            continue
        assert p["cluster"] == cl
        out = torch.full((n_out, rec), 0x77, dtype=torch.uint8, device="cuda")
        dpg.dpg_retrieve(dev(src), dev(rids), dst=out, path=6, cluster=cl, log2_run=s)
        assert np.array_equal(host(out), oracle.retrieve(src, rids)), s
        dpg.dpg_sync_status()


@pytest.mark.parametrize("rec,n_src,n_out,kind,s1", [(8, 300_001, 250_000, "repl", 16),
                                                      (16, 200_000, 200_000, "perm", 15),
                                                      (4, 70_000, 90_001, "sorted", 14),
                                                      (32, 123_457, 99_999, "equal", 15),
                                                      (12, 100_000, 150_000, "repl", 12)])
def test_twolevel(dpg, rec, n_src, n_out, kind, s1):
    """Two-level DPG (path 7; the paper's multi-pass DPG): the
    rids distributed into super-runs of 2^s1 records, each super-run retrieved
    by its own plan, the rows gathered back in output order -- bit-exact,
    including an invalid rid (reported, row unwritten)."""
    src, rids = _case(rec + s1, n_src, rec, n_out, kind)
    rids[n_out // 3] = n_src + 1
    p = dpg.dpg_plan(rec, n_src, n_out, path=7, log2_run=s1)
    assert p["path"] == 7 and p["num_runs"] == (n_src + (1 << s1) - 1) >> s1
    out = torch.full((n_out, rec), 0x3D, dtype=torch.uint8, device="cuda")
    dpg.dpg_retrieve(dev(src), dev(rids), dst=out, path=7, log2_run=s1)
    assert dpg.last_path() == 7
    with pytest.raises(dpg.DPGError) as e:
        dpg.dpg_sync_status()
    assert e.value.index == n_out // 3
    got = host(out)
    ok = rids < n_src
    assert np.array_equal(got[ok], oracle.retrieve(src, rids[ok]))
    assert (got[~ok] == 0x3D).all()
