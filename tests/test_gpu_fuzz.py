"""Seeded randomised parity: mid-size retrievals and joins (up to a few
million rows, many tiles and runs, ragged tails) with record sizes off the
powers of two, rid distributions the paper's section 2.3 worries about
(uniform, permutation, zipf, one hot run, sorted, strided, constant) and
invalid rids planted at random, through every plan that accepts the shape
(auto, direct, forced paths 1-7, the radix Phase I, clustered path 6).
Every row is compared with the oracle; rows whose rid is invalid must keep the
canary and the status must name the smallest bad position (dpg.h, error
contract).  Bit-exact: record retrieval is a byte copy."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

CANARY = 0xA5
RECS = [1, 2, 3, 5, 6, 7, 9, 12, 15, 20, 24, 31, 33, 40, 48, 63, 65, 96, 100, 127, 129,
        200, 255, 257, 384, 1000]
KINDS = ["uniform", "perm", "zipf", "hot", "sorted", "strided", "equal", "reverse"]
VARIANTS = [
    ("auto", {}),
    ("p1g1", {"path": 1, "gather": 1}),
    ("p1g2", {"path": 1, "gather": 2}),
    ("p2", {"path": 2}),
    ("p2radix", {"path": 2, "hist_mode": 3}),
    ("p2global", {"path": 2, "hist_mode": 2}),
    ("p3", {"path": 3}),
    ("p4", {"path": 4}),
    ("p5", {"path": 5}),
    ("p6", {"path": 6}),
    ("p6c2", {"path": 6, "cluster": 2}),
    ("p7", {"path": 7}),                    # log2_run chosen per case: 2..16 top-level runs
]


def _opts(name, opts, n_src):
    if name == "p7":
        return dict(opts, log2_run=max(1, int(n_src - 1).bit_length() - 3))
    return opts


@pytest.fixture(scope="module")
def dpg():
    import paper_cs_0308004_b200 as m
    return m


def dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).cuda()


def _rids(rng, kind, n_src, n_out):
    if kind == "uniform":
        return rng.integers(0, n_src, n_out).astype(np.uint32)
    if kind == "perm":                     # permutations end to end
        reps = -(-n_out // n_src) if n_out else 0
        return np.concatenate([rng.permutation(n_src) for _ in range(reps)] +
                              [np.zeros(0, np.int64)])[:n_out].astype(np.uint32)
    if kind == "zipf":
        return ((rng.zipf(1.3, n_out) - 1) % n_src).astype(np.uint32)
    if kind == "hot":                      # 90 % of the rids in one 4096-row range
        lo = int(rng.integers(0, n_src))
        r = rng.integers(0, n_src, n_out)
        hot = rng.random(n_out) < 0.9
        r[hot] = (lo + rng.integers(0, 4096, int(hot.sum()))) % n_src
        return r.astype(np.uint32)
    if kind == "sorted":
        return np.sort(rng.integers(0, n_src, n_out)).astype(np.uint32)
    if kind == "reverse":
        return np.sort(rng.integers(0, n_src, n_out))[::-1].astype(np.uint32)
    if kind == "strided":
        return ((np.arange(n_out, dtype=np.uint64) * 2654435761) % n_src).astype(np.uint32)
    if kind == "equal":
        return np.full(n_out, rng.integers(0, n_src), dtype=np.uint32)
    raise KeyError(kind)


def _cases():
    rng = np.random.default_rng(20260)
    out = []
    for k in range(64):
        rec = RECS[k % len(RECS)]
        kind = KINDS[k % len(KINDS)]
        budget = 48 << 20                                  # bytes of source and of output
        n_src = int(min(budget // rec, np.exp(rng.uniform(np.log(2), np.log(4 << 20)))))
        n_out = int(min(budget // rec, np.exp(rng.uniform(np.log(1), np.log(4 << 20)))))
        if kind == "perm":
            n_out = min(n_out, n_src)
        n_bad = int(rng.integers(1, 6)) if k % 3 == 0 and n_out > 0 else 0
        out.append((k, rec, kind, n_src, n_out, n_bad))
    # sources beyond the L2, where the planner's automatic choice changes
    out += [(100, 8, "uniform", 1 << 25, 1 << 23, 3), (101, 4, "perm", 1 << 26, 1 << 22, 0),
            (102, 100, "zipf", 2 << 20, 1 << 21, 2), (103, 16, "hot", 12 << 20, 3 << 20, 0),
            (104, 64, "strided", 3 << 20, 1 << 22, 1), (105, 12, "sorted", 20 << 20, 1 << 21, 0)]
    return out


def _problem(k, rec, kind, n_src, n_out, n_bad):
    rng = np.random.default_rng(1000 + k)
    src = rng.integers(0, 256, (n_src, rec), dtype=np.uint8)
    rids = _rids(rng, kind, n_src, n_out)
    bad = np.zeros(0, np.int64)
    if n_bad:
        bad = np.unique(rng.integers(0, n_out, n_bad))
        vals = np.array([n_src, n_src + 7, 0xFFFFFFFF, max(1 << 31, n_src)], dtype=np.uint32)
        rids[bad] = vals[rng.integers(0, len(vals), bad.size)]
    return src, rids, bad


def _check_rows(got, src, rids, bad):
    ok = np.ones(rids.size, bool)
    ok[bad] = False
    assert np.array_equal(got[ok], oracle.retrieve(src, rids[ok]))
    assert (got[~ok] == CANARY).all()


@pytest.mark.parametrize("k,rec,kind,n_src,n_out,n_bad", _cases())
def test_retrieve_fuzz(dpg, k, rec, kind, n_src, n_out, n_bad):
    src, rids, bad = _problem(k, rec, kind, n_src, n_out, n_bad)
    s, r = dev(src), dev(rids)
    ran = 0
    for name, opts in VARIANTS + [("direct", None)]:
        d = torch.full((n_out, rec), CANARY, dtype=torch.uint8, device="cuda")
        try:
            if opts is None:
                dpg.dpg_retrieve_direct(s, r, dst=d)
            else:
                dpg.dpg_retrieve(s, r, dst=d, **_opts(name, opts, n_src))
        except dpg.DPGError as e:
            assert opts and "path" in opts and e.status == dpg.DPG_ERR_UNSUPPORTED, (name, e)
            continue
        ran += 1
        if bad.size:
            with pytest.raises(dpg.DPGError) as e:
                dpg.dpg_sync_status()
            assert e.value.index == int(bad.min()), name
        else:
            dpg.dpg_sync_status()
        torch.cuda.synchronize()
        try:
            _check_rows(d.cpu().numpy(), src, rids, bad)
        except AssertionError as e:
            raise AssertionError(f"{name}: {e}") from None
    assert ran >= 3                       # auto, direct and at least one forced plan


def _join_cases():
    rng = np.random.default_rng(777)
    out = []
    for k in range(12):
        fb = [4, 8, 12, 16, 7, 100][k % 6]
        rec = [8, 16, 4, 100, 33, 256][(k // 2) % 6]
        n_dim = int(np.exp(rng.uniform(np.log(16), np.log(2 << 20))))
        n_fact = int(np.exp(rng.uniform(np.log(1), np.log(3 << 20))))
        n_fact = min(n_fact, (64 << 20) // (fb + rec))
        out.append((k, fb, rec, n_dim, n_fact, k % 3 == 1))
    return out


@pytest.mark.parametrize("k,fb,rec,n_dim,n_fact,with_bad", _join_cases())
def test_fk_join_fuzz(dpg, k, fb, rec, n_dim, n_fact, with_bad):
    """DPG-Move (every plan the join takes), DPG-Sort and the direct join on
    the same random shapes.  Fact rows whose fk is out of range are left
    unwritten by DPG-Move and the direct join; DPG-Sort reports them and
    leaves its output unspecified (reading A19)."""
    rng = np.random.default_rng(5000 + k)
    dim = rng.integers(0, 256, (n_dim, rec), dtype=np.uint8)
    fact = rng.integers(0, 256, (n_fact, fb), dtype=np.uint8)
    fk = _rids(rng, KINDS[k % len(KINDS)], n_dim, n_fact)
    bad = np.zeros(0, np.int64)
    if with_bad and n_fact:
        bad = np.unique(rng.integers(0, n_fact, 3))
        fk[bad] = n_dim + np.arange(bad.size, dtype=np.uint32)
    ok = np.ones(n_fact, bool)
    ok[bad] = False
    want = oracle.fk_join(fact[ok], fk[ok], dim)
    f, c, d = dev(fact), dev(fk), dev(dim)
    runs = [("move", lambda o: dpg.dpg_fk_join(f, c, d, out=o)),
            ("move_p6", lambda o: dpg.dpg_fk_join(f, c, d, out=o, path=6)),
            ("move_p2", lambda o: dpg.dpg_fk_join(f, c, d, out=o, path=2)),
            ("sort", lambda o: dpg.dpg_fk_join_sort(f, c, d, out=o)),
            ("direct", lambda o: dpg.dpg_fk_join_direct(f, c, d, out=o))]
    for name, fn in runs:
        o = torch.full((n_fact, fb + rec), CANARY, dtype=torch.uint8, device="cuda")
        try:
            fn(o)
        except dpg.DPGError as e:
            assert name.startswith("move_p") and e.status == dpg.DPG_ERR_UNSUPPORTED, (name, e)
            continue
        if bad.size:
            with pytest.raises(dpg.DPGError) as e:
                dpg.dpg_sync_status()
            assert e.value.index == int(bad.min()), name
            if name == "sort":
                continue
        else:
            dpg.dpg_sync_status()
        got = o.cpu().numpy()
        if name == "sort":
            assert np.array_equal(got, oracle.fk_join_sort(fact, fk, dim)), name
            continue
        assert np.array_equal(got[ok], want), name
        assert (got[~ok] == CANARY).all(), name


@pytest.mark.parametrize("k,rec,kind,n_src,n_out,n_bad", _cases()[:48:3])
def test_bounds_segments_host_fuzz(dpg, k, rec, kind, n_src, n_out, n_bad):
    """The other retrieval entry points on the same random problems: DPG over
    random run boundaries (dpg_retrieve_bounds, section 2.3), the output split
    into random segments at odd byte offsets (dpg_retrieve_segments), and the
    host-buffer entry (dpg_retrieve_host)."""
    src, rids, bad = _problem(k, rec, kind, n_src, n_out, n_bad)
    ok = np.ones(n_out, bool)
    ok[bad] = False
    want = np.full((n_out, rec), CANARY, np.uint8)
    want[ok] = oracle.retrieve(src, rids[ok])
    rng = np.random.default_rng(9000 + k)
    s, r = dev(src), dev(rids)

    def settle():
        if bad.size:
            with pytest.raises(dpg.DPGError) as e:
                dpg.dpg_sync_status()
            assert e.value.index == int(bad.min())
        else:
            dpg.dpg_sync_status()

    # random run boundaries: strictly increasing cuts inside (0, n_src)
    nb = int(rng.integers(1, min(64, n_src) + 1))
    cuts = np.unique(rng.integers(1, n_src, nb - 1)) if n_src > 1 else np.zeros(0, np.int64)
    bounds = np.concatenate([[0], cuts, [n_src]]).astype(np.uint32)
    d = torch.full((n_out, rec), CANARY, dtype=torch.uint8, device="cuda")
    try:
        dpg.dpg_retrieve_bounds(s, r, bounds, dst=d)
    except dpg.DPGError as e:
        assert e.status == dpg.DPG_ERR_UNSUPPORTED, e     # a run too large for shared memory
    else:
        settle()
        assert np.array_equal(d.cpu().numpy(), want), "bounds"
    # random segments (some empty), each at a byte offset of 0..3
    nseg = int(rng.integers(1, 6))
    sizes = np.diff(np.sort(np.concatenate([[0, n_out], rng.integers(0, n_out + 1, nseg - 1)])))
    shifts = rng.integers(0, 4, nseg)
    bufs = [torch.full((int(n) * rec + 8,), CANARY, dtype=torch.uint8, device="cuda")
            for n in sizes]
    dpg.dpg_retrieve_segments(s, r, [int(n) for n in sizes],
                              [b.data_ptr() + int(o) for b, o in zip(bufs, shifts)])
    settle()
    row = 0
    for n, b, o in zip(sizes, bufs, shifts):
        h = b.cpu().numpy()
        assert (h[:o] == CANARY).all() and (h[o + n * rec:] == CANARY).all(), "segment bounds"
        assert np.array_equal(h[o:o + n * rec].reshape(n, rec), want[row:row + n]), "segments"
        row += n
    # host buffers in and out
    hs = torch.from_numpy(src).pin_memory()
    hr = torch.from_numpy(rids.view(np.int32)).pin_memory()
    hd = torch.full((n_out, rec), CANARY, dtype=torch.uint8).pin_memory()
    dpg.dpg_retrieve_host(hs, hr, hd)
    settle()
    if not bad.size:                      # (a bad rid's row in a host dst is unspecified)
        assert np.array_equal(hd.numpy(), want), "host"


@pytest.mark.parametrize("k", range(8))
def test_sort_fuzz(dpg, k):
    """dpg_sort / dpg_sort_rids on random record sizes, key offsets and
    lengths, with key alphabets from all-equal to full bytes (ties resolved
    by rid: the stable order)."""
    rng = np.random.default_rng(7000 + k)
    rec = int(rng.integers(1, 130))
    kb = int(rng.integers(1, min(rec, 12) + 1))
    off = int(rng.integers(0, rec - kb + 1))
    n = int(np.exp(rng.uniform(0, np.log(1 << 21))))
    alpha = [1, 2, 4, 26, 256][k % 5]
    src = rng.integers(0, 256, (n, rec), dtype=np.uint8)
    src[:, off:off + kb] = rng.integers(0, alpha, (n, kb), dtype=np.uint8)
    want = oracle.sort_rids(src, off, kb)
    got = dpg.dpg_sort_rids(dev(src), off, kb)
    torch.cuda.synchronize()
    assert np.array_equal(got.cpu().numpy().view(np.uint32), want)
    out = dpg.dpg_sort(dev(src), off, kb)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.sort(src, off, kb))
