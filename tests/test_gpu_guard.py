"""Guard bands around the output of every plan (no sanitizer on this pool):
the destination is the middle of a larger buffer whose margins hold a canary
pattern; after each call the margins must be unchanged and the rows equal the
oracle's.  Covers the round-2 kernels (path 2's radix Phase I and work items,
boundary runs, path 6 with clusters, path 7) on ragged sizes and heavy runs."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

MARGIN = 4096 + 48


@pytest.fixture(scope="module")
def dpg():
    import paper_cs_0308004_b200 as m
    return m


def dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).cuda()


def _guarded(n, rec):
    buf = torch.full((MARGIN + n * rec + MARGIN,), 0xC3, dtype=torch.uint8, device="cuda")
    return buf, buf[MARGIN:MARGIN + n * rec].view(n, rec)


def _check(buf, dst, n, rec, want):
    torch.cuda.synchronize()
    h = buf.cpu().numpy()
    assert (h[:MARGIN] == 0xC3).all(), "write before dst"
    assert (h[MARGIN + n * rec:] == 0xC3).all(), "write past dst"
    assert np.array_equal(h[MARGIN:MARGIN + n * rec].reshape(n, rec), want)


CASES = [
    # (name, rec, n_src, n_out, opts)
    ("p2 radix", 24, 20011, 50021, dict(path=2, hist_mode=3, log2_run=3)),
    ("p2 radix 3 passes", 12, 300007, 70001, dict(path=2, hist_mode=3, log2_run=0)),
    ("p2 counting", 40, 30001, 40009, dict(path=2, hist_mode=1, log2_run=5)),
    ("p2 global", 8, 40009, 30011, dict(path=2, hist_mode=2, log2_run=2)),
    ("p6", 8, 100003, 120011, dict(path=6, log2_run=8)),
    ("p6 cluster 4", 16, 200003, 150001, dict(path=6, log2_run=12, cluster=4)),
    ("p1", 64, 50021, 60013, dict(path=1, log2_run=6)),
    ("auto", 100, 70001, 90001, dict()),
]


@pytest.mark.parametrize("name,rec,n_src,n_out,opts", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("kind", ["uniform", "heavy"])
def test_output_guard_bands(dpg, name, rec, n_src, n_out, opts, kind):
    rng = np.random.default_rng(rec * 7 + n_out)
    src = rng.integers(0, 256, (n_src, rec), dtype=np.uint8)
    rids = rng.integers(0, n_src, n_out).astype(np.uint32)
    if kind == "heavy":
        rids[rng.random(n_out) < 0.6] = n_src // 3      # one run with most of the rids
    buf, dst = _guarded(n_out, rec)
    try:
        dpg.dpg_retrieve(dev(src), dev(rids), dst=dst, **opts)
    except dpg.DPGError as e:
        assert e.status == dpg.DPG_ERR_UNSUPPORTED
        pytest.skip("plan refused")
    _check(buf, dst, n_out, rec, oracle.retrieve(src, rids))
    dpg.dpg_sync_status()


def test_bounds_guard_bands(dpg):
    rng = np.random.default_rng(5)
    n_src, rec, n = 90001, 20, 120007
    src = rng.integers(0, 256, (n_src, rec), dtype=np.uint8)
    rids = rng.integers(0, n_src, n).astype(np.uint32)
    rids[::3] = 17
    bounds = oracle.skew_partition(rids, n_src, 300, 8192, 2)
    buf, dst = _guarded(n, rec)
    dpg.dpg_retrieve_bounds(dev(src), dev(rids), bounds, dst=dst)
    _check(buf, dst, n, rec, oracle.retrieve(src, rids))
