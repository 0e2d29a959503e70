"""The multi-GPU path's GPU pieces on one GPU: the owner partition kernel
against a plain definition, and the whole exchange (NCCL, world size 1)
against the oracle.  Multi-rank exchanges are covered on CPU by
tests/test_dist_gloo.py (no second GPU in this environment)."""
import os
import socket

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


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
@pytest.mark.parametrize("parts,log2_span,n_total", [(4, 10, 4096), (8, 7, 1000), (1, 12, 3000)])
def test_partition_groups_by_owner(dpg, dtype, parts, log2_span, n_total):
    rng = np.random.default_rng(parts * 100 + log2_span)
    rids = rng.integers(0, n_total, 5000).astype(dtype)
    local, pos, counts = dpg.dpg_partition(torch.from_numpy(rids).cuda(), n_total, log2_span, parts)
    torch.cuda.synchronize()
    counts = counts.cpu().numpy()
    m = int(counts.sum())
    local = local[:m].cpu().numpy().astype(np.int64)
    pos = pos[:m].cpu().numpy().astype(np.int64)
    owner = rids.astype(np.int64) >> log2_span
    assert np.array_equal(counts, np.bincount(owner, minlength=parts))
    start = np.concatenate([[0], np.cumsum(counts)])
    for o in range(parts):
        seg_pos = pos[start[o]:start[o + 1]]
        seg_loc = local[start[o]:start[o + 1]]
        want = np.nonzero(owner == o)[0]
        assert np.array_equal(np.sort(seg_pos), want)
        assert np.array_equal(seg_loc + (o << log2_span), rids[seg_pos].astype(np.int64))


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
@pytest.mark.parametrize("parts,log2_span,n_total", [(4, 10, 4096), (8, 7, 1000), (1, 12, 3000),
                                                     (300, 4, 4800)])
def test_partition_inv(dpg, dtype, parts, log2_span, n_total):
    """Requests owner by owner (stable within each owner), inv = each row's
    request position; the reply gather restores output order."""
    rng = np.random.default_rng(parts * 10 + log2_span)
    rids = rng.integers(0, n_total, 7777).astype(dtype)
    rids[[5, 600]] = n_total + 3                       # out of range: no request
    local, inv, counts = dpg.dpg_partition_inv(torch.from_numpy(rids).cuda(), n_total, log2_span,
                                               parts)
    with pytest.raises(dpg.DPGError):
        dpg.dpg_sync_status()
    counts = counts.cpu().numpy()
    inv = inv.cpu().numpy().astype(np.int64)
    local = local.cpu().numpy().astype(np.int64)
    ok = rids.astype(np.int64) < n_total
    owner = rids.astype(np.int64) >> log2_span
    assert np.array_equal(counts, np.bincount(owner[ok], minlength=parts))
    assert np.all(inv[~ok] == -1)
    assert np.array_equal(np.sort(inv[ok]), np.arange(ok.sum()))
    assert np.array_equal(local[inv[ok]] + (owner[ok] << log2_span), rids[ok].astype(np.int64))
    start = np.concatenate([[0], np.cumsum(counts)])
    assert np.all((inv[ok] >= start[owner[ok]]) & (inv[ok] < start[owner[ok] + 1]))
    # the reply gather: rows of the requests in request order -> output order
    rows = torch.from_numpy(rng.integers(0, 256, (int(ok.sum()), 36), dtype=np.uint8)).cuda()
    dst = torch.zeros((rids.size, 36), dtype=torch.uint8, device="cuda")
    dpg.dpg_gather_rows(rows, torch.from_numpy(inv.astype(np.int32)).cuda(), dst)
    d = dst.cpu().numpy()
    assert np.array_equal(d[ok], rows.cpu().numpy()[inv[ok]])
    assert np.all(d[~ok] == 0)


def test_retrieve_dist_single_rank_nccl(dpg):
    import torch.distributed as dist
    from paper_cs_0308004_b200.dist import retrieve_dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(3)
        src = rng.integers(0, 256, (50000, 100), dtype=np.uint8)
        rids = rng.integers(0, 50000, 70000).astype(np.int64)
        out = retrieve_dist(torch.from_numpy(src).cuda(), torch.from_numpy(rids).cuda(), 50000,
                            max_rows_per_round=30000)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), oracle.retrieve(src, rids.astype(np.uint64)))
    finally:
        dist.destroy_process_group()


def test_retrieve_dist_fused_single_rank_nccl(dpg):
    """The fused exchange at P = 1: the owner's retrieval writes into the
    rank's own receive window (dpg_ipc_alloc), Phase III gathers from it."""
    import torch.distributed as dist
    from paper_cs_0308004_b200.dist import retrieve_dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(4)
        src = rng.integers(0, 256, (50000, 100), dtype=np.uint8)
        rids = rng.integers(0, 50000, 70000).astype(np.int64)
        out = retrieve_dist(torch.from_numpy(src).cuda(), torch.from_numpy(rids).cuda(), 50000,
                            max_rows_per_round=30000, fused=True)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), oracle.retrieve(src, rids.astype(np.uint64)))
    finally:
        dist.destroy_process_group()


def _ipc_child(handle, n_rows, rec, seed, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch as t
    import paper_cs_0308004_b200 as m
    try:
        rng = np.random.default_rng(seed)
        src = rng.integers(0, 256, (5000, rec), dtype=np.uint8)
        rids = rng.integers(0, 5000, n_rows).astype(np.uint32)
        win = m.ipc_open(handle)
        # two segments into the parent's window: rows [0, 1000) at row 3000 of
        # the window, the rest at row 0 -- the owner side of the fused exchange
        m.dpg_retrieve_segments(t.from_numpy(src).cuda(), t.from_numpy(rids.view(np.int32)).cuda(),
                                [1000, n_rows - 1000], [win + 3000 * rec, win])
        t.cuda.synchronize()
        m.ipc_close(win)
        q.put("ok")
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(repr(e))


def test_ipc_window_written_by_another_process(dpg):
    """A receive window allocated here and written by a second process that
    maps it from its IPC handle (the same GPU stands in for the peer: the
    mapping and the segment addressing are what is tested; no kernel waits on
    another process)."""
    import multiprocessing as mpp
    rec, n_rows = 100, 3000
    ptr, handle = dpg.ipc_alloc((n_rows + 1000) * rec)
    try:
        ctx = mpp.get_context("spawn")
        q = ctx.Queue()
        p = ctx.Process(target=_ipc_child, args=(handle, n_rows, rec, 9, q))
        p.start()
        msg = q.get(timeout=240)
        p.join(60)
        assert msg == "ok", msg
        got = torch.empty((n_rows + 1000, rec), dtype=torch.uint8, device="cuda")
        dpg.dpg_gather_rows(ptr, torch.arange(n_rows + 1000, dtype=torch.int32, device="cuda"), got,
                            n_rows=n_rows + 1000)
        got = got.cpu().numpy()
        rng = np.random.default_rng(9)
        src = rng.integers(0, 256, (5000, rec), dtype=np.uint8)
        rids = rng.integers(0, 5000, n_rows).astype(np.uint32)
        want = oracle.retrieve(src, rids)
        assert np.array_equal(got[3000:4000], want[:1000])
        assert np.array_equal(got[:n_rows - 1000], want[1000:])
    finally:
        dpg.ipc_free(ptr)


def test_c_abi_retrieve_dist_single_rank(dpg):
    """dpg_comm_create / dpg_retrieve_dist / dpg_comm_destroy at one rank:
    the native exchange (NCCL loaded by the library, the rank's own window)
    against the oracle, including a rank whose block is empty and an invalid
    rid."""
    comm = dpg.dpg_comm_create(dpg.dpg_get_unique_id(), 1, 0)
    try:
        rng = np.random.default_rng(11)
        for n_total, rec, n_out in ((50000, 100, 70000), (1000, 12, 0), (3, 8, 500),
                                    (4096, 64, 4096)):
            src = rng.integers(0, 256, (n_total, rec), dtype=np.uint8)
            rids = rng.integers(0, n_total, n_out).astype(np.int64)
            out = dpg.dpg_retrieve_dist(comm, torch.from_numpy(src).cuda(), n_total,
                                        torch.from_numpy(rids).cuda())
            torch.cuda.synchronize()
            assert np.array_equal(out.cpu().numpy(), oracle.retrieve(src, rids.astype(np.uint64)))
        rids = np.arange(100, dtype=np.int64)
        rids[37] = 5000
        dpg.dpg_retrieve_dist(comm, torch.zeros((100, 8), dtype=torch.uint8, device="cuda"), 100,
                              torch.from_numpy(rids).cuda())
        with pytest.raises(dpg.DPGError) as e:
            dpg.dpg_sync_status()
        assert e.value.index == 37
    finally:
        dpg.dpg_comm_destroy(comm)


def _owner_span(n_total, P):
    per = max(1, -(-n_total // P))
    return 1 << (per - 1).bit_length()


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_loopback_exchange_config5_down_scaled(dpg, P):
    """The multi-GPU exchange for P virtual ranks on one GPU
    (dpg_retrieve_dist_loopback): config 5's shape down-scaled -- 2^20 records
    of 100 B from the c5 source stream, rids = the c5 Feistel permutation
    (uint64), block-partitioned by output position -- through the same owner
    partition, count matrix, request and window-row offsets, segmented owner
    DPG and Phase III as dpg_retrieve_dist; every rank's output against the
    oracle (64-bit rids)."""
    n_total, rec = 1 << 20, 100
    src = datagen.records(n_total, rec, datagen.STREAMS[("c5", "src")])
    rids = datagen.feistel(n_total, 0, n_total, datagen.STREAMS[("c5", "rids")])
    S = _owner_span(n_total, P)
    shards = [torch.from_numpy(src[r * S:min(n_total, (r + 1) * S)]).cuda() for r in range(P)]
    blocks = [rids[r * n_total // P:(r + 1) * n_total // P] for r in range(P)]
    outs = dpg.dpg_retrieve_dist_loopback(shards, n_total,
                                          [torch.from_numpy(b.view(np.int64)).cuda() for b in blocks])
    torch.cuda.synchronize()
    for b, o in zip(blocks, outs):
        assert np.array_equal(o.cpu().numpy(), oracle.retrieve(src, b))


@pytest.mark.parametrize("P,rec", [(2, 12), (5, 8), (8, 64), (3, 100)])
def test_loopback_exchange_uneven_and_repeated(dpg, P, rec):
    """Uneven output blocks (one empty), repeated rids (with replacement), a
    source size that is not a multiple of P (the last owner's shard short),
    and an invalid rid (reported, row left unwritten)."""
    rng = np.random.default_rng(P * 100 + rec)
    n_total = 100_003
    src = rng.integers(0, 256, (n_total, rec), dtype=np.uint8)
    S = _owner_span(n_total, P)
    shards = [torch.from_numpy(src[r * S:min(n_total, (r + 1) * S)]).cuda() for r in range(P)]
    sizes = [int(x) for x in rng.integers(0, 60_000, P)]
    sizes[1] = 0
    blocks = [rng.integers(0, n_total, n).astype(np.uint64) for n in sizes]
    blocks[0][7] = n_total + 5                         # invalid rid at rank 0, row 7
    outs = [torch.full((n, rec), 0x6B, dtype=torch.uint8, device="cuda") for n in sizes]
    dpg.dpg_retrieve_dist_loopback(shards, n_total,
                                   [torch.from_numpy(b.view(np.int64)).cuda() for b in blocks], outs)
    with pytest.raises(dpg.DPGError) as e:
        dpg.dpg_sync_status()
    assert e.value.index == 7
    for r, (b, o) in enumerate(zip(blocks, outs)):
        got = o.cpu().numpy()
        ok = b < np.uint64(n_total)
        assert np.array_equal(got[ok], oracle.retrieve(src, b[ok])), r
        assert np.all(got[~ok] == 0x6B)
