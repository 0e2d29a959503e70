"""The native multi-GPU exchange's arithmetic (comm.cu `exchange_plan`, through
`dpg_exchange_plan`) driving an exchange on CPU: every requester's rows end up
where the plan puts them, for P = 1..8 ranks simulated in one process and for
two gloo processes exchanging the requests and the replies with all-to-alls at
the plan's offsets.  The local steps here (owner partition, the owner's
retrieval, the gather back) are numpy; checked against the oracle of the
global problem.  No GPU."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


@pytest.fixture(scope="module")
def dpg():
    from tools.buildall import build_dpg
    build_dpg()
    import paper_cs_0308004_b200 as m
    return m


def _partition(rids, span, P):
    """Rows grouped by owner (stable): the requests (owner-local offsets) owner
    by owner, the count per owner, and each row's position in that list."""
    owner = rids // span
    order = np.argsort(owner, kind="stable")
    req = rids[order] - owner[order] * span
    inv = np.empty(rids.size, np.int64)
    inv[order] = np.arange(rids.size)
    return req, np.bincount(owner, minlength=P), inv


def _problem(seed, P, n_total, rec, empty_last=True):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, 256, (n_total, rec), dtype=np.uint8)
    span = -(-n_total // P)
    sizes = rng.integers(1, 3 * n_total // P + 2, P)
    rids = [rng.integers(0, n_total, int(m)) for m in sizes]
    if P > 2 and empty_last:
        rids[-1] = np.zeros(0, np.int64)        # a rank with no rows
    return src, span, rids


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 8])
def test_plan_drives_the_exchange(dpg, P):
    import oracle
    src, span, rids = _problem(P, P, 5000, 7)
    parts = [_partition(r, span, P) for r in rids]
    C = np.zeros((P, P + 1), np.uint64)
    for q in range(P):
        C[q, :P] = parts[q][1]
        C[q, P] = rids[q].size
    plans = [dpg.dpg_exchange_plan(C, me) for me in range(P)]
    windows = [np.full((max(1, int(plans[0]["cap"])), 7), 0xEE, np.uint8) for _ in range(P)]
    for o in range(P):
        x = plans[o]
        # requests: requester q's segment for owner o, at soff_q[o], lands at roff_o[q]
        recv = np.zeros(int(x["n_req"]), np.int64)
        for q in range(P):
            sq = plans[q]["soff"]
            seg = parts[q][0][int(sq[o]):int(sq[o + 1])]
            recv[int(x["roff"][q]):int(x["roff"][q + 1])] = seg
            assert seg.size == int(C[q, o])
        # the owner's replies (its shard's records), requester by requester,
        # written into q's window from win_row_o[q]
        shard = src[o * span:(o + 1) * span]
        rep = shard[recv]
        for q in range(P):
            a, b = int(x["roff"][q]), int(x["roff"][q + 1])
            w = int(x["win_row"][q])
            windows[q][w:w + b - a] = rep[a:b]
    for q in range(P):
        got = windows[q][parts[q][2]] if rids[q].size else np.zeros((0, 7), np.uint8)
        assert np.array_equal(got, oracle.retrieve(src, rids[q].astype(np.uint64))), q


def test_plan_rejects_bad_arguments(dpg):
    C = np.zeros((2, 3), np.uint64)
    with pytest.raises(dpg.DPGError):
        dpg.dpg_exchange_plan(C, 2)
    with pytest.raises(ValueError):
        dpg.dpg_exchange_plan(np.zeros((2, 2), np.uint64), 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import paper_cs_0308004_b200 as dpg
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        src, span, rids = _problem(11, world, 3001, 9, empty_last=False)
        req, cnt, inv = _partition(rids[rank], span, world)
        # the count matrix: one all-gather of each rank's row
        row = torch.tensor(list(cnt) + [rids[rank].size], dtype=torch.int64)
        rows = [torch.zeros(world + 1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(rows, row)
        C = torch.stack(rows).numpy().astype(np.uint64)
        x = dpg.dpg_exchange_plan(C, rank)
        # requests to their owners at the plan's offsets
        recv = torch.zeros(int(x["n_req"]), dtype=torch.int64)
        dist.all_to_all_single(recv, torch.from_numpy(req.astype(np.int64)),
                               output_split_sizes=[int(C[qq, rank]) for qq in range(world)],
                               input_split_sizes=[int(C[rank, o]) for o in range(world)])
        assert np.array_equal(np.diff(x["roff"].astype(np.int64)),
                              [int(C[qq, rank]) for qq in range(world)])
        shard = src[rank * span:(rank + 1) * span]
        rep = torch.from_numpy(shard[recv.numpy()].copy())
        # replies back: the owner's row offset in each requester's window travels
        # with them and must equal the requester's own running count
        wr = torch.from_numpy(x["win_row"].astype(np.int64))
        wrs = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(wrs, wr)
        win = torch.zeros((int(rids[rank].size), 9), dtype=torch.uint8)
        dist.all_to_all_single(win.view(-1), rep.view(-1),
                               output_split_sizes=[int(C[rank, o]) * 9 for o in range(world)],
                               input_split_sizes=[int(C[qq, rank]) * 9 for qq in range(world)])
        starts = np.concatenate([[0], np.cumsum([int(C[rank, o]) for o in range(world)])])[:-1]
        assert [int(wrs[o][rank]) for o in range(world)] == list(starts)
        q.put((rank, win.numpy()[inv] if rids[rank].size else np.zeros((0, 9), np.uint8)))
    finally:
        dist.destroy_process_group()


def test_plan_with_gloo_world_size_2():
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=180) for _ in range(2))
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    src, span, rids = _problem(11, 2, 3001, 9, empty_last=False)
    for r in range(2):
        assert np.array_equal(got[r], oracle.retrieve(src, rids[r].astype(np.uint64))), r
