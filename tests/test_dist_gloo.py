"""Multi-process tests of the multi-GPU exchange logic (paper_cs_0308004_b200
/dist.py) on CPU with the gloo backend, world size 2 (and 1).  The local steps
(owner partition, local retrieval, reply gather) are numpy stand-ins here --
test scaffolding for the host logic; on GPUs the same function runs the
libdpg.so kernels (CudaOps).  The result is checked against the oracle of the
global problem."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class NumpyOps:
    """Plain stand-ins of the GPU steps: a stable partition by owner with the
    request position of every row, retrieval, and the gather by position."""

    def partition(self, rids, n_src_total, log2_span, parts):
        r = rids.numpy().astype(np.int64)
        ok = (r >= 0) & (r < n_src_total)
        idx = np.nonzero(ok)[0]
        owner = r[idx] >> log2_span
        order = np.argsort(owner, kind="stable")
        idx = idx[order]
        local = (r[idx] - (owner[order] << log2_span)).astype(np.int32)
        counts = np.bincount(owner, minlength=parts).tolist()
        inv = np.full(r.size, -1, dtype=np.int64)
        inv[idx] = np.arange(idx.size)
        return torch.from_numpy(local), torch.from_numpy(inv.astype(np.int32)), counts

    def empty_u32(self, n, like):
        return torch.empty(n, dtype=torch.int32)

    def empty_rows(self, n, rec, like):
        return torch.zeros((n, rec), dtype=torch.uint8)

    def retrieve(self, src_shard, requests):
        return src_shard[requests.long()].contiguous()

    def gather(self, replies, inv, dst):
        i = inv.long()
        ok = i >= 0
        dst[ok] = replies[i[ok]]

    def counts_tensor(self, counts, like):
        return torch.tensor(counts, dtype=torch.int64)

    # fused exchange: a window is a local byte tensor; the owner's writes into
    # a peer's window are emulated by all-to-alls that carry the rows and the
    # owner-computed row offset, which the receiver honours as given
    def window_alloc(self, nbytes):
        return torch.zeros(max(nbytes, 1), dtype=torch.uint8), b"emulated"

    def window_open(self, handle):
        return None

    def window_close(self, ptr):
        pass

    def window_free(self, ptr):
        pass

    def push(self, src_shard, requests, rcounts, targets, win, group=None):
        world = len(rcounts)
        rec = src_shard.shape[1]
        rows = src_shard[requests.long()].contiguous().view(-1)
        send_n = torch.tensor(rcounts, dtype=torch.int64)
        recv_n = torch.empty(world, dtype=torch.int64)
        dist.all_to_all_single(recv_n, send_n, group=group)
        send_off = torch.tensor([off for _, off in targets], dtype=torch.int64)
        assert [q for q, _ in targets] == list(range(world))
        recv_off = torch.empty(world, dtype=torch.int64)
        dist.all_to_all_single(recv_off, send_off, group=group)
        recv_n = recv_n.tolist()
        got = torch.empty(sum(recv_n) * rec, dtype=torch.uint8)
        dist.all_to_all_single(got, rows, output_split_sizes=[x * rec for x in recv_n],
                               input_split_sizes=[x * rec for x in rcounts], group=group)
        k = 0
        for o in range(world):
            off = int(recv_off[o])
            win.local[off * rec:(off + recv_n[o]) * rec] = got[k:k + recv_n[o] * rec]
            k += recv_n[o] * rec

    def window_barrier(self, like, group=None):
        dist.barrier(group=group)

    def window_gather(self, win, n_rows, inv, dst):
        rec = dst.shape[1]
        self.gather(win.local[:n_rows * rec].view(n_rows, rec), inv, dst)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_total, rec, n_out, seed, round_rows, q, fused=False):
    sys.path.insert(0, ROOT)
    from paper_cs_0308004_b200.dist import owned_range, retrieve_dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        rng = np.random.default_rng(seed)
        src = rng.integers(0, 256, (n_total, rec), dtype=np.uint8)
        rids = rng.integers(0, n_total, n_out).astype(np.int64)
        rids[: min(n_out, n_total)] = rng.permutation(n_total)[: min(n_out, n_total)]
        lo, hi = owned_range(rank, world, n_total)
        b0 = rank * n_out // world
        b1 = (rank + 1) * n_out // world
        out = retrieve_dist(torch.from_numpy(src[lo:hi].copy()), torch.from_numpy(rids[b0:b1].copy()),
                            n_total, ops=NumpyOps(), max_rows_per_round=round_rows, fused=fused)
        q.put((rank, b0, out.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("world,n_total,rec,n_out,round_rows", [
    (2, 1000, 12, 1500, None),      # uneven ranges: rank 1 owns 488 records
    (2, 4096, 100, 4096, 700),      # permutation, several rounds
    (2, 37, 3, 500, 64),            # tiny source, many duplicates
    (1, 300, 7, 450, None),
    (2, 1, 5, 9, None),             # rank 1 owns nothing
])
def test_retrieve_dist_matches_oracle(world, n_total, rec, n_out, round_rows, fused):
    sys.path.insert(0, ROOT)
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker,
                         args=(r, world, port, n_total, rec, n_out, 7, round_rows, q, fused))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = sorted((q.get(timeout=180) for _ in range(world)), key=lambda t: t[0])  # drain, then join
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    got = np.concatenate([o for _, _, o in parts])
    rng = np.random.default_rng(7)
    src = rng.integers(0, 256, (n_total, rec), dtype=np.uint8)
    rids = rng.integers(0, n_total, n_out).astype(np.int64)
    rids[: min(n_out, n_total)] = rng.permutation(n_total)[: min(n_out, n_total)]
    assert np.array_equal(got, oracle.retrieve(src, rids.astype(np.uint64)))


def test_span_and_ranges():
    sys.path.insert(0, ROOT)
    from paper_cs_0308004_b200.dist import owned_range, span_log2
    assert span_log2(1 << 30, 8) == 27
    assert span_log2(1000, 2) == 9
    assert owned_range(1, 2, 1000) == (512, 1000)
    assert owned_range(1, 2, 1) == (1, 1)
    covered = [owned_range(r, 4, 1 << 20) for r in range(4)]
    assert covered[0][0] == 0 and covered[-1][1] == 1 << 20
    assert all(covered[i][1] == covered[i + 1][0] for i in range(3))
