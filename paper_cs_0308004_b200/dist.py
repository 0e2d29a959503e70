"""Multi-GPU DPG record retrieval (BASELINE.json config 5).

One process per GPU.  The source file is range-partitioned: rank r owns
records ``[r*S, (r+1)*S)`` with ``S = 2^log2_span`` (the last ranks may own
fewer, or none).  Output positions are block-partitioned: each rank passes the
rids of its own block of output rows and receives those rows.  The global
result equals the single-GPU retrieval ``D[i] = R[S_rid[i]]`` of the whole
problem (reading A14).

The paper's three phases map onto the cluster:

* Phase I, distribute by owner -- ``dpg_partition_inv``: one run per owner
  (runs of ``S`` records), producing owner-local offsets (requests, owner by
  owner) and, for every output row, the position of its request;
* exchange 1 -- ``all_to_all_single`` of the per-owner counts, then of the
  requests (NCCL over NVLink / NVSwitch);
* Phase II+III on the owner -- the local DPG (``dpg_retrieve``) of the
  requests it received, rows written in request order;
* exchange 2 -- ``all_to_all_single`` of the rows back to the requesters;
* Phase III: ``dst[i] = reply[inv[i]]`` in output order (``dpg_gather_rows``;
  sequential output writes, the replies read as one stream per owner).

Fused exchange (``fused=True``): exchange 2 and the
requester's reply buffer disappear.  Every rank owns a receive window (a CUDA
IPC buffer mapped into every peer process, ``PeerWindows``); after exchange 1
the owner's local DPG writes each requester's replies straight into that
requester's window over NVLink (``dpg_retrieve_segments``: one output
segment per requester, at the offset the requester's count row implies), a
stream-ordered one-word all-reduce orders those writes before the reads, and
Phase III gathers from the window.  The counts travel as one all-gather of
the P x P count matrix (each owner needs every requester's offsets).

Every step on the data runs in libdpg.so kernels (``CudaOps``); this module
only sizes buffers and drives ``torch.distributed``.  The local-step object is
a parameter so the exchange logic can be tested with ``gloo`` on CPU.
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist


def span_log2(n_src_total: int, world: int) -> int:
    """log2 of the records each owner holds: the smallest power of two S with
    world * S >= n_src_total (owner of rid r is r >> log2_span)."""
    per = max(1, -(-n_src_total // world))
    return max(0, math.ceil(math.log2(per)))


def owned_range(rank: int, world: int, n_src_total: int) -> tuple[int, int]:
    """[lo, hi) of the source records rank `rank` owns."""
    s = 1 << span_log2(n_src_total, world)
    lo = min(n_src_total, rank * s)
    return lo, min(n_src_total, lo + s)


class CudaOps:
    """The local steps on the GPU, through the C ABI."""

    def __init__(self):
        import paper_cs_0308004_b200 as dpg
        self.dpg = dpg

    def partition(self, rids, n_src_total, log2_span, parts):
        local, inv, counts = self.dpg.dpg_partition_inv(rids, n_src_total, log2_span, parts)
        counts = [int(c) for c in counts.cpu().tolist()]
        m = sum(counts)
        return local[:m], inv, counts

    def empty_u32(self, n, like):
        return torch.empty(n, dtype=torch.int32, device=like.device)

    def empty_rows(self, n, rec, like):
        return torch.empty((n, rec), dtype=torch.uint8, device=like.device)

    def retrieve(self, src_shard, requests):
        return self.dpg.dpg_retrieve(src_shard, requests)

    def gather(self, replies, inv, dst):
        if inv.numel():
            self.dpg.dpg_gather_rows(replies, inv, dst)

    def counts_tensor(self, counts, like):
        return torch.tensor(counts, dtype=torch.int64, device=like.device)

    # ---- fused exchange: receive windows in peer memory ----
    def window_alloc(self, nbytes):
        return self.dpg.ipc_alloc(max(nbytes, 256))

    def window_open(self, handle):
        return self.dpg.ipc_open(handle)

    def window_close(self, ptr):
        self.dpg.ipc_close(ptr)

    def window_free(self, ptr):
        self.dpg.ipc_free(ptr)

    def push(self, src_shard, requests, rcounts, targets, win, group=None):
        """Owner: the rows of the requests from rank q go to targets[q] =
        (q, row offset in q's window), written into q's memory by the local
        DPG kernels."""
        rec = src_shard.shape[1]
        if requests.numel():
            self.dpg.dpg_retrieve_segments(src_shard, requests, rcounts,
                                           [win.ptrs[q] + off * rec for q, off in targets])

    def window_barrier(self, like, group=None):
        # stream-ordered: every rank's push kernels precede its contribution
        t = torch.zeros(1, dtype=torch.int32, device=like.device)
        dist.all_reduce(t, group=group)

    def window_gather(self, win, n_rows, inv, dst):
        if inv.numel():
            self.dpg.dpg_gather_rows(win.local, inv, dst, n_rows=n_rows)


class PeerWindows:
    """A receive window of ``nbytes`` on every rank, mapped into every peer
    process: ``ptrs[q]`` is rank q's window as seen from this process,
    ``local`` this rank's own."""

    def __init__(self, nbytes: int, group=None, ops=None):
        self.ops = ops or CudaOps()
        self.group = group
        self.me = dist.get_rank(group)
        world = dist.get_world_size(group)
        self.nbytes = nbytes
        self.local, handle = self.ops.window_alloc(nbytes)
        handles = [None] * world
        dist.all_gather_object(handles, handle, group=group)
        self.ptrs = [self.local if q == self.me else self.ops.window_open(handles[q])
                     for q in range(world)]

    def close(self):
        for q, p in enumerate(self.ptrs):
            if q != self.me:
                self.ops.window_close(p)
        self.ops.window_free(self.local)
        self.ptrs = []


def retrieve_dist(src_shard, rids, n_src_total: int, group=None, ops=None,
                  max_rows_per_round: int | None = None, fused: bool = False, windows=None):
    """Rows ``D[i]`` for this rank's block of output positions.

    src_shard: uint8 [hi - lo, rec], the records this rank owns (``owned_range``);
    rids: this rank's block of the global rid sequence (int32/int64, values in
    [0, n_src_total)).  Returns uint8 [len(rids), rec].  ``max_rows_per_round``
    bounds the exchange buffers by cutting the block into rounds.  ``fused``:
    replies written straight into the requesters' windows (``windows``, a
    ``PeerWindows`` of at least the round's rows, created here if omitted)."""
    ops = ops or CudaOps()
    world = dist.get_world_size(group)
    log2_span = span_log2(n_src_total, world)
    rec = src_shard.shape[1]
    n = rids.numel()
    dst = ops.empty_rows(n, rec, src_shard)
    step = max(1, n if not max_rows_per_round else max_rows_per_round)
    # every rank takes part in the same number of rounds (collectives match)
    rounds = ops.counts_tensor([max(1, -(-n // step))], src_shard)
    dist.all_reduce(rounds, op=dist.ReduceOp.MAX, group=group)
    if fused:
        return _retrieve_fused(src_shard, rids, n_src_total, group, ops, step, int(rounds.item()),
                               dst, windows)
    for k in range(int(rounds.item())):
        lo = min(n, k * step)
        hi = min(n, lo + step)
        chunk = rids[lo:hi]
        local, inv, counts = ops.partition(chunk, n_src_total, log2_span, world)
        send_c = ops.counts_tensor(counts, src_shard)
        recv_c = torch.empty_like(send_c)
        dist.all_to_all_single(recv_c, send_c, group=group)
        rcounts = [int(c) for c in recv_c.cpu().tolist()]
        requests = ops.empty_u32(sum(rcounts), src_shard)
        dist.all_to_all_single(requests, local, output_split_sizes=rcounts,
                               input_split_sizes=counts, group=group)
        rows = ops.retrieve(src_shard, requests) if requests.numel() else \
            ops.empty_rows(0, rec, src_shard)
        back = ops.empty_rows(sum(counts), rec, src_shard)
        dist.all_to_all_single(back.view(-1), rows.reshape(-1),
                               output_split_sizes=[c * rec for c in counts],
                               input_split_sizes=[c * rec for c in rcounts], group=group)
        ops.gather(back, inv, dst[lo:hi])
    return dst


def _retrieve_fused(src_shard, rids, n_src_total, group, ops, step, rounds, dst, windows):
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    log2_span = span_log2(n_src_total, world)
    rec = src_shard.shape[1]
    n = rids.numel()
    # every rank receives at most its round's rows: windows of the largest round
    cap = ops.counts_tensor([min(step, n)], src_shard)
    dist.all_reduce(cap, op=dist.ReduceOp.MAX, group=group)
    own = windows is None
    win = windows or PeerWindows(max(1, int(cap.item())) * rec, group=group, ops=ops)
    try:
        for k in range(rounds):
            lo = min(n, k * step)
            hi = min(n, lo + step)
            local, inv, counts = ops.partition(rids[lo:hi], n_src_total, log2_span, world)
            # the count matrix C[q][o] (rows rank q requests from owner o); this
            # collective also orders the previous round's window reads before
            # this round's writes
            c = ops.counts_tensor(counts, src_shard)
            cm = torch.empty(world * world, dtype=c.dtype, device=c.device)
            dist.all_gather_into_tensor(cm, c, group=group)
            cm = [int(x) for x in cm.cpu().tolist()]
            C = [cm[q * world:(q + 1) * world] for q in range(world)]
            rcounts = [C[q][me] for q in range(world)]
            requests = ops.empty_u32(sum(rcounts), src_shard)
            dist.all_to_all_single(requests, local, output_split_sizes=rcounts,
                                   input_split_sizes=counts, group=group)
            # my replies to q start after the rows q requests from owners before me
            targets = [(q, sum(C[q][:me])) for q in range(world)]
            ops.push(src_shard, requests, rcounts, targets, win, group=group)
            ops.window_barrier(src_shard, group=group)
            ops.window_gather(win, sum(counts), inv, dst[lo:hi])
    finally:
        if own:
            ops.window_barrier(src_shard, group=group)   # no peer still writes into it
            win.close()
    return dst
