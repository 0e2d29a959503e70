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


def retrieve_dist(src_shard, rids, n_src_total: int, group=None, ops=None,
                  max_rows_per_round: int | None = None):
    """Rows ``D[i]`` for this rank's block of output positions.

    src_shard: uint8 [hi - lo, rec], the records this rank owns (``owned_range``);
    rids: this rank's block of the global rid sequence (int32/int64, values in
    [0, n_src_total)).  Returns uint8 [len(rids), rec].  ``max_rows_per_round``
    bounds the exchange buffers by cutting the block into rounds."""
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
