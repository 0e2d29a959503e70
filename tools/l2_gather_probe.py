"""Experiment: DPG with the L2 as the cache and one run (K = 1).  Stage the
whole source run into L2 sequentially (bulk L2 prefetch), then probe it in
rid order with sequential output writes.  Compared with the direct gather."""
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_cs_0308004_b200 as dpg  # noqa: E402

flush = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")


def timed(pre, fn, reps=7):
    ms = []
    for _ in range(reps):
        flush.fill_(1)
        if pre:
            pre()
            torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return sorted(ms)[len(ms) // 2] * 1e3


for rec in (100, 64, 128):
    for n in (1 << 18, 1 << 19, 1 << 20, 1 << 21):
        g = torch.Generator(device="cuda")
        g.manual_seed(0)
        src = torch.randint(0, 256, (n, rec), dtype=torch.uint8, device="cuda")
        rids = torch.randperm(n, device="cuda", generator=g).to(torch.int32)
        dst = torch.empty_like(src)
        alg = n * (2 * rec + 4)
        r = {
            "naive": timed(None, lambda: dpg.dpg_retrieve_direct(src, rids, dst=dst)),
            "pf+gather": timed(None, lambda: (dpg.dpg_l2_prefetch(src),
                                              dpg.dpg_retrieve_direct_ex(src, rids, dst=dst, hint=2))),
            "prefetch": timed(None, lambda: dpg.dpg_l2_prefetch(src)),
            "gather|L2": timed(lambda: dpg.dpg_l2_prefetch(src),
                               lambda: dpg.dpg_retrieve_direct_ex(src, rids, dst=dst, hint=2)),
            "gather|L2 h0": timed(lambda: dpg.dpg_l2_prefetch(src),
                                  lambda: dpg.dpg_retrieve_direct_ex(src, rids, dst=dst, hint=0)),
            "dpg": timed(None, lambda: dpg.dpg_retrieve(src, rids, dst=dst)),
        }
        print(f"rec {rec} n {n:8d} ({n*rec/2**20:6.1f} MB) " + "  ".join(
            f"{k} {v:7.1f}us/{alg/v/1e3:5.0f}GB/s" for k, v in r.items()), flush=True)
        del src, dst, rids
