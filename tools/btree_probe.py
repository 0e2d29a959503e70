"""Experiment: batch lookup in an enhanced B+-tree, DPG vs the
direct descent, L2 flushed before every rep.

    python tools/btree_probe.py [--keys-log2 24] [--q-log2 26] [--runs 0 20]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_cs_0308004_b200 as dpg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--keys-log2", type=int, nargs="+", default=[24])
    ap.add_argument("--q-log2", type=int, default=26)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--runs", type=int, nargs="*", default=[0])
    a = ap.parse_args()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    flush2 = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for kl in a.keys_log2:
        w = datagen.hash_workload(1 << kl, kl, 1 << a.q_log2)
        levels, rids = datagen.btree_index(w["keys"])
        lv, ln, r = dpg.btree_to_device(levels, rids)
        q = torch.from_numpy(w["queries"].view(np.int32)).cuda()
        out = torch.empty_like(q)
        n = q.numel()
        idx = np.random.default_rng(0).integers(0, n, 4096)
        want = oracle.batch_lookup(w["keys"], w["queries"][idx])
        for name, kw in [("direct", {"direct": True})] + [(f"dpg/{x}", {"log2_run": x}) for x in a.runs]:
            dpg.dpg_btree_lookup(lv, ln, r, q, out=out, **kw)
            torch.cuda.synchronize()
            assert np.array_equal(out.cpu().numpy().view(np.uint32)[idx], want), name
            ms = []
            for _ in range(a.reps):
                flush.fill_(1)
                flush2.view(torch.int32).max()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                dpg.dpg_btree_lookup(lv, ln, r, q, out=out, **kw)
                e1.record()
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
            ms.sort()
            med = ms[len(ms) // 2]
            print(f"keys 2^{kl} ({len(levels)} levels) queries 2^{a.q_log2}: {name:9s} {med:8.3f} ms  "
                  f"{n / med / 1e6:7.2f} G lookups/s", flush=True)


if __name__ == "__main__":
    main()
