"""Microbenchmark: what do random record-granular reads and writes cost on
this GPU's HBM?  (The paper's premise: random access pays DRAM
page switches and whole-block over-fetch.)  Times, with L2 flushed before
each rep:
  copy     : torch copy_ of n*rec bytes (sequential read + write)
  gather   : dpg_retrieve_direct  dst[i] = src[perm[i]]   (random reads)
  scatter  : dpg_scatter_rows     dst[perm[k]] = rows[k]  (random writes)
  dpg      : dpg_retrieve          (sequential source runs, random writes)
Reports GB/s counting 2*n*rec (+4n for the index) bytes.

    python tools/access_bench.py [--total-mb 1024]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--total-mb", type=int, default=1024)
    ap.add_argument("--recs", default="8,16,32,64,100,128,256,512,1024,4096")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch

    import paper_cs_0308004_b200 as dpg
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def t(fn):
        fn()
        ms = []
        for _ in range(args.reps):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        return sorted(ms)[len(ms) // 2]

    for rec in [int(x) for x in args.recs.split(",")]:
        n = (args.total_mb << 20) // rec
        g = torch.Generator(device="cuda")
        g.manual_seed(0)
        src = torch.randint(0, 256, (n, rec), dtype=torch.uint8, device="cuda")
        perm = torch.randperm(n, device="cuda", generator=g).to(torch.int32)
        dst = torch.empty_like(src)
        nb = 2 * n * rec + 4 * n
        res = {"copy": t(lambda: dst.copy_(src)),
               "gather": t(lambda: dpg.dpg_retrieve_direct(src, perm, dst=dst)),
               "scatter": t(lambda: dpg.dpg_scatter_rows(src, perm, dst)),
               "dpg": t(lambda: dpg.dpg_retrieve(src, perm, dst=dst))}
        plan = dpg.dpg_plan(rec, n, n, sm_count=torch.cuda.get_device_properties(0).multi_processor_count)
        print(f"rec {rec:5d} n {n:10d} " + " ".join(
            f"{k} {v*1e3:8.1f}us {nb/(v*1e-3)/1e9:7.0f}GB/s" for k, v in res.items())
            + f"  [dpg path {plan['path']} L {plan['run_len']}]", flush=True)
        del src, dst, perm


if __name__ == "__main__":
    main()
