"""Record-size sweep (BASELINE.json config 3 shape): every retrieval plan on
n random records of rec bytes, rids a permutation (c3a) or uniform with
replacement (c3b); L2 flushed (write then read > L2) before every rep.

    python tools/sweep.py [--n 16777216] [--recs 8,16,32,64,128,256] [--kind perm]
"""
import argparse
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_cs_0308004_b200 as dpg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 24)
    ap.add_argument("--recs", default="8,16,32,64,100,128,256")
    ap.add_argument("--kind", default="perm")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--plans", default="direct,gather,auto,fused1,fused2,multi")
    args = ap.parse_args()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    flush2 = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    lib = dpg.raw_lib()
    lib.dpg_debug_flags.argtypes = [ctypes.c_uint32]
    lib.dpg_debug_flags.restype = None

    def timed(fn):
        ms = []
        for _ in range(args.reps):
            flush.fill_(1)
            flush2.view(torch.int32).max()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        ms.sort()
        return ms[len(ms) // 2] * 1e3

    def gather_nostage(src, rids, out):
        lib.dpg_debug_flags(4)
        try:
            dpg.dpg_retrieve(src, rids, dst=out, path=3)
        finally:
            lib.dpg_debug_flags(0)

    plans = {
        "direct": lambda s, r, o: dpg.dpg_retrieve_direct(s, r, dst=o),
        "gather": gather_nostage,
        "auto": lambda s, r, o: dpg.dpg_retrieve(s, r, dst=o),
        "fused1": lambda s, r, o: dpg.dpg_retrieve(s, r, dst=o, path=1, gather=1),
        "fused2": lambda s, r, o: dpg.dpg_retrieve(s, r, dst=o, path=1, gather=2),
        "multi": lambda s, r, o: dpg.dpg_retrieve(s, r, dst=o, path=2),
    }
    for rec in [int(x) for x in args.recs.split(",")]:
        n = args.n
        g = torch.Generator(device="cuda")
        g.manual_seed(rec)
        src = torch.randint(0, 256, (n, rec), dtype=torch.uint8, device="cuda", generator=g)
        if args.kind == "perm":
            rids = torch.randperm(n, device="cuda", generator=g).to(torch.int32)
        else:
            rids = torch.randint(0, n, (n,), device="cuda", generator=g, dtype=torch.int32)
        ref = src[rids.long()]
        out = torch.empty_like(ref)
        alg = n * (2 * rec + 4)
        row = [f"rec {rec:4d} n {n} {args.kind}"]
        for name in args.plans.split(","):
            try:
                out.zero_()
                plans[name](src, rids, out)
                torch.cuda.synchronize()
                ok = "ok" if torch.equal(out, ref) else "BAD"
                t = timed(lambda: plans[name](src, rids, out))
                row.append(f"{name} {t:8.1f}us {alg / t / 1e3:5.0f}GB/s {ok}")
            except Exception as e:  # noqa: BLE001
                row.append(f"{name} -- {str(e)[:30]}")
        print("  ".join(row), flush=True)
        del src, rids, ref, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
