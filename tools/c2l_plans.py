"""The automatic plan against forced paths 5 (K L2 runs) and 1 (fused) for
sources beyond the L2 with 36..116-byte records (rids: permutations, L2
flushed, CUDA events, median of 10).
    python tools/c2l_plans.py [--shapes 24:100,25:100,...]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_cs_0308004_b200 as dpg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="23:100,24:100,25:100,24:72,25:48,24:116,26:36,24:52")
ap.add_argument("--variants", default="auto,p1,p5,p2,p6,p3,direct")
ap.add_argument("--fan", type=float, default=1.0,
                help="n_out = fan * n_src; != 1: rids uniform with replacement")
a = ap.parse_args()
fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for sh in a.shapes.split(","):
    lg, rec = map(int, sh.split(":"))
    n = 1 << lg
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    src = torch.randint(0, 256, (n, rec), dtype=torch.uint8, device="cuda", generator=g)
    if a.fan == 1.0:
        rids = torch.randperm(n, device="cuda", generator=g).to(torch.int32)
    else:
        rids = torch.randint(0, n, (max(1, int(n * a.fan)),), device="cuda",
                             generator=g).to(torch.int32)
    out = torch.empty((rids.numel(), rec), dtype=torch.uint8, device="cuda")
    want = dpg.dpg_retrieve_direct(src, rids)
    line = [f"2^{lg} x {rec} B ({n * rec / 2**30:.2f} GiB):"]
    for name, kw in [v for v in (("auto", {}), ("p1", {"path": 1, "gather": 2}),
                                 ("p5", {"path": 5}), ("p2", {"path": 2}), ("p6", {"path": 6}),
                                 ("p3", {"path": 3}), ("direct", None))
                     if v[0] in a.variants.split(",")]:
        fn = (lambda: dpg.dpg_retrieve_direct(src, rids, dst=out)) if kw is None else \
            (lambda kw=kw: dpg.dpg_retrieve(src, rids, dst=out, **kw))
        try:
            fn()
            torch.cuda.synchronize()
        except dpg.DPGError:
            line.append(f"{name} n/a")
            continue
        ts = []
        for _ in range(10):
            fl.fill_(1)
            fl.max()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ok = torch.equal(out, want)
        line.append(f"{name}{'' if kw is None else '(p%d)' % dpg.last_path()} "
                    f"{np.median(ts) * 1000:.0f}{'' if ok else ' WRONG'}")
    print("  ".join(line), flush=True)
    del src, rids, out, want
    torch.cuda.empty_cache()
