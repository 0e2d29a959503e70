"""One retrieval (after a warm-up) on the c3 shape, for ncu captures:
    python tools/one_seq3.py --rec 8 [--n 16777216] [--kind perm] [--path 6] [--hist-mode 3]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_cs_0308004_b200 as dpg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 24)
ap.add_argument("--rec", type=int, default=8)
ap.add_argument("--kind", default="perm")
ap.add_argument("--path", type=int, default=6)
ap.add_argument("--direct", action="store_true")
ap.add_argument("--hist-mode", type=int, default=0)
a = ap.parse_args()
g = torch.Generator(device="cuda")
g.manual_seed(0)
n = a.n
rids = (torch.randperm(n, device="cuda", generator=g) if a.kind == "perm"
        else torch.randint(0, n, (n,), device="cuda", generator=g)).to(torch.int32)
src = torch.randint(0, 256, (n, a.rec), dtype=torch.uint8, device="cuda", generator=g)
out = torch.empty_like(src)
fn = (lambda: dpg.dpg_retrieve_direct(src, rids, dst=out)) if a.direct else \
    (lambda: dpg.dpg_retrieve(src, rids, dst=out, path=a.path, hist_mode=a.hist_mode))
fn()
torch.cuda.synchronize()
fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
fl.fill_(1)
torch.cuda.synchronize()
fn()
torch.cuda.synchronize()
assert torch.equal(out, src[rids.long()])
print("ok")
