"""One DPG call on a synthetic permutation (for ncu captures).

    python tools/one_call.py --rec 100 --n 1048576 --path 3 --flags 0 [--direct]
"""
import argparse
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_cs_0308004_b200 as dpg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rec", type=int, default=100)
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--path", type=int, default=0)
ap.add_argument("--flags", type=lambda x: int(x, 0), default=0)
ap.add_argument("--direct", action="store_true")
ap.add_argument("--calls", type=int, default=2)
ap.add_argument("--noflush", action="store_true", help="keep the L2 warm between calls")
a = ap.parse_args()
g = torch.Generator(device="cuda")
g.manual_seed(0)
src = torch.randint(0, 256, (a.n, a.rec), dtype=torch.uint8, device="cuda")
rids = torch.randperm(a.n, device="cuda", generator=g).to(torch.int32)
out = torch.empty_like(src)
lib = dpg.raw_lib()
lib.dpg_debug_flags.argtypes = [ctypes.c_uint32]
lib.dpg_debug_flags.restype = None
lib.dpg_debug_flags(a.flags)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(a.calls):
    if not a.noflush:
        flush.fill_(1)
    if a.direct:
        dpg.dpg_retrieve_direct(src, rids, dst=out)
    else:
        dpg.dpg_retrieve(src, rids, dst=out, path=a.path)
torch.cuda.synchronize()
ref = src[rids.long()]
print("ok" if torch.equal(out, ref) or a.flags & 6 else "MISMATCH")
