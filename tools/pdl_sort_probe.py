"""A/B of PDL inside dpg_sort (c2's 1 Mi x 100 B records, 10-byte keys):
flags 0 (PDL) and 0x40000 (plain launches), interleaved, L2 flushed."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_cs_0308004_b200 as dpg  # noqa: E402

lib = dpg.raw_lib()
lib.dpg_debug_flags.argtypes = [ctypes.c_uint32]
fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
g = torch.Generator(device="cuda")
g.manual_seed(3)
n = 1 << 20
src = torch.randint(0, 256, (n, 100), dtype=torch.uint8, device="cuda", generator=g)
out = torch.empty_like(src)
rids = torch.empty(n, dtype=torch.int32, device="cuda")
for name, fn in (("dpg_sort", lambda: dpg.dpg_sort(src, 0, 10, dst=out)),
                 ("dpg_sort_rids", lambda: dpg.dpg_sort_rids(src, 0, 10, rids=rids))):
    res = {0: [], 0x40000: []}
    ref = None
    for rep in range(3):
        for flag in res:
            lib.dpg_debug_flags(flag)
            fn()
            torch.cuda.synchronize()
            for _ in range(20):
                fl.fill_(1)
                fl.view(torch.int32).max()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                fn()
                e1.record(st)
                torch.cuda.synchronize()
                res[flag].append(e0.elapsed_time(e1) * 1e3)
            got = (out if name == "dpg_sort" else rids).clone()
            if ref is None:
                ref = got
            assert torch.equal(got, ref), (name, flag)
    lib.dpg_debug_flags(0)
    print(f"{name}: launches {dpg.last_launch_count()}  " +
          "  ".join(f"{f:#x}: {np.median(v):.1f}" for f, v in res.items()) + " us", flush=True)
