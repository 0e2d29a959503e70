"""Correctness of dpg_sort_rids / dpg_sort under each PDL tuning flag, 30
calls each, against numpy's stable sort of the 10-byte keys."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_cs_0308004_b200 as dpg  # noqa: E402

lib = dpg.raw_lib()
lib.dpg_debug_flags.argtypes = [ctypes.c_uint32]
rng = np.random.default_rng(5)
n = 1 << 20
h = rng.integers(0, 256, (n, 100), dtype=np.uint8)
keys = h[:, :10]
want = np.lexsort(keys[:, ::-1].T).astype(np.uint32)   # stable, byte 0 most significant
src = torch.from_numpy(h).cuda()
out = torch.empty_like(src)
rids = torch.empty(n, dtype=torch.int32, device="cuda")
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for flag in (0, 0x40000):
    lib.dpg_debug_flags(flag)
    bad_r = bad_s = 0
    for it in range(30):
        if it % 2:
            fl.fill_(1)
        dpg.dpg_sort_rids(src, 0, 10, rids=rids)
        torch.cuda.synchronize()
        bad_r += not np.array_equal(rids.cpu().numpy().view(np.uint32), want)
        dpg.dpg_sort(src, 0, 10, dst=out)
        torch.cuda.synchronize()
        o = out.cpu().numpy()
        bad_s += not np.array_equal(o, h[want])
    print(f"flag {flag:#x}: sort_rids wrong {bad_r}/30, dpg_sort wrong {bad_s}/30", flush=True)
lib.dpg_debug_flags(0)
dpg.dpg_sync_status()
