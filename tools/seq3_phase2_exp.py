"""Tuning experiment: Phase II of path 6 with parts disabled (dpg_debug_flags
bits 0x10000: no RID_RUN loads, 0x20000: no INTERNAL stores; outputs then
wrong).  Times Phase II alone on the c3 shape."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_cs_0308004_b200 as dpg  # noqa: E402

lib = dpg.raw_lib()
lib.dpg_debug_flags.argtypes = [ctypes.c_uint32]
n = 1 << 24
g = torch.Generator(device="cuda")
g.manual_seed(0)
rids = torch.randperm(n, device="cuda", generator=g).to(torch.int32)
fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for rec in (8, 16):
    src = torch.randint(0, 256, (n, rec), dtype=torch.uint8, device="cuda", generator=g)
    out = torch.empty_like(src)
    for flags in (0, 0x10000, 0x20000, 0x30000, 0x70000, 0x40000):
        lib.dpg_debug_flags(flags)
        res = []
        for _ in range(5):
            fl.fill_(1)
            dpg.dpg_phase_times_ex()
            dpg.dpg_phase_timing(True)
            dpg.dpg_retrieve(src, rids, dst=out, path=6)
            torch.cuda.synchronize()
            dpg.dpg_phase_timing(False)
            res.append(dpg.dpg_phase_times_ex())
        res.sort(key=lambda r: r[1])
        r = res[2]
        print(f"rec {rec} flags {flags:#x}: I {r[0]*1e3:.1f} II {r[1]*1e3:.1f} III {r[2]*1e3:.1f} us", flush=True)
    lib.dpg_debug_flags(0)
