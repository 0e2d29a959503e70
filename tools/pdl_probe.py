"""A/B of programmatic dependent launch between a plan's kernels: the same
retrieval timed (L2 flushed before each step, CUDA events, no phase events)
with PDL (default) and with the tuning flag 0x40000 (plain launches),
interleaved.  python tools/pdl_probe.py [--cases c3a4,c3a8,...]"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_cs_0308004_b200 as dpg  # noqa: E402

CASES = {"c3a4": (1 << 24, 4, {}), "c3a8": (1 << 24, 8, {}), "c3a16": (1 << 24, 16, {}),
         "c3a32": (1 << 24, 32, {}), "n26r8": (1 << 26, 8, {}), "n26r4": (1 << 26, 4, {}),
         "c3a256": (1 << 24, 256, {}), "c3a128": (1 << 24, 128, {}),
         "c2L": (1 << 24, 100, {}), "c2": (1 << 20, 100, {}), "n23r68": (1 << 23, 68, {}),
         "n24r36": (1 << 24, 36, {})}
ap = argparse.ArgumentParser()
ap.add_argument("--cases", default="c3a4,c3a8,c3a16,c3a32,n26r8,c3a256")
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
lib = dpg.raw_lib()
lib.dpg_debug_flags.argtypes = [ctypes.c_uint32]
fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()


def flush():
    fl.fill_(1)
    fl.view(torch.int32).max()


for name in a.cases.split(","):
    n, rec, opts = CASES[name]
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    src = torch.randint(0, 256, (n, rec), dtype=torch.uint8, device="cuda", generator=g)
    rids = torch.randperm(n, device="cuda", generator=g).to(torch.int32)
    out = torch.empty_like(src)
    want = dpg.dpg_retrieve_direct(src, rids)
    FL = [0, 0x40000]
    res = {f: [] for f in FL}
    for rep in range(3):
        for flag in FL:
            lib.dpg_debug_flags(flag)
            dpg.dpg_retrieve(src, rids, dst=out, **opts)
            torch.cuda.synchronize()
            for _ in range(a.steps):
                flush()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                dpg.dpg_retrieve(src, rids, dst=out, **opts)
                e1.record(st)
                torch.cuda.synchronize()
                res[flag].append(e0.elapsed_time(e1) * 1e3)
            assert torch.equal(out, want), (name, flag)
    lib.dpg_debug_flags(0)
    p = dpg.last_path()
    print(f"{name}: path {p} launches {dpg.last_launch_count()}  " +
          "  ".join(f"{f:#x}: {np.median(res[f]):.1f}" for f in FL) + " us", flush=True)
    del src, rids, out, want
    torch.cuda.empty_cache()
