"""Experiment: the path-3 window-gather engine with its run L2-resident
(no staging, no flush: a 3rd call on a warm L2), and with its issue or consume
step switched off (debug bits 20 / 21), to see which half bounds it.

    python tools/engine_probe.py [--n 524288] [--rec 100]
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
    ap.add_argument("--n", type=int, default=524288)
    ap.add_argument("--rec", type=int, default=100)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    lib = dpg.raw_lib()
    lib.dpg_debug_flags.argtypes = [ctypes.c_uint32]
    lib.dpg_debug_flags.restype = None
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    src = torch.randint(0, 256, (a.n, a.rec), dtype=torch.uint8, device="cuda")
    rids = torch.randperm(a.n, device="cuda", generator=g).to(torch.int32)
    out = torch.empty_like(src)
    for name, flags in (("full", 4), ("issue only", 4 | 1 << 20), ("consume only", 4 | 1 << 21),
                        ("neither", 4 | 3 << 20)):
        lib.dpg_debug_flags(flags)
        for _ in range(3):
            dpg.dpg_retrieve(src, rids, dst=out, path=3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(20_000_000)      # the GPU waits while the host queues every call
        e0.record()
        for _ in range(a.reps):
            dpg.dpg_retrieve(src, rids, dst=out, path=3)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / a.reps * 1e3
        print(f"rec {a.rec} n {a.n}: {name:12s} {us:7.1f} us  {a.n / us / 1e3:6.1f} G rows/s")
    lib.dpg_debug_flags(0)


if __name__ == "__main__":
    main()
