"""Where do the c2 step's ~9 us outside the L2-run kernel go?  Times, after the
bench's L2 flush, (a) the retrieval alone between two events, (b) the same
preceded (inside the events' window, timed separately) by a one-warp path-3
call on a tiny source -- the same kernel, so the same shared-memory carve-out
-- and (c) the kernel duration from the library's own phase events.
    python tools/launch_gap_probe.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_cs_0308004_b200 as dpg  # noqa: E402

n, rec = 1 << 20, 100
g = torch.Generator(device="cuda")
g.manual_seed(0)
src = torch.randint(0, 256, (n, rec), dtype=torch.uint8, device="cuda", generator=g)
rids = torch.randperm(n, device="cuda", generator=g).to(torch.int32)
out = torch.empty_like(src)
tsrc = src[:64].clone()
trids = torch.zeros(32, dtype=torch.int32, device="cuda")
tout = torch.empty((32, rec), dtype=torch.uint8, device="cuda")
fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()


def flush():
    fl.fill_(1)
    fl.sum()


def ev():
    return torch.cuda.Event(enable_timing=True)


def run(mode, steps=30):
    res = []
    for _ in range(steps):
        flush()
        e0, e1, e2 = ev(), ev(), ev()
        if mode == "pre_tiny":
            dpg.dpg_retrieve(tsrc, trids, dst=tout, path=3)
        elif mode == "pre_sleep":
            torch.cuda._sleep(20000)
        e0.record(st)
        if mode == "two_events":
            ev().record(st)
            ev().record(st)
        dpg.dpg_retrieve(src, rids, dst=out)
        e1.record(st)
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(res[5:]))


for m in ("plain", "pre_tiny", "pre_sleep", "two_events", "plain"):
    print(m, round(run(m), 2), "us")
dpg.dpg_phase_timing(True)
print("plain with the library's phase events", round(run("plain"), 2), "us")
dpg.dpg_phase_timing(False)
dpg.dpg_phase_timing(True)
dpg.dpg_phase_times_ex()
run("plain", 20)
a, b, c, calls = dpg.dpg_phase_times_ex()
dpg.dpg_phase_timing(False)
print("phase events: I %.2f II %.2f III %.2f us per call" % (a / calls * 1e3, b / calls * 1e3,
                                                             c / calls * 1e3))
