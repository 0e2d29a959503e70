"""Config 4's DPG-Move join on path 6 with each cluster size (0 = the plan's
choice): time and Phase I / II / III (ms).  python tools/join_cluster_probe.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_cs_0308004_b200 as dpg  # noqa: E402

w = datagen.make("c4")
fact = torch.from_numpy(w["fact"]).cuda(); fk = torch.from_numpy(w["fk"].view(np.int32)).cuda(); dim = torch.from_numpy(w["dim"]).cuda()
out = torch.empty((w["fk"].size, 80), dtype=torch.uint8, device="cuda")
ref = torch.empty_like(out)
dpg.dpg_fk_join_direct(fact, fk, dim, out=ref)
fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
def timed(f):
    ms = []
    for _ in range(5):
        fl.fill_(1); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    return sorted(ms)[2]
for cl in (0, 1, 2, 4, 8):
    try:
        dpg.dpg_phase_times_ex(); dpg.dpg_phase_timing(True)
        t = timed(lambda: dpg.dpg_fk_join(fact, fk, dim, out=out, path=6, cluster=cl))
        dpg.dpg_phase_timing(False); ph = dpg.dpg_phase_times_ex()
        print("cluster", cl, round(t, 3), "ms", [round(x / max(1, ph[3]), 3) for x in ph[:3]], torch.equal(out, ref), flush=True)
    except dpg.DPGError as e:
        print("cluster", cl, e)
