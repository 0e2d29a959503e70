"""Profiling: per-CTA %globaltimer stamps of Phase II (path 6) runs --
start, stage landed, run done -- on the c3 shape.  Prints the average
durations and the stall before the stage lands."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_cs_0308004_b200 as dpg  # noqa: E402

lib = dpg.raw_lib()
lib.dpg_debug_phase_stamps.argtypes = [ctypes.c_void_p]
n = 1 << 24
g = torch.Generator(device="cuda")
g.manual_seed(0)
rids = torch.randperm(n, device="cuda", generator=g).to(torch.int32)
fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for rec in (8, 16):
    src = torch.randint(0, 256, (n, rec), dtype=torch.uint8, device="cuda", generator=g)
    out = torch.empty_like(src)
    ts = torch.zeros(148 * 16 * 4 + 148 * 16 * 2 * 4, dtype=torch.int64, device="cuda")
    dpg.dpg_retrieve(src, rids, dst=out, path=6)
    fl.fill_(1)
    torch.cuda.synchronize()
    lib.dpg_debug_phase_stamps(ts.data_ptr())
    dpg.dpg_retrieve(src, rids, dst=out, path=6)
    torch.cuda.synchronize()
    lib.dpg_debug_phase_stamps(None)
    allts = ts.cpu().numpy().astype("float64")
    t = allts[:148 * 16 * 4].reshape(148, 16, 4)

    t0 = t[:, 0, 0][t[:, 0, 0] > 0].min()
    wait, work, gap = [], [], []
    for c in range(148):
        for r in range(16):
            if t[c, r, 0] == 0:
                continue
            wait.append(t[c, r, 1] - t[c, r, 0])
            work.append(t[c, r, 2] - t[c, r, 1])
    end = t[:, :, 2].max() - t0
    import numpy as np
    print(f"rec {rec}: phase II span {end/1e3:.1f} us; per run: stage wait {np.mean(wait)/1e3:.2f} us "
          f"(max {np.max(wait)/1e3:.2f}), work {np.mean(work)/1e3:.2f} us (max {np.max(work)/1e3:.2f}); "
          f"runs/CTA {len(wait)/148:.1f}", flush=True)
    print("  CTA 0:", [(round((t[0, r, 1]-t[0, r, 0])/1e3, 2), round((t[0, r, 2]-t[0, r, 1])/1e3, 2)) for r in range(16) if t[0, r, 0]])
