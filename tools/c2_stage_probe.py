"""Experiment: config 2 on the one-L2-run plan (path 3) with only the first
X MB of the source staged (dpg_debug_flags (X << 24); X = 0: the direct window
gather), with the bench's protocol (flush before, write-back after).

    python tools/c2_stage_probe.py [--mbs 0,16,32,48,64,80,105]
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_cs_0308004_b200 as dpg  # noqa: E402
from bench import Steps, med  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mbs", default="0,16,32,48,64,80,105")
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
lib = dpg.raw_lib()
lib.dpg_debug_flags.argtypes = [ctypes.c_uint32]
w = datagen.make("c2")
src = torch.from_numpy(w["src"]).cuda()
rids = torch.from_numpy(w["rids"].view(np.int32)).cuda()
out = torch.empty_like(src)
st = Steps(torch, torch.device("cuda", 0))
alg = w["rids"].size * 204
for mb in [int(x) for x in a.mbs.split(",")]:
    flags = (4 if mb == 0 else (mb << 24))
    lib.dpg_debug_flags(flags)
    for _ in range(3):
        dpg.dpg_retrieve(src, rids, dst=out, path=3)
    torch.cuda.synchronize()
    tot, step, wb, _, ph = st.run(lambda: dpg.dpg_retrieve(src, rids, dst=out, path=3), a.steps,
                                  phase_lib=dpg)
    ok = np.array_equal(out[:5000].cpu().numpy(), w["src"][w["rids"][:5000].astype(np.int64)])
    print(f"staged {mb:4d} MB: step {med(tot)*1e3:6.1f} us (kernel {ph[1]*1e3:6.1f} us, frac "
          f"{alg / (ph[1] * 1e-3) / 1e9 / 6544.3:.3f}), write-back {med(wb)*1e3:5.1f} us "
          f"{'ok' if ok else 'BAD'}", flush=True)
lib.dpg_debug_flags(0)
