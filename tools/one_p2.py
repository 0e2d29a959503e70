"""One retrieval of the skew-probe shapes (after a warm-up), for ncu captures:
    python tools/one_p2.py [--n-src 16777216] [--n-out 67108864] [--rec 256] [--kind uniform]
                           [--path 2] [--hist-mode 0]"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402
import paper_cs_0308004_b200 as dpg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n-src", type=int, default=1 << 24)
ap.add_argument("--n-out", type=int, default=1 << 26)
ap.add_argument("--rec", type=int, default=256)
ap.add_argument("--kind", default="uniform")
ap.add_argument("--path", type=int, default=2)
ap.add_argument("--hist-mode", type=int, default=0)
a = ap.parse_args()
rng = np.random.default_rng(0)
if a.kind == "exp":
    h = datagen.exp_fk(a.n_out, a.n_src, sid=42)
else:
    h = rng.integers(0, a.n_src, a.n_out).astype(np.uint32)
rids = torch.from_numpy(h.view(np.int32)).cuda()
src = torch.empty((a.n_src, a.rec), dtype=torch.uint8, device="cuda")
datagen.random_bytes_cuda(src, sid=41)
out = torch.empty((a.n_out, a.rec), dtype=torch.uint8, device="cuda")
fn = lambda: dpg.dpg_retrieve(src, rids, dst=out, path=a.path, hist_mode=a.hist_mode)  # noqa: E731
fn()
torch.cuda.synchronize()
fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
fl.fill_(1)
torch.cuda.synchronize()
fn()
torch.cuda.synchronize()
print("ok")
