"""One DPG-Sort join on config 4 (after a warm-up), for ncu launch lists:
    python tools/one_sortjoin.py [--cfg c4]"""
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
ap.add_argument("--cfg", default="c4")
a = ap.parse_args()
w = datagen.make(a.cfg)
fact = torch.from_numpy(w["fact"]).cuda()
fk = torch.from_numpy(w["fk"].view(np.int32)).cuda()
dim = torch.from_numpy(w["dim"]).cuda()
out = torch.empty((w["fk"].size, 80), dtype=torch.uint8, device="cuda")
for _ in range(2):
    dpg.dpg_fk_join_sort(fact, fk, dim, out=out)
torch.cuda.synchronize()
print("ok")
