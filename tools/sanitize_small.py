"""Small calls of the round-2 kernels for compute-sanitizer (memcheck,
racecheck, synccheck): path 2 with radix Phase I and work items, the skew
partition, boundary runs, path 6, the key sort.
    compute-sanitizer --tool memcheck python tools/sanitize_small.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_cs_0308004_b200 as dpg  # noqa: E402


def dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).cuda()


rng = np.random.default_rng(1)
n_src, rec, n = 20000, 24, 50000
src = rng.integers(0, 256, (n_src, rec), dtype=np.uint8)
rids = rng.integers(0, n_src, n).astype(np.uint32)
rids[:5000] = 7                                   # a heavy run
want = src[rids]
S, R = dev(src), dev(rids)
for kw in (dict(path=2, hist_mode=3, log2_run=3), dict(path=2, log2_run=4), dict(path=6, log2_run=6),
           dict(path=1, log2_run=5)):
    got = dpg.dpg_retrieve(S, R, **kw).cpu().numpy()
    assert np.array_equal(got, want), kw
# path 6 with 4-byte records and a tile shrunk for two Phase I CTAs per SM
s4 = rng.integers(0, 256, (300000, 4), dtype=np.uint8)
r4 = rng.permutation(300000).astype(np.uint32)
assert dpg.dpg_plan(4, 300000, 300000, path=6, log2_run=9)["tile"] < 18768
got = dpg.dpg_retrieve(dev(s4), dev(r4), path=6, log2_run=9).cpu().numpy()
assert np.array_equal(got, s4[r4])
b = dpg.dpg_skew_partition(R, n_src, 64, sample_size=4096, seed=3)
got = dpg.dpg_retrieve_bounds(S, R, b).cpu().numpy()
assert np.array_equal(got, want)
keys = rng.integers(0, 256, (30000, 16), dtype=np.uint8)
order = dpg.dpg_sort_rids(dev(keys), 0, 10) if hasattr(dpg, "dpg_sort_rids") else None
torch.cuda.synchronize()
dpg.dpg_sync_status()
print("ok")
