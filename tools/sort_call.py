"""One dpg_sort_rids call on config-2-shaped records (for ncu captures)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_cs_0308004_b200 as dpg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
src = torch.randint(0, 256, (n, 100), dtype=torch.uint8, device="cuda")
for _ in range(2):
    r = dpg.dpg_sort_rids(src, 0, 10)
torch.cuda.synchronize()
print("ok", int(r[0]))
