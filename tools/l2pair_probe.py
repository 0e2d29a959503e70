"""Per-phase %globaltimer stamps of the two-L2-run kernels (path 4)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_cs_0308004_b200 as dpg  # noqa: E402

n, rec = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20, 100
g = torch.Generator(device="cuda")
g.manual_seed(0)
src = torch.randint(0, 256, (n, rec), dtype=torch.uint8, device="cuda", generator=g)
rids = torch.randperm(n, device="cuda", generator=g).to(torch.int32)
out = torch.empty_like(src)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
flush2 = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
G = torch.cuda.get_device_properties(0).multi_processor_count
ts = torch.zeros(G * 16, dtype=torch.int64, device="cuda")
lib = dpg.raw_lib()
lib.dpg_debug_phase_stamps.argtypes = [ctypes.c_void_p]
lib.dpg_debug_phase_stamps.restype = None
lib.dpg_debug_flags.argtypes = [ctypes.c_uint32]
lib.dpg_debug_flags.restype = None
for _ in range(3):
    dpg.dpg_retrieve(src, rids, dst=out, path=4)
assert torch.equal(out, src[rids.long()])
for rep in range(6):
    fl = 0
    lib.dpg_debug_flags(fl)
    flush.fill_(1)
    flush2.view(torch.int32).max()
    ts.zero_()
    lib.dpg_debug_phase_stamps(ctypes.c_void_p(ts.data_ptr()))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    dpg.dpg_retrieve(src, rids, dst=out, path=4)
    b.record()
    torch.cuda.synchronize()
    lib.dpg_debug_phase_stamps(ctypes.c_void_p(0))
    t = ts.view(G, 16)[:, :10].cpu().double()
    t = (t - t[:, 0].min()) / 1e3
    names = ["start", "stage0+distribute", "barrier", "probe0->INTERNAL", "stage1", "barrier",
             "gather", "-", "ld", "fence"]
    lib.dpg_debug_flags(0)
    print(f"flags {fl} event {a.elapsed_time(b)*1e3:7.1f}us | " + " | ".join(
        f"{nm} {t[:, k].median():6.1f}/{t[:, k].max():6.1f}" for k, nm in enumerate(names)), flush=True)
