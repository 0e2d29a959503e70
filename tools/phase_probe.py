"""Profiling helper: per-CTA phase timeline of the fused DPG kernel from the
%globaltimer stamps it writes when dpg_debug_phase_stamps() is set.

    python tools/phase_probe.py [--config c2] [--reps 5]
"""
import argparse
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--rec", type=int, default=None)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--gather", type=int, default=0)
    ap.add_argument("--n", type=int, default=0, help="synthetic permutation of n records of --rec bytes")
    ap.add_argument("--flags", type=lambda x: int(x, 0), default=0, help="dpg_debug_flags")
    ap.add_argument("--log2-run", type=int, default=0)
    ap.add_argument("--dump", action="store_true", help="per-CTA consume times of the last rep")
    args = ap.parse_args()
    import torch

    import datagen
    import paper_cs_0308004_b200 as dpg
    if args.n:
        g = torch.Generator(device="cuda")
        g.manual_seed(0)
        src = torch.randint(0, 256, (args.n, args.rec or 100), dtype=torch.uint8, device="cuda")
        rids = torch.randperm(args.n, device="cuda", generator=g).to(torch.int32)
    else:
        w = datagen.make(args.config, rec=args.rec) if args.rec else datagen.make(args.config)
        src = torch.from_numpy(w["src"]).cuda()
        rids = torch.from_numpy(w["rids"].view(np.int32)).cuda()
    out = torch.empty((rids.numel(), src.shape[1]), dtype=torch.uint8, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    G = torch.cuda.get_device_properties(0).multi_processor_count
    ts = torch.zeros(G * 16, dtype=torch.int64, device="cuda")
    lib = dpg.raw_lib()
    lib.dpg_debug_phase_stamps.argtypes = [ctypes.c_void_p]
    lib.dpg_debug_phase_stamps.restype = None
    lib.dpg_debug_flags.argtypes = [ctypes.c_uint32]
    lib.dpg_debug_flags.restype = None
    lib.dpg_debug_flags(args.flags)
    for _ in range(3):
        dpg.dpg_retrieve(src, rids, dst=out, log2_run=args.log2_run)
    names = ["init", "distribute", "barrier", "probe", "overflow"]
    for rep in range(args.reps):
        flush.fill_(1)
        ts.zero_()
        lib.dpg_debug_phase_stamps(ctypes.c_void_p(ts.data_ptr()))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dpg.dpg_retrieve(src, rids, dst=out, gather=args.gather, log2_run=args.log2_run)
        e1.record()
        torch.cuda.synchronize()
        lib.dpg_debug_phase_stamps(None)
        t = ts.view(G, 16)[:, :6].cpu().numpy().astype(np.float64)
        t0 = t[:, 0].min()
        rel = (t - t0) / 1e3  # us
        line = [f"event {e0.elapsed_time(e1)*1e3:6.1f}us", f"spread {rel[:,0].max():4.1f}"]
        for k, n in enumerate(names):
            d = rel[:, k + 1] - rel[:, k]
            line.append(f"{n} {np.median(d):5.1f}/{d.max():5.1f} @{rel[:, k+1].max():5.1f}")
        d = (ts.view(G, 16).cpu().numpy().astype(np.float64) - t0) / 1e3
        sub = [("count", 1, 6), ("prefix", 6, 7), ("reserve", 7, 8), ("scatter", 8, 2),
               ("consume", 3, 9), ("tail", 9, 5)]
        line.append("  [" + " ".join(f"{n} {np.median(d[:, b] - d[:, a]):.1f}" for n, a, b in sub) + "]")
        line.append(f"consume-end max @{d[:, 9].max():.1f}")
        print(" | ".join(line))
    if args.dump:
        d = (ts.view(G, 16).cpu().numpy().astype(np.float64) - t0) / 1e3
        order = np.argsort(d[:, 9])
        print("per-CTA [cta: barrier-end consume-end] sorted by consume end:")
        print(" ".join(f"{c}:{d[c, 3]:.0f}-{d[c, 9]:.0f}" for c in order))
    print("plan", dpg.dpg_plan(src.shape[1], src.shape[0], rids.numel(), sm_count=G,
                               log2_run=args.log2_run), "flags", args.flags)


if __name__ == "__main__":
    main()
