"""Experiment: the L2-run DPG kernel (path 3) vs the smem-run fused kernel
(path 1) vs the direct gather, L2 flushed before every rep; per-phase times
of path 3 from its %globaltimer stamps.

    python tools/l2run_probe.py [--recs 100,64,128] [--ns 262144,1048576]
"""
import argparse
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_cs_0308004_b200 as dpg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--recs", default="100,64,128")
    ap.add_argument("--ns", default="65536,262144,524288,1048576,1310720")
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--flags", default="0")
    args = ap.parse_args()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    flush2 = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    class F:
        @staticmethod
        def fill_(v):
            flush.fill_(v)                                  # write > L2 ...
            flush2.view(torch.int32).max()                  # ... then read > L2: no dirty lines left
    G = torch.cuda.get_device_properties(0).multi_processor_count
    print("L2 bytes", torch.cuda.get_device_properties(0).L2_cache_size, flush=True)
    ts = torch.zeros(G * 16, dtype=torch.int64, device="cuda")
    lib = dpg.raw_lib()
    lib.dpg_debug_phase_stamps.argtypes = [ctypes.c_void_p]
    lib.dpg_debug_phase_stamps.restype = None
    lib.dpg_debug_flags.argtypes = [ctypes.c_uint32]
    lib.dpg_debug_flags.restype = None
    flags = [int(x, 0) for x in args.flags.split(",")]

    def timed(fn, reps):
        ms = []
        for _ in range(reps):
            F.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        ms.sort()
        return ms[len(ms) // 2] * 1e3

    for rec in [int(x) for x in args.recs.split(",")]:
        for n in [int(x) for x in args.ns.split(",")]:
            g = torch.Generator(device="cuda")
            g.manual_seed(0)
            src = torch.randint(0, 256, (n, rec), dtype=torch.uint8, device="cuda")
            rids = torch.randperm(n, device="cuda", generator=g).to(torch.int32)
            ref = dpg.dpg_retrieve_direct(src, rids)
            out = torch.empty_like(src)
            res = {}
            cands = [("direct", lambda: dpg.dpg_retrieve_direct(src, rids, dst=out))]
            for fl in flags:
                def run(fl=fl):
                    lib.dpg_debug_flags(fl)
                    dpg.dpg_retrieve(src, rids, dst=out, path=3)
                    lib.dpg_debug_flags(0)
                cands.append((f"l2run/{fl}", run))
            if 0 in flags:
                cands.append(("fused", lambda: dpg.dpg_retrieve(src, rids, dst=out, path=1)))
            for name, fn in cands:
                try:
                    out.zero_()
                    fn()
                    torch.cuda.synchronize()
                    okk = bool(torch.equal(out, ref)) or name.startswith("l2run/") and int(name[6:]) & 6
                    res[name] = (timed(fn, args.reps), okk)
                except Exception as e:  # noqa: BLE001
                    res[name] = (float("nan"), str(e)[:40])
            # phase stamps of path 3
            ph = ""
            try:
                F.fill_(1)
                ts.zero_()
                lib.dpg_debug_phase_stamps(ctypes.c_void_p(ts.data_ptr()))
                dpg.dpg_retrieve(src, rids, dst=out, path=3)
                torch.cuda.synchronize()
                lib.dpg_debug_phase_stamps(ctypes.c_void_p(0))
                t = ts.view(G, 16)[:, :4].cpu().double()
                t0 = t[:, 0].min()
                t = (t - t0) / 1e3
                ph = (f"load {t[:, 1].median():6.1f}/{t[:, 1].max():6.1f} barrier-out {t[:, 2].max():6.1f} "
                      f"gather-end {t[:, 3].median():6.1f}/{t[:, 3].max():6.1f}")
            except Exception as e:  # noqa: BLE001
                ph = str(e)[:60]
            alg = n * (2 * rec + 4)
            print(f"rec {rec:4d} n {n:8d} ({n*rec/1e6:7.1f} MB) " + "  ".join(
                f"{k} {v[0]:7.1f}us {alg/v[0]/1e3:5.0f}GB/s {'ok' if v[1] is True else v[1]}"
                for k, v in res.items()) + "  | " + ph, flush=True)
            del src, rids, out, ref


if __name__ == "__main__":
    main()
