"""DPG under data skew (section 2.3): times of the plans on skewed
rid lists against the direct gather.  Workload: n_src records of rec bytes,
n_out rids drawn as the paper's exponential keys (datagen.exp_fk),
a hot set (90% of the rids on 1% of the records), floor(n_src u^6) ("zipf":
6% of the rids on record 0) or uniform.  Lines:
  direct       dpg_retrieve_direct
  auto         dpg_retrieve (plan + skew check; path 5 when the sample shows skew)
  p1 / p2      the fused / multi-kernel plan on high-bit runs (path 1 / 2)
  p1g2         path 1 with Fig. 1's INTERNAL file and a Phase III gather (gather=2)
  p6 / p7      the three sequential passes / two DPG levels
  p2r / p2g    path 2 with Phase I as radix passes / global-atomic counting (hist_mode 3 / 2)
  p5           the K L2 runs (path 5)
  bounds       dpg_retrieve_bounds over runs from dpg_skew_partition (the
               partition timed separately: 'part')
L2 flushed before every rep; CUDA events on the current stream; median.

    python tools/skew_probe.py [--n-src 16777216] [--n-out 67108864] [--recs 64,256]
                               [--kinds exp,hot,zipf,uniform] [--runs 1024,8192] [--sample 32768]
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402
import paper_cs_0308004_b200 as dpg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-src", type=int, default=1 << 24)
    ap.add_argument("--n-out", type=int, default=1 << 26)
    ap.add_argument("--recs", default="64,256")
    ap.add_argument("--kinds", default="exp,hot,zipf,uniform")
    ap.add_argument("--runs", default="1024,8192", help="quantile runs asked for")
    ap.add_argument("--sample", type=int, default=32768)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--variants", default="p2,p5", help="of p1,p2,p2r,p5")
    ap.add_argument("--dbg", type=lambda x: int(x, 0), default=0, help="dpg_debug_flags (tuning A/B)")
    args = ap.parse_args()
    lib = dpg.raw_lib()
    lib.dpg_debug_flags.argtypes = [ctypes.c_uint32]
    lib.dpg_debug_flags.restype = None
    lib.dpg_debug_flags(args.dbg)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    flush2 = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    phases = {}

    def timed(fn, name=None):
        ms, ph = [], []
        for _ in range(args.reps):
            flush.fill_(1)
            flush2.view(torch.int32).max()
            if name:
                dpg.dpg_phase_times_ex()
                dpg.dpg_phase_timing(True)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            if name:
                dpg.dpg_phase_timing(False)
                ph.append(dpg.dpg_phase_times_ex()[:3])
            ms.append(a.elapsed_time(b))
        o = sorted(range(len(ms)), key=lambda i: ms[i])[len(ms) // 2]
        if name:
            phases[name] = "/".join(f"{x * 1e3:.0f}" for x in ph[o])
        return ms[o] * 1e3

    n_src, n_out = args.n_src, args.n_out
    rng = np.random.default_rng(0)
    for kind in args.kinds.split(","):
        if kind == "exp":
            h = datagen.exp_fk(n_out, n_src, sid=42)
        elif kind == "hot":
            h = rng.integers(0, n_src, n_out).astype(np.uint32)
            hot = rng.random(n_out) < 0.9
            h[hot] = rng.integers(0, max(1, n_src // 100), int(hot.sum())).astype(np.uint32)
        elif kind == "perm":
            h = rng.permutation(n_src)[:n_out].astype(np.uint32)
        elif kind == "zipf":    # floor(n_src * u^6): 6% of the rids on record 0
            u = rng.random(n_out)
            h = np.minimum(n_src - 1, np.floor(n_src * u ** 6)).astype(np.uint32)
        else:
            h = rng.integers(0, n_src, n_out).astype(np.uint32)
        rids = torch.from_numpy(h.view(np.int32)).cuda()
        for rec in [int(x) for x in args.recs.split(",")]:
            src = torch.empty((n_src, rec), dtype=torch.uint8, device="cuda")
            datagen.random_bytes_cuda(src, sid=41)
            out = torch.empty((n_out, rec), dtype=torch.uint8, device="cuda")
            ref = torch.empty_like(out)
            line = f"{kind:8s} rec {rec:4d}"
            t = timed(lambda: dpg.dpg_retrieve_direct(src, rids, dst=ref))
            line += f"  direct {t:8.1f}"
            t = timed(lambda: dpg.dpg_retrieve(src, rids, dst=out))
            ok = torch.equal(out, ref)
            line += f"  auto(p{dpg.last_path()}) {t:8.1f}{'' if ok else ' MISMATCH'}"
            variants = [("p1", dict(path=1)), ("p1g2", dict(path=1, gather=2)), ("p2", dict(path=2)),
                        ("p2r", dict(path=2, hist_mode=3)), ("p2g", dict(path=2, hist_mode=2)),
                        ("p5", dict(path=5)), ("p6", dict(path=6)), ("p7", dict(path=7))]
            for name, kw in variants:
                if name not in args.variants.split(","):
                    continue
                try:
                    t = timed(lambda: dpg.dpg_retrieve(src, rids, dst=out, **kw), name)
                    ok = torch.equal(out, ref)
                    line += f"  {name} {t:8.1f} [{phases[name]}]{'' if ok else ' MISMATCH'}"
                except dpg.DPGError as e:
                    line += f"  {name} --({e})"
            for K in [int(x) for x in args.runs.split(",") if x]:
                S = max(args.sample, K)
                holder = {}
                t_part = timed(lambda: holder.__setitem__(
                    "b", dpg.dpg_skew_partition(rids, n_src, K, sample_size=S, seed=1)))
                b = holder["b"]
                t = timed(lambda: dpg.dpg_retrieve_bounds(src, rids, b, dst=out), "bounds")
                ok = torch.equal(out, ref)
                line += f"  part {t_part:6.1f} (K {K} -> {b.size - 1}) bounds {t:8.1f}" \
                        f" [{phases['bounds']}]{'' if ok else ' MISMATCH'}"
            print(line, flush=True)
            del src, out, ref


if __name__ == "__main__":
    main()
