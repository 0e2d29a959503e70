"""Phase times of the three sequential passes (path 6) against the direct
gather, on the record-size sweep shape (BASELINE.json config 3: n records of
rec bytes, rids a permutation or uniform with replacement).  L2 flushed
(write then read > L2) before every rep; CUDA events on the current stream.

    python tools/seq3_probe.py [--n 16777216] [--recs 8,16,32,64] [--kind perm|repl]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_cs_0308004_b200 as dpg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 24)
    ap.add_argument("--recs", default="8,16,32,64")
    ap.add_argument("--kinds", default="perm,repl")
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--stage-kb", default="")
    ap.add_argument("--twolevel", action="store_true", help="also time path 7")
    ap.add_argument("--clusters", default="", help="also path 6 with these cluster sizes, e.g. 2,4")
    args = ap.parse_args()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    flush2 = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def timed(fn, phases=False):
        ms, ph = [], []
        for _ in range(args.reps):
            flush.fill_(1)
            flush2.view(torch.int32).max()
            if phases:
                dpg.dpg_phase_times_ex()
                dpg.dpg_phase_timing(True)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            if phases:
                dpg.dpg_phase_timing(False)
                ph.append(dpg.dpg_phase_times_ex()[:3])
            ms.append(a.elapsed_time(b))
        o = sorted(range(len(ms)), key=lambda i: ms[i])[len(ms) // 2]
        return ms[o] * 1e3, ([x * 1e3 for x in ph[o]] if phases else None)

    n = args.n
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    for kind in args.kinds.split(","):
        if kind == "perm":
            rids = torch.randperm(n, device="cuda", generator=g).to(torch.int32)
        else:
            rids = torch.randint(0, n, (n,), device="cuda", generator=g, dtype=torch.int32)
        for rec in [int(x) for x in args.recs.split(",")]:
            src = torch.randint(0, 256, (n, rec), dtype=torch.uint8, device="cuda", generator=g)
            out = torch.empty_like(src)
            want = src[rids.long()]
            alg = n * (2 * rec + 4)
            line = f"rec {rec:4d} {kind}"
            t, _ = timed(lambda: dpg.dpg_retrieve_direct(src, rids, dst=out))
            ok = torch.equal(out, want)
            line += f"  direct {t:8.1f}us {alg / t / 1e3:6.0f}GB/s {'ok' if ok else 'BAD'}"
            out.zero_()
            try:
                t, ph = timed(lambda: dpg.dpg_retrieve(src, rids, dst=out, path=6), phases=True)
                ok = torch.equal(out, want)
                p = dpg.dpg_plan(rec, n, n, path=6)
                line += (f"  seq3 {t:8.1f}us {alg / t / 1e3:6.0f}GB/s {'ok' if ok else 'BAD'}"
                         f" [I {ph[0]:.1f} II {ph[1]:.1f} III {ph[2]:.1f}] K={p['num_runs']}")
            except dpg.DPGError as e:
                line += f"  seq3 -- {e}"
            for nb in (1, 2):
                out.zero_()
                try:
                    t, ph = timed(lambda: dpg.dpg_retrieve(src, rids, dst=out, path=6, gather=nb),
                                  phases=True)
                    ok = torch.equal(out, want)
                    line += (f"  nbuf{nb} {t:7.1f}us {'ok' if ok else 'BAD'}"
                             f" [{ph[0]:.0f}/{ph[1]:.0f}/{ph[2]:.0f}]")
                except dpg.DPGError as e:
                    line += f"  nbuf{nb} -- {e}"
            for cl in [int(x) for x in args.clusters.split(",") if x]:
                out.zero_()
                try:
                    t, ph = timed(lambda: dpg.dpg_retrieve(src, rids, dst=out, path=6, cluster=cl),
                                  phases=True)
                    ok = torch.equal(out, want)
                    line += (f"  cl{cl} {t:7.1f}us {'ok' if ok else 'BAD'}"
                             f" [{ph[0]:.0f}/{ph[1]:.0f}/{ph[2]:.0f}]")
                except dpg.DPGError as e:
                    line += f"  cl{cl} -- {e}"
            if args.twolevel:
                out.zero_()
                try:
                    t, ph = timed(lambda: dpg.dpg_retrieve(src, rids, dst=out, path=7), phases=True)
                    ok = torch.equal(out, want)
                    line += (f"  two-level {t:7.1f}us {'ok' if ok else 'BAD'}"
                             f" [{ph[0]:.0f}/{ph[1]:.0f}/{ph[2]:.0f}]")
                except dpg.DPGError as e:
                    line += f"  two-level -- {e}"
            out.zero_()
            t, _ = timed(lambda: dpg.dpg_retrieve(src, rids, dst=out))
            ok = torch.equal(out, want)
            line += f"  auto(path {dpg.last_path()}) {t:8.1f}us {'ok' if ok else 'BAD'}"
            print(line, flush=True)
            del src, out, want


if __name__ == "__main__":
    main()
