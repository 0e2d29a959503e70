"""Digest of an ncu report: headline metrics, stall reasons, and the CUDA
source lines with the most executed instructions.

    python tools/ncu_digest.py report.ncu-rep [--lines 30]
"""
import argparse
import csv
import io
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--lines", type=int, default=30)
    ap.add_argument("--kernel", default=None, help="regex: only this kernel's launches")
    a = ap.parse_args()
    filt = ["--kernel-name", f"regex:{a.kernel}"] if a.kernel else []
    rows = list(csv.reader(io.StringIO(ncu(a.rep, *filt, "--page", "raw", "--csv"))))
    d = dict(zip(rows[0], rows[2] if len(rows) > 2 else rows[1]))
    for k in KEYS:
        print(f"{k:60s} {d.get(k)}")
    st = [(k, float(v.replace(",", "") or 0)) for k, v in d.items()
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")]
    print("stalls:", ", ".join(f"{k[34:-29]} {v:.2f}" for k, v in sorted(st, key=lambda x: -x[1])[:8]))
    cur, out = None, []
    for r in csv.reader(io.StringIO(ncu(a.rep, *filt, "--page", "source", "--csv", "--print-source", "cuda,sass"))):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) > 8 and r[2] == "-":
            try:
                e, s = int(r[7]), int(r[4])
            except ValueError:
                continue
            if e:
                out.append((e, s, cur, r[0], r[1][:80]))
    print("total executed", sum(x[0] for x in out), "samples", sum(x[1] for x in out))
    for e, s, f, ln, src in sorted(out, reverse=True)[:a.lines]:
        print(f"{e:9d} {s:5d} {f}:{ln} {src}")


if __name__ == "__main__":
    main()
