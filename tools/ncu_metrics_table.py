"""Tabulate an `ncu --metrics ... --csv` log (one row per kernel launch).

    python tools/ncu_metrics_table.py log.csv [--last N]
"""
import argparse
import csv
import io


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("log")
    ap.add_argument("--last", type=int, default=0, help="only the last N launches")
    a = ap.parse_args()
    lines = [l for l in open(a.log) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    launches, order = {}, []
    for r in rows:
        k = r["ID"]
        if k not in launches:
            launches[k] = {"kernel": r["Kernel Name"]}
            order.append(k)
        launches[k][r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
    if a.last:
        order = order[-a.last:]
    metrics = sorted({m for k in order for m in launches[k] if m != "kernel"})
    print("| id | kernel | " + " | ".join(metrics) + " |")
    print("|---" * (len(metrics) + 2) + "|")
    for k in order:
        L = launches[k]
        vals = [f"{L[m][0]} {L[m][1]}" if m in L else "" for m in metrics]
        print(f"| {k} | {L['kernel'][:60]} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main()
