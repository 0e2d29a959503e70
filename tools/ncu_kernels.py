"""Per-kernel headline metrics of an ncu report (every captured launch).

    python tools/ncu_kernels.py report.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "us", 1e-3), ("dram__bytes_read.sum", "MB_rd", 1),
        ("dram__bytes_write.sum", "MB_wr", 1), ("lts__t_requests.sum", "Mreq", 1e-6),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%", 1),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%", 1),
        ("smsp__inst_executed.sum", "Minst", 1e-6),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "Mbankc", 1e-6),
        ("lts__t_sector_hit_rate.pct", "L2hit%", 1)]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    print("| kernel | " + " | ".join(k[1] for k in KEYS) + " |")
    print("|---" * (len(KEYS) + 1) + "|")
    for r in rows[2:]:
        d = dict(zip(h, r))
        vals = []
        for k, _, sc in KEYS:
            try:
                v = float(d.get(k, "nan").replace(",", "")) * sc
                vals.append(f"{v:.1f}")
            except ValueError:
                vals.append("?")
        print(f"| {d.get('Kernel Name', '')[:40]} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main()
