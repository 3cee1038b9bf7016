"""Summarise an ncu --set full report: duration, DRAM traffic, occupancy, stall reasons.
Usage: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram %peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__warps_active.avg.per_cycle_active", "warps/SM"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp instr"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("l1tex__t_bytes.sum", "L1 bytes"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        print(d.get("Kernel Name", "?")[:80])
        for k, name in KEYS:
            if k in d:
                print(f"  {name:12s} {d[k]} {u.get(k, '')}")
        st = []
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith(
                    "_per_issue_active.ratio"):
                try:
                    f = float(v)
                except ValueError:
                    continue
                if f >= 0.05:
                    st.append((f, k[len("smsp__average_warps_issue_stalled_"):-len(
                        "_per_issue_active.ratio")]))
        print("  stalls/issue: " + ", ".join(f"{n} {f:.2f}" for f, n in sorted(st, reverse=True)))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
