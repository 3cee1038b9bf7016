"""The counters BASELINE.json's north_star names, per committed ncu report: duration, DRAM
bytes and throughput, sectors per global-load request, L2 hit rate, IPC, warps per SM.
Usage: python tools/ncu_counters.py report.ncu-rep [...]   (prints a markdown table)"""
import csv
import io
import subprocess
import sys

UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12, "usecond": 1e-6,
        "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "ns": 1e-9, "nsecond": 1e-9, "second": 1.0,
        "s": 1.0}


def rows_of(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        yield dict(zip(head, r)), dict(zip(head, units))


def num(d, u, k):
    try:
        return float(d[k].replace(",", "")) * UNIT.get(u.get(k, ""), 1.0)
    except (KeyError, ValueError):
        return float("nan")


print("| report | kernel | us | DRAM read + written (GB) | DRAM TB/s | % of ncu's DRAM peak | sectors / "
      "global-load request | L2 hit % | IPC | warps / SM |")
print("|---|---|---:|---:|---:|---:|---:|---:|---:|---:|")
for path in sys.argv[1:]:
    for d, u in rows_of(path):
        t = num(d, u, "gpu__time_duration.sum")
        rd, wr = num(d, u, "dram__bytes_read.sum"), num(d, u, "dram__bytes_write.sum")
        sec = num(d, u, "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum")
        req = num(d, u, "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum")
        name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "").replace(
            "unnamed>::", "")
        print(f"| `{path.split('/')[-1]}` | `{name[:40]}` | {t * 1e6:.1f} | {rd / 1e9:.3f} + "
              f"{wr / 1e9:.3f} | {(rd + wr) / t / 1e12:.2f} | "
              f"{num(d, u, 'dram__bytes_read.sum.pct_of_peak_sustained_elapsed') + num(d, u, 'dram__bytes_write.sum.pct_of_peak_sustained_elapsed'):.1f} | "
              f"{(sec / req if req else float('nan')):.1f} | "
              f"{num(d, u, 'lts__t_sector_hit_rate.pct'):.1f} | "
              f"{num(d, u, 'sm__inst_executed.avg.per_cycle_active'):.2f} | "
              f"{num(d, u, 'sm__warps_active.avg.per_cycle_active'):.1f} |")
