"""Top stalled SASS instructions of one kernel in an ncu report, with their dominant stall
reasons.  Usage: python tools/ncu_sass_top.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
items = []
for r in rows:
    if len(r) > 5 and r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    try:
        s = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except ValueError:
        continue
    items.append((s, len(items), r))
tot = sum(i[0] for i in items)
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
order = {idx: r for _, idx, r in items}
for s, idx, r in sorted(items, reverse=True)[:top]:
    reasons = sorted(((float(r[c] or 0), hdr[c]) for c in stall_cols), reverse=True)[:3]
    prev = order.get(idx - 1)
    print(f"{100*s/tot:5.1f}%  {r[1].strip()[:70]:70s} "
          + ", ".join(f"{n[6:]} {int(v)}" for v, n in reasons if v > 0))
    if prev:
        print(f"        (after {prev[1].strip()[:70]})")
