"""Per-source-line instruction and stall shares of one kernel in an ncu report.
Usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
f = None
agg, st, src = collections.Counter(), collections.Counter(), {}
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].strip().isdigit():
        continue
    ie = hdr.index("Instructions Executed")
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    num = lambda x: float(x) if x not in ("", "-") else 0.0
    k = (f, int(r[0]))
    try:  # ncu does not escape quotes inside source text: skip rows it mangles
        v, s_ = num(r[ie]), num(r[i_s])
    except ValueError:
        continue
    agg[k] += v
    st[k] += s_
    src[k] = r[1].strip()[:72]
tot = sum(agg.values()) or 1.0
ts = sum(st.values()) or 1.0
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{k[0]:22s}{k[1]:5d} {100 * v / tot:5.1f}% instr {100 * st[k] / ts:5.1f}% stall  {src[k]}")
