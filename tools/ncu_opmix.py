"""Opcode mix of one kernel in an ncu report (SASS page): executed warp instructions and stall
samples per opcode.  Usage: python tools/ncu_opmix.py report.ncu-rep [top]"""
import collections
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
ins, smp = collections.Counter(), collections.Counter()
for r in rows:
    if len(r) > 5 and r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    try:
        n = float(r[hdr.index("Instructions Executed")])
        s = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except ValueError:
        continue
    t = r[1].split()
    op = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
    op = ".".join(op.split(".")[:2])
    ins[op] += n
    smp[op] += s
ti, ts = sum(ins.values()), sum(smp.values())
print(f"total {ti/1e6:.1f} M warp instructions, {ts:.0f} stall samples")
for op, n in ins.most_common(top):
    print(f"  {op:22s} {n/1e6:8.1f} M  {100*n/ti:5.1f} %   samples {100*smp[op]/max(ts,1):5.1f} %")
