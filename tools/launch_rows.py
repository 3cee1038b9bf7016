"""Per-launch rows (duration, DRAM read/write) of an ncu --csv metrics log.
Usage: python tools/launch_rows.py gpurun_out/x.csv [--last N]"""
import csv
import sys
from collections import OrderedDict

path = sys.argv[1]
last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else 40
hdr, L = None, OrderedDict()
for r in csv.reader(open(path)):
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        e = L.setdefault(d["ID"], {"name": d["Kernel Name"]})
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
for k, v in list(L.items())[-last:]:
    t = v.get("gpu__time_duration.sum", 0) / 1e3
    rd = v.get("dram__bytes_read.sum", 0) / 1e6
    wr = v.get("dram__bytes_write.sum", 0) / 1e6
    name = v["name"].split("(")[0].split("::")[-1][:28]
    print(f"{k:>4} {name:28s} {t:9.1f} us  read {rd:8.1f} MB  write {wr:8.1f} MB  "
          f"{(rd + wr) / max(t, 1e-9):6.2f} TB/s")
