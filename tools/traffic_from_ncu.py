"""Record the DRAM traffic of one profiled sweep launch in profiles/traffic.json (read by
bench.py for roofline.traffic).  Usage:
  python tools/traffic_from_ncu.py report.ncu-rep config1_broadcast ALGO_BYTES [dest]"""
import csv
import io
import json
import subprocess
import sys


def main(rep, key, algo, dest="profiles/traffic.json"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    d = dict(zip(rows[0], rows[2]))
    units = dict(zip(rows[0], rows[1]))

    def val(k):
        v = float(d[k].replace(",", ""))
        u = units.get(k, "")
        return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12,
                    "msecond": 1e-3, "usecond": 1e-6, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "nsecond": 1e-9, "second": 1.0}.get(u, 1.0)

    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    try:
        tr = json.load(open(dest))
    except OSError:
        tr = {}
    tr[key] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
               "duration_s": val("gpu__time_duration.sum"), "algorithmic_bytes": int(algo),
               "kernel": d.get("Kernel Name", "")[:80],
               "source": f"{rep} (ncu --set full, one launch)"}
    json.dump(tr, open(dest, "w"), indent=1)
    print(key, tr[key])


if __name__ == "__main__":
    main(*sys.argv[1:])
