"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) as markdown.
Usage: python tools/launch_summary.py launches.csv "command line" > profiles/rNN_launches.md"""
import collections
import csv
import sys


def main(path, cmd):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    head = rows[0]
    ik, iv, iu = head.index("Kernel Name"), head.index("Metric Value"), head.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        v = float(r[iv].replace(",", ""))
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(r[iu], 1e-6)
        name = r[ik].split("(")[0][:90]
        tot[name] += v * scale
        cnt[name] += 1
    all_ms = sum(tot.values())
    print(f"# ncu launch list of `{cmd}`")
    print("# (gpu__time_duration.sum, --clock-control none; cold-cache and serialised: "
          "compare SHARES)")
    print(f"# total kernel time {all_ms:.3f} ms over {sum(cnt.values())} launches\n")
    print("| kernel | launches | total ms | share |")
    print("|---|---:|---:|---:|")
    for name, ms in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| `{name}` | {cnt[name]} | {ms:.3f} | {100 * ms / all_ms:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
