"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel launch counts, total and mean device time, and share of the total.
python tools/launch_summary.py launches.csv [--only REGEX]"""
import collections
import csv
import re
import sys


def main():
    path = sys.argv[1]
    only = re.compile(sys.argv[sys.argv.index("--only") + 1]) if "--only" in sys.argv else None
    hdr, agg = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", d["Kernel Name"])[:70]
        if only and not only.search(name):
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3}.get(
            d["Metric Unit"], 1.0)
        e = agg.setdefault(name, [0, 0.0, d["Grid Size"], d["Block Size"]])
        e[0] += 1
        e[1] += float(d["Metric Value"].replace(",", "")) * scale
    tot = sum(e[1] for e in agg.values()) or 1.0
    print(f"{'launches':>8} {'total_us':>11} {'us/launch':>10} {'share':>6}  kernel [grid block]")
    for name, (n, t, g, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n:8d} {t:11.1f} {t / n:10.2f} {t / tot:6.3f}  {name} [{g} {b}]")


if __name__ == "__main__":
    main()
