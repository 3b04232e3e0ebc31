"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel.

  python tools/launch_summary.py launches.csv "<command line that produced it>"
"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, agg = None, collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(
                d.get("Metric Unit", "ns"), 1e-6)
            k = d["Kernel Name"].split("(")[0].replace("void ", "")
            a = agg.setdefault(k, [0.0, 0])
            a[0] += v * scale
            a[1] += 1
    tot = sum(v for v, _ in agg.values()) or 1.0
    print(f"# launch list: ncu --metrics gpu__time_duration.sum --clock-control none --csv {sys.argv[2] if len(sys.argv) > 2 else ''}")
    print("# (cold-cache, serialised per-launch times: compare SHARES)")
    for k, (v, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{k:40s} n={n:4d} total={v:10.3f} ms  mean={v / n:8.3f} ms  share={100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main()
