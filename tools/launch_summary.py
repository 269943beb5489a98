"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

usage: python tools/launch_summary.py launches.csv [title]
Times are cold-cache and serialised under ncu: compare SHARES, not absolutes.
"""
import csv
import sys
from collections import OrderedDict

SCALE = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    head = rows[0]
    ix = {k: i for i, k in enumerate(head)}
    agg = OrderedDict()
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]]
        ms = float(r[ix["Metric Value"]].replace(",", "")) * SCALE[r[ix["Metric Unit"]]]
        t, n = agg.get(name, (0.0, 0))
        agg[name] = (t + ms, n + 1)
    total = sum(t for t, _ in agg.values())
    if len(sys.argv) > 2:
        print(sys.argv[2])
    print("(ncu, cold-cache and serialised: compare SHARES)\n")
    print(f"{'total ms':>12} {'share':>7} {'launches':>9} {'ms/launch':>10}  kernel")
    for name, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{t:12.3f} {100 * t / total:6.2f}% {n:9d} {t / n:10.4f}  {name[:110]}")


if __name__ == "__main__":
    main()
