"""Aggregate an ncu launch-list CSV (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)
        name = r[ki].split("(")[0][:70]
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    print(f"{'us total':>10} {'share':>6} {'launches':>8} {'avg us':>9}  kernel")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t:10.1f} {100 * t / tot:5.1f}% {c:8d} {t / c:9.1f}  {n}")
    print(f"total {tot / 1e3:.3f} ms over {sum(c for c, _ in agg.values())} launches (ncu: serialized, cold cache)")


if __name__ == "__main__":
    main(sys.argv[1])
