"""Aggregate an ncu launch-list CSV by kernel: device time per launch (gpu__time_duration.sum) and,
when the capture also has dram__bytes_read.sum / dram__bytes_write.sum, DRAM traffic per launch."""
import collections
import csv
import sys

SCALE_T = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
SCALE_B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    t = collections.defaultdict(lambda: [0, 0.0])
    by = collections.defaultdict(float)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        metric = r[mi] if mi is not None else "gpu__time_duration.sum"
        v = float(r[vi].replace(",", ""))
        name = r[ki].split("(")[0][:70]
        if metric == "gpu__time_duration.sum":
            t[name][0] += 1
            t[name][1] += v * SCALE_T.get(r[ui], 1e-3)
        elif metric.startswith("dram__bytes"):
            by[name] += v * SCALE_B.get(r[ui], 1)
    tot = sum(x for _, x in t.values())
    hdr = f"{'us total':>10} {'share':>6} {'launches':>8} {'avg us':>9}"
    print(hdr + (f" {'MB/launch':>10} {'GB/s':>7}" if by else "") + "  kernel")
    for n, (c, x) in sorted(t.items(), key=lambda kv: -kv[1][1]):
        line = f"{x:10.1f} {100 * x / tot:5.1f}% {c:8d} {x / c:9.1f}"
        if by:
            line += f" {by[n] / c / 1e6:10.1f} {by[n] / (x * 1e-6) / 1e9:7.0f}"
        print(line + f"  {n}")
    print(f"total {tot / 1e3:.3f} ms over {sum(c for c, _ in t.values())} launches (ncu: serialized, cold cache)")


if __name__ == "__main__":
    main(sys.argv[1])
