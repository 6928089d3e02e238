"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`.

python tools/ncu_source_top.py file.csv [kernel_substring] [N]"""
import csv
import sys


def blocks(path):
    rows = list(csv.reader(open(path)))
    cur, name = None, None
    for r in rows:
        if r and r[0] == "Kernel Name":
            if cur:
                yield name, cur
            name, cur = r[1], []
        elif r and r[0] == "Address":
            hdr = r
            cur.append(("H", hdr))
        elif cur is not None:
            cur.append(("D", r))
    if cur:
        yield name, cur


def main():
    path = sys.argv[1]
    want = sys.argv[2] if len(sys.argv) > 2 else ""
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    for name, items in blocks(path):
        if want not in name:
            continue
        hdr = [r for k, r in items if k == "H"][0]
        data = [dict(zip(hdr, r)) for k, r in items if k == "D" and len(r) == len(hdr)]
        samp = lambda d: int(d["Warp Stall Sampling (All Samples)"] or 0)  # noqa: E731
        stalls = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
        tot = sum(samp(d) for d in data)
        agg = {c[6:]: sum(int(d[c] or 0) for d in data) for c in stalls}
        print(f"== {name[:90]}\n   samples {tot}; by reason: " +
              ", ".join(f"{k}={v}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
        for d in sorted(data, key=lambda d: -samp(d))[:n]:
            br = sorted(((int(d[c] or 0), c[6:]) for c in stalls), reverse=True)[:2]
            print(f"   {d['Address'][-5:]} {samp(d):6d} {d['Instructions Executed']:>9} {d['Source'][:64]:64s} {br}")
        break


if __name__ == "__main__":
    main()
