"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0]
        k = k.replace("void ", "").replace("stmgb::", "").replace("<unnamed>::", "")[:70]
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        v = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"{'us':>10} {'share':>6} {'n':>5}  kernel")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t:10.1f} {100 * t / tot:5.1f}% {n:5d}  {k}")
    print(f"{tot:10.1f} total us")


if __name__ == "__main__":
    main(sys.argv[1])
