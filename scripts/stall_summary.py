"""Stall-reason totals of one kernel from `ncu -i X --page source --csv --print-source sass`."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
h = rows[hi[0]]
I = {k: i for i, k in enumerate(h)}
body = rows[hi[0] + 1:(hi[1] if len(hi) > 1 else len(rows))]
cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = collections.Counter()
for r in body:
    if len(r) != len(h):
        continue
    for k in cols:
        try:
            tot[k] += int(r[I[k]] or 0)
        except ValueError:
            pass
s = sum(tot.values())
print(" ".join(f"{k[6:]}:{100 * v / s:.0f}%" for k, v in tot.most_common(10)))
