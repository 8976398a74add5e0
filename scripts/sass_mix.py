"""Executed-instruction mix and stall samples per SASS opcode of one kernel,
from `ncu -i X --page source --csv --print-source sass > file.csv`."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
h = rows[hi[0]]
I = {k: i for i, k in enumerate(h)}
body = rows[hi[0] + 1:(hi[1] if len(hi) > 1 else len(rows))]
ex, st = collections.Counter(), collections.Counter()
for r in body:
    if len(r) != len(h):
        continue
    op = r[I["Source"]].split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    o = o.split(".")[0]
    try:
        ex[o] += int(r[I["Instructions Executed"]] or 0)
        st[o] += int(r[I["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        pass
te, ts = sum(ex.values()), sum(st.values())
print(f"{'op':10s} {'exec%':>7s} {'stall%':>7s}")
for o, v in ex.most_common(18):
    print(f"{o:10s} {100 * v / te:7.1f} {100 * st[o] / ts:7.1f}")
print("total warp instructions", te)
