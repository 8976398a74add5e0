"""Executed fp64 flops of one kernel launch from its ncu SASS source page
(`ncu -i X --page source --csv --print-source sass`): predicated-on thread
instructions, DFMA = 2 flops, DADD / DMUL = 1 (division / rcp sequences are
counted by their DFMA/DMUL steps)."""
import csv
import sys


def flops(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    h = rows[hi[0]]
    I = {k: i for i, k in enumerate(h)}
    body = rows[hi[0] + 1:(hi[1] if len(hi) > 1 else len(rows))]
    tot = {"DFMA": 0, "DADD": 0, "DMUL": 0}
    for r in body:
        if len(r) != len(h):
            continue
        op = r[I["Source"]].split()
        if not op:
            continue
        o = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
        if o in tot:
            tot[o] += int(r[I["Predicated-On Thread Instructions Executed"]] or 0)
    return 2 * tot["DFMA"] + tot["DADD"] + tot["DMUL"], tot


if __name__ == "__main__":
    f, t = flops(sys.argv[1])
    print(f"executed fp64 flops {f:.4e}  ({t})")
