"""Summarise an `ncu --page source --csv --print-source sass` export: warp
instructions executed and stall samples per opcode, plus the hottest lines."""
import collections
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {k: i for i, k in enumerate(hdr)}
    ops = collections.Counter()
    st = collections.Counter()
    lines = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        src = r[ix["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        n = float(r[ix["Instructions Executed"]] or 0)
        s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        ops[op] += n
        st[op] += s
        lines.append((s, n, src))
    tot, tots = sum(ops.values()), sum(st.values())
    print(f"{'op':12s} {'inst%':>6s} {'stall%':>6s}")
    for op, n in ops.most_common(top):
        print(f"{op:12s} {100 * n / tot:6.1f} {100 * st[op] / max(tots, 1):6.1f}")
    print(f"total warp inst {tot:.3e}, samples {tots:.0f}")
    print("-- hottest instructions by stall samples")
    for s, n, src in sorted(lines, reverse=True)[:top]:
        print(f"{100 * s / max(tots, 1):5.1f}% {n:10.0f}  {src[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
