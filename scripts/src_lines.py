"""Per-CUDA-source-line totals (instructions, stall samples) from
`ncu -i X --page source --csv --print-source cuda,sass`."""
import csv
import subprocess
import sys


def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    I = {k: i for i, k in enumerate(hdr)}
    res = []
    for r in rows:
        if len(r) == len(hdr) and r[0] not in ("", "Line No"):
            try:
                res.append((int(r[I["Warp Stall Sampling (All Samples)"]] or 0), int(r[I["Instructions Executed"]] or 0),
                            r[0], r[1][:90]))
            except ValueError:
                pass
    ts = sum(x[0] for x in res) or 1
    ti = sum(x[1] for x in res) or 1
    print(f"{'samp%':>6} {'inst%':>6} line  source")
    for s, i, ln, src in sorted(res, reverse=True)[:top]:
        print(f"{100 * s / ts:6.1f} {100 * i / ti:6.1f} {ln:>5} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
