"""Per-launch DRAM bytes and executed fp64 flops of an ncu --set full report
into profiles/ncu_kernels.json (read by bench.py for roofline.traffic and the
fp64 fraction).

  python scripts/ncu_kernels_json.py REPORT WORKLOAD key=regex [key=regex ...]

Launches of one key that form one logical operation (the interior / boundary
pair of the FDM sweep) are summed per occurrence: the figure stored is
(sum over the key's launches) / (launches of its first kernel name)."""
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rows_of(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        d["_units"] = dict(zip(hdr, units))
        out.append(d)
    return out


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def num(d, k):
    """the value in bytes (byte metrics) or ms (time metrics)"""
    v = d.get(k, "") or "0"
    return float(v.replace(",", "")) * SCALE.get(d["_units"].get(k, ""), 1.0)


def main():
    path, workload = sys.argv[1], sys.argv[2]
    pairs = [a.split("=", 1) for a in sys.argv[3:]]
    rows = rows_of(path)
    dst = os.path.join(ROOT, "profiles", "ncu_kernels.json")
    table = json.load(open(dst)) if os.path.exists(dst) else {}
    for key, rx in pairs:
        sel = [d for d in rows if re.search(rx, d["Kernel Name"])]
        if not sel:
            print(f"{key}: no launch matches {rx}")
            continue
        first = sel[0]["Kernel Name"]
        n = sum(1 for d in sel if d["Kernel Name"] == first)
        dram = sum(num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum") for d in sel) / n
        flops = sum((2 * num(d, "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed")
                     + num(d, "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed")
                     + num(d, "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed"))
                    * num(d, "smsp__cycles_elapsed.avg") for d in sel) / n
        ms = sum(num(d, "gpu__time_duration.sum") for d in sel) / n
        names = sorted({d["Kernel Name"].split("(")[0] for d in sel})
        table[f"{workload}:{key}"] = {"dram_bytes_per_launch": dram, "fp64_flops_per_launch": flops,
                                      "ncu_ms_per_launch": ms, "kernels": names,
                                      "report": os.path.basename(path)}
        print(f"{key}: {dram / 1e9:.3f} GB, {flops / 1e9:.2f} GFLOP, {ms:.3f} ms  {names}")
    with open(dst, "w") as f:
        json.dump(table, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
