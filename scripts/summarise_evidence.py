"""Prints the bench line's key figures (gpurun_out/bench.log)."""
import json
import sys

for l in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("step", d["ms_per_step"], "value", d["value"], "frac", d["roofline"]["frac"], d["roofline"]["kernel"],
              "traffic", d["roofline"]["traffic"])
        for k, v in d["kernels"].items():
            print(" ", k, {a: (round(b, 4) if isinstance(b, float) else b) for a, b in v.items()
                           if a in ("ms", "hbm_frac", "streamed_frac")})
        print("e2e", d["e2e"]["value"], d["e2e"]["ms_per_step"], d["e2e"].get("pinned_pipelined", {}).get("ms_per_step"))
        print("solve", d["solve"])
        print("cpu", d.get("cpu_baseline"))
        for c, v in d.get("per_config", {}).items():
            print(c, {k: (round(x["ms"], 3), round(x["hbm_frac"], 3)) for k, x in v["kernels"].items()},
                  v.get("solve", {}).get("iterations"), round(v.get("solve", {}).get("ms", 0), 1))
        print(d["clocks"], d["gpu_launches"])
