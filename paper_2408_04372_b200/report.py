"""Run reports in the reference tool's formats (tools/stmg.cpp:17-104):
report.json (report_to_json), probes.csv, sections.csv and the convergence
study's eoc.csv, so tooling written for the reference reads device runs.
Reals in the CSV files use the tool's "%.16e"."""
from __future__ import annotations

import json
import math
import os
from typing import Any, Dict, List, Sequence


def fmt_real(v: float) -> str:
    """fmt_real (tools/stmg.cpp:17-21)."""
    if math.isnan(v):
        return "nan"
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return "%.16e" % v


def report_to_json(run: Dict[str, Any]) -> Dict[str, Any]:
    """report_to_json (tools/stmg.cpp:30-62): the RunReport keys (probe
    series are written to probes.csv, not report.json)."""
    out = {
        "converged": run["converged"],
        "n_space_dofs": run["n_space_dofs"],
        "n_steps_total": run["n_steps_total"],
        "n_batches": run["n_batches"],
        "dofs_global": run["dofs_global"],
        "mean_iterations": run["mean_iterations"],
        "work": run["work"],
        "batches": [{"iterations": b["iterations"], "final_residual": b["final_residual"],
                     "converged": b["converged"]} for b in run["batches"]],
        "hierarchy": [{k: l[k] for k in ("coarsening", "mesh_level", "p", "k", "n_steps", "n_dofs", "omega")}
                      for l in run["hierarchy"]],
        "sections": {k: run["sections"][k] for k in ("total", "smoother", "gmg_wo_smoother", "operator_wo_gmg",
                                                     "other")},
    }
    for key in ("error_u", "error_v"):
        if run.get(key) is not None:
            out[key] = {k: run[key][k] for k in ("l2_l2", "linf_l2", "linf_linf")}
    return out


def dumps(obj: Dict[str, Any]) -> str:
    """nlohmann's dump(2) layout: objects with sorted keys, 2-space indent."""
    return json.dumps(obj, indent=2, sort_keys=True) + "\n"


def write_text(path: str, text: str) -> None:
    try:
        with open(path, "w") as f:
            f.write(text)
    except OSError as e:
        raise RuntimeError(f"cannot write {path}") from e


def write_report(out_dir: str, report: Dict[str, Any]) -> None:
    write_text(os.path.join(out_dir, "report.json"), dumps(report))


def probes_csv(run: Dict[str, Any], n_probes: int) -> str:
    """write_probes (tools/stmg.cpp:69-84)."""
    lines = ["t" + "".join(f",u_probe{i + 1}" for i in range(n_probes))]
    for row, t in enumerate(run["probe_times"]):
        lines.append(fmt_real(t) + "".join("," + fmt_real(col[row]) for col in run["probe_values"]))
    return "\n".join(lines) + "\n"


def write_probes(out_dir: str, run: Dict[str, Any], probes: Sequence) -> None:
    if not probes:
        return
    write_text(os.path.join(out_dir, "probes.csv"), probes_csv(run, len(probes)))


def sections_csv(run: Dict[str, Any]) -> str:
    """write_sections (tools/stmg.cpp:86-104)."""
    s = run["sections"]
    total = s["total"] if s["total"] > 0.0 else 1.0
    rows = [("GMG w/o Smoother", s["gmg_wo_smoother"]), ("Smoother", s["smoother"]),
            ("Operator w/o GMG", s["operator_wo_gmg"]), ("Other", s["other"]), ("Total", s["total"])]
    return "section,seconds,share\n" + "".join(f"{n},{fmt_real(v)},{fmt_real(v / total)}\n" for n, v in rows)


def write_sections(out_dir: str, run: Dict[str, Any]) -> None:
    write_text(os.path.join(out_dir, "sections.csv"), sections_csv(run))


def eoc_csv(runs: List[Dict[str, Any]], refinements: List[int], wave: bool) -> str:
    """eoc.csv of the convergence command (tools/stmg.cpp:157-184)."""
    head = "r,dofs_global,err_l2_l2_u,err_linf_l2_u,err_linf_linf_u"
    if wave:
        head += ",err_l2_l2_v"
    head += ",eoc_l2_l2_u,mean_iterations,work\n"
    out = [head]
    zero = {"l2_l2": 0.0, "linf_l2": 0.0, "linf_linf": 0.0}
    for i, run in enumerate(runs):
        e = run.get("error_u") or zero
        eoc = float("nan")
        prev = runs[i - 1].get("error_u") if i > 0 else None
        if prev is not None and run.get("error_u") is not None and run["error_u"]["l2_l2"] > 0.0:
            eoc = math.log2(prev["l2_l2"] / run["error_u"]["l2_l2"])
        row = f"{refinements[i]},{run['dofs_global']},{fmt_real(e['l2_l2'])},{fmt_real(e['linf_l2'])}," \
              f"{fmt_real(e['linf_linf'])}"
        if wave:
            ev = run.get("error_v")
            row += "," + fmt_real(ev["l2_l2"] if ev is not None else 0.0)
        row += f",{fmt_real(eoc)},{fmt_real(run['mean_iterations'])},{fmt_real(run['work'])}\n"
        out.append(row)
    return "".join(out)
