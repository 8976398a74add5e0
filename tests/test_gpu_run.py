"""GPU parity of configured runs: the
device march(spec, probes) behind stmg_run against the reference's own
parse_config -> make_problem -> march on the same config (oracle/_ref), and
the CLI's output files.

Bars: per-batch convergence flags equal, GMRES iterations within +-1 of the
reference per batch, the level hierarchy equal (relaxation factors 1e-8),
error norms within 1e-6 relative (they are differences of solutions that
agree to ~1e-10), probe series within 1e-8 of the largest probe value, and
section times that add up to the total."""
import json
import math
import os

import pytest

from paper_2408_04372_b200 import cli
from paper_2408_04372_b200 import run as R

pytestmark = pytest.mark.gpu

RUNS = {
    "heat-dg-2d": {"dim": 2, "p": 2, "k": 1, "refinements": 2, "batch": 2},
    "heat-dg-3d": {"dim": 3, "p": 2, "k": 1, "refinements": 1, "batch": 2, "frequency": 1.0},
    "heat-cgp-3d-perturbed": {"dim": 3, "p": 1, "k": 2, "scheme": "cgp", "refinements": 2, "batch": 4,
                              "perturb": 0.2, "frequency": 0.5},
    "wave-cgp-2d": {"equation": "wave", "scheme": "cgp", "dim": 2, "p": 2, "k": 2, "refinements": 2, "batch": 2},
    "wave-dg-2d": {"equation": "wave", "scheme": "dg", "dim": 2, "p": 3, "k": 1, "refinements": 1, "batch": 4,
                   "frequency": 1.0},
    "shm-2d-probes": {"equation": "wave", "scheme": "cgp", "problem": "shm", "dim": 2, "p": 2, "k": 1,
                      "refinements": 1, "batch": 4, "probe_samples_per_step": 4},
    "zero-rho-random": {"problem": "zero", "dim": 2, "p": 1, "k": 0, "refinements": 2, "batch": 2,
                        "rho_random_lo": 1.0, "rho_random_hi": 100.0, "rel_tol": 1e-10, "abs_tol": 0.0},
    "heat-strategy-nsmooth": {"dim": 2, "p": 2, "k": 2, "refinements": 2, "batch": 4, "n_smooth": 2,
                              "strategy": ["time-k", "space-p", "space-h", "time-tau"],
                              "probes": [[0.3, 0.6], [0.9, 0.1]]},
    "heat-unpreconditioned": {"dim": 2, "p": 1, "k": 1, "refinements": 1, "batch": 2, "precondition": False,
                              "rel_tol": 1e-10, "abs_tol": 0.0},
    "manufactured-rho-random-3d": {"dim": 3, "p": 2, "k": 1, "refinements": 1, "batch": 2, "base_cells": 2,
                                   "rho_random_lo": 0.5, "rho_random_hi": 2.0, "seed": 3},
}


def _close(a, b, rel):
    return abs(a - b) <= rel * max(abs(a), abs(b), 1e-300)


def _compare(ours, theirs):
    assert ours["converged"] == theirs["converged"]
    for key in ("n_space_dofs", "n_steps_total", "n_batches", "dofs_global"):
        assert ours[key] == theirs[key], key
    assert len(ours["batches"]) == len(theirs["batches"])
    for a, b in zip(ours["batches"], theirs["batches"]):
        assert a["converged"] == b["converged"]
        assert abs(a["iterations"] - b["iterations"]) <= 1, (a, b)
    assert len(ours["hierarchy"]) == len(theirs["hierarchy"])
    for a, b in zip(ours["hierarchy"], theirs["hierarchy"]):
        for key in ("coarsening", "mesh_level", "p", "k", "n_steps", "n_dofs"):
            assert a[key] == b[key], (key, a, b)
        assert _close(a["omega"], b["omega"], 1e-8), (a, b)
    for key in ("error_u", "error_v"):
        assert (ours[key] is None) == (key not in theirs), key
        if ours[key] is not None:
            for n in ("l2_l2", "linf_l2", "linf_linf"):
                assert _close(ours[key][n], theirs[key][n], 1e-6), (key, n, ours[key], theirs[key])
    assert len(ours["probe_times"]) == len(theirs["probe_times"])
    for a, b in zip(ours["probe_times"], theirs["probe_times"]):
        assert abs(a - b) <= 1e-14 * max(1.0, abs(b))
    scale = max([abs(v) for col in theirs["probe_values"] for v in col] + [1e-300])
    for ca, cb in zip(ours["probe_values"], theirs["probe_values"]):
        assert len(ca) == len(cb)
        assert max(abs(x - y) for x, y in zip(ca, cb)) <= 1e-8 * scale
    s = ours["sections"]
    assert s["total"] > 0.0 and s["smoother"] >= 0.0 and s["gmg_wo_smoother"] >= 0.0 and s["operator_wo_gmg"] > 0.0
    assert math.isclose(s["smoother"] + s["gmg_wo_smoother"] + s["operator_wo_gmg"] + s["other"], s["total"],
                        rel_tol=1e-12)


@pytest.mark.parametrize("name", list(RUNS))
def test_run_matches_reference_march(cuda, ref, name):
    config = RUNS[name]
    theirs = ref.run_json(config)
    ours = R.solve(config)["runs"][0]
    ours.setdefault("error_u", None)
    ours.setdefault("error_v", None)
    ours.setdefault("probe_times", [])
    ours.setdefault("probe_values", [])
    _compare(ours, theirs)
    if name == "heat-unpreconditioned":
        assert ours["hierarchy"] == [] and ours["sections"]["smoother"] == 0.0


def test_non_converged_batch_stops_the_march(cuda, ref):
    config = {"dim": 2, "p": 2, "k": 1, "refinements": 2, "batch": 2, "max_iters": 2, "restart": 2}
    theirs = ref.run_json(config)
    ours = R.solve(config)["runs"][0]
    assert not theirs["converged"] and not ours["converged"]
    assert len(ours["batches"]) == len(theirs["batches"]) == 1
    assert ours["batches"][0]["iterations"] == theirs["batches"][0]["iterations"] == 2


def test_cli_solve_profile_convergence_write_reports(cuda, tmp_path, capsys):
    cfg_path = tmp_path / "shm.json"
    cfg_path.write_text(json.dumps({"equation": "wave", "scheme": "cgp", "problem": "shm", "dim": 2, "p": 1, "k": 1,
                                    "refinements": 1, "batch": 2}))
    out = tmp_path / "solve"
    assert cli.main(["solve", "--config", str(cfg_path), "--output", str(out)]) == 0
    rep = json.loads((out / "report.json").read_text())
    assert rep["command"] == "solve" and rep["config"]["problem"] == "shm" and rep["runs"][0]["converged"]
    lines = (out / "probes.csv").read_text().splitlines()
    assert lines[0] == "t,u_probe1,u_probe2,u_probe3"
    assert len(lines) == 1 + 1 + rep["runs"][0]["n_steps_total"] * 16
    out = tmp_path / "profile"
    assert cli.main(["--config", str(cfg_path), "profile", "--output", str(out)]) == 0
    rep = json.loads((out / "report.json").read_text())
    assert rep["throughput_dofs_per_second"] > 0.0
    rows = [line.split(",") for line in (out / "sections.csv").read_text().splitlines()[1:]]
    assert [r[0] for r in rows] == ["GMG w/o Smoother", "Smoother", "Operator w/o GMG", "Other", "Total"]
    assert math.isclose(sum(float(r[1]) for r in rows[:4]), float(rows[4][1]), rel_tol=1e-12)
    out = tmp_path / "eoc"
    assert cli.main(["convergence", "--set", "p=2", "--set", "k=1", "--set", "r_min=1", "--set", "r_max=3",
                     "--set", "batch=2", "--set", "frequency=0.5", "--output", str(out)]) == 0
    rows = [line.split(",") for line in (out / "eoc.csv").read_text().splitlines()]
    assert rows[0][:3] == ["r", "dofs_global", "err_l2_l2_u"]
    # dG(1) in time, Q2 in space, h ~ tau: the L2(L2) error falls at ~2nd order or better
    assert float(rows[3][5]) > 1.5
    rep = json.loads((out / "report.json").read_text())
    assert [r["refinement"] for r in rep["runs"]] == [1, 2, 3]
    assert "mean_iters=" in capsys.readouterr().out
    assert not os.path.exists(tmp_path / "eoc" / "probes.csv")
