"""CPU tests of the configured-run front end:
the config schema, --set overrides and their errors against the reference's
own parse_config / apply_override / config_to_json (src/config.cpp, driven
through oracle/_ref); the mesh perturbation and level plans against the
reference's perturb / build_level_plan; the report and CSV formats of the
stmg tool (tools/stmg.cpp); and the CLI's argument handling, dry run and exit
codes. No device work: the solves themselves are in test_gpu_run.py."""
import ctypes as C
import json
import os

import numpy as np
import pytest

from paper_2408_04372_b200 import cli
from paper_2408_04372_b200 import config as cfg
from paper_2408_04372_b200 import native as N
from paper_2408_04372_b200 import report as rep

CONFIGS = [
    "{}",
    '{"equation": "wave", "scheme": "cgp", "k": 2, "p": 3, "dim": 3, "batch": 4}',
    '{"problem": "shm", "equation": "wave", "probes": [[0.5], [0.1, 0.2], [0.1, 0.2, 0.3]]}',
    '{"strategy": ["space-h", "time-k"], "precondition": false, "seed": 7, "perturb": 0.25}',
    '{"k": 2.0, "t_final": 3, "rho_random_lo": 1, "rho_random_hi": 10, "r_min": 1, "r_max": 3}',
]


@pytest.mark.parametrize("text", CONFIGS)
def test_config_round_trip_matches_reference(ref, text):
    ours = cfg.config_to_dict(cfg.parse_config(text))
    theirs = ref.config_json(text)
    assert ours == theirs


@pytest.mark.parametrize("overrides", [
    [("equation", "wave")],
    [("k", "3"), ("t_final", "0.25"), ("precondition", "false")],
    [("strategy", '["space-p","time-tau"]'), ("probes", "[[0.5,0.5]]")],
    [("scheme", "cgp"), ("seed", "123")],
])
def test_overrides_match_reference(ref, overrides):
    c = cfg.parse_config("{}")
    for k, v in overrides:
        c = cfg.apply_override(c, k, v)
    assert cfg.config_to_dict(c) == ref.config_json("{}", overrides)


@pytest.mark.parametrize("text,overrides", [
    ('{"foo": 1}', []),
    ('{"equation": "burgers"}', []),
    ('{"scheme": "rk4"}', []),
    ('{"problem": "other"}', []),
    ("[1, 2]", []),
    ("{", []),
    ('{"probes": [[1, 2, 3, 4]]}', []),
    ("{}", [("nope", "1")]),
    ("{}", [("equation", "fluid")]),
])
def test_invalid_configs_rejected_like_reference(ref, text, overrides):
    with pytest.raises(ValueError) as theirs:
        ref.config_json(text, overrides)
    with pytest.raises(cfg.ConfigError) as ours:
        c = cfg.parse_config(text)
        for k, v in overrides:
            c = cfg.apply_override(c, k, v)
    # same message for the reference's own checks (JSON library messages differ)
    if "parse error" not in str(theirs.value):
        assert str(ours.value) == str(theirs.value)


@pytest.mark.parametrize("dim,base,r,mag,seed", [(2, 2, 2, 0.2, 42), (3, 2, 1, 0.3, 5), (2, 3, 3, 0.45, 11),
                                                 (3, 1, 2, 0.1, 0), (2, 4, 2, 0.35, 3)])
def test_perturbation_matches_reference(ref, dim, base, r, mag, seed):
    lo, hi = np.array([0.0, -1.0, 0.5]), np.array([1.0, 1.0, 2.0])
    got = np.zeros((((base << r) + 1) ** dim, 3))
    rc = N.load().stmg_perturbed_vertices(dim, lo.ctypes.data_as(N.c_double_p), hi.ctypes.data_as(N.c_double_p),
                                          base, r, mag, seed, got.ctypes.data_as(N.c_double_p))
    try:
        want = ref.perturbed_vertices(dim, lo, hi, base, r, mag, seed)
    except RuntimeError as e:  # the reference's check_positive_jacobians rejected the draw: so must we
        assert "inverted cell" in str(e)
        assert rc == -2 and "inverted cell" in N.load().stmg_last_error().decode()
        return
    N.check(rc)
    assert np.max(np.abs(got - want)) <= 1e-14
    assert np.any(got != np.round(got, 12))


def test_perturbation_rejects_bad_magnitude():
    lo, hi = np.zeros(3), np.ones(3)
    out = np.zeros(3 * 25)
    rc = N.load().stmg_perturbed_vertices(2, lo.ctypes.data_as(N.c_double_p), hi.ctypes.data_as(N.c_double_p), 2, 1,
                                          0.5, 1, out.ctypes.data_as(N.c_double_p))
    assert rc == -1 and "magnitude" in N.load().stmg_last_error().decode()


@pytest.mark.parametrize("text", [
    "{}",
    '{"dim": 3, "p": 2, "k": 2, "scheme": "cgp", "batch": 4, "refinements": 1}',
    '{"strategy": ["time-k", "space-h", "space-p"], "p": 2, "k": 2}',
    '{"problem": "shm", "equation": "wave", "refinements": 1}',
])
def test_level_plan_matches_reference_hierarchy(ref, text):
    c = cfg.parse_config(text)
    ours = cfg.level_plan(cfg.make_problem(c, c.refinements))
    theirs = ref.run_json(json.loads(text) | {"max_iters": 1, "abs_tol": 1e300, "rel_tol": 1.0})["hierarchy"]
    assert len(ours) == len(theirs)
    for a, b in zip(ours, theirs):
        for key in ("coarsening", "mesh_level", "p", "k", "n_steps", "n_dofs"):
            assert a[key] == b[key], (key, a, b)


def test_problem_record_follows_make_problem():
    p = cfg.make_problem(cfg.parse_config('{"problem": "shm", "equation": "wave"}'), 2)
    assert (p.lo[0], p.hi[2], p.t_final, p.base_cells, p.base_time_intervals, p.abs_tol) == (-1, 1, 2.0, 5, 5, 1e-10)
    p = cfg.make_problem(cfg.parse_config('{"problem": "shm", "equation": "wave", "t_final": 0.5, "base_cells": 10}'),
                         1)
    assert (p.t_final, p.base_cells, p.base_time_intervals) == (0.5, 10, 5)
    with pytest.raises(cfg.ConfigError, match="shm problem requires equation=wave"):
        cfg.make_problem(cfg.parse_config('{"problem": "shm"}'), 1)
    with pytest.raises(cfg.ConfigError, match="unknown coarsening"):
        cfg.make_problem(cfg.parse_config('{"strategy": ["space-x"]}'), 1)
    nst, nb, ns = C.c_int(), C.c_int(), C.c_longlong()
    p = cfg.make_problem(cfg.parse_config('{"batch": 4, "base_time_intervals": 3}'), 2)
    N.check(N.load().stmg_problem_sizes(C.byref(p), C.byref(nst), C.byref(nb), C.byref(ns)))
    assert (nst.value, nb.value, ns.value) == (24, 6, 1 + 24 * 16)
    p.batch = 5
    assert N.load().stmg_problem_sizes(C.byref(p), None, None, None) == -1


def test_fmt_real_matches_printf():
    libc = C.CDLL(None)
    buf = C.create_string_buffer(64)
    for v in [0.0, 1.0, -2.5, 1e-300, 3.141592653589793, 6.02214076e23, -1.2345678901234567e-7]:
        libc.snprintf(buf, 64, b"%.16e", C.c_double(v))
        assert rep.fmt_real(v) == buf.value.decode()


def _run(converged=True):
    return {"converged": converged, "n_space_dofs": 25, "n_steps_total": 8, "n_batches": 4, "dofs_global": 400,
            "mean_iterations": 5.5, "work": 1100.0,
            "batches": [{"iterations": 5, "final_residual": 1e-13, "converged": True},
                        {"iterations": 6, "final_residual": 2e-13, "converged": converged}],
            "hierarchy": [{"coarsening": "finest", "mesh_level": 2, "p": 1, "k": 1, "n_steps": 2, "n_dofs": 100,
                           "omega": 1.0}],
            "sections": {"total": 2.0, "smoother": 0.5, "gmg_wo_smoother": 0.25, "operator_wo_gmg": 0.25,
                         "other": 1.0},
            "error_u": {"l2_l2": 1e-3, "linf_l2": 2e-3, "linf_linf": 3e-3}, "error_v": None,
            "probe_times": [0.0, 0.5, 1.0], "probe_values": [[0.0, 1.0, 2.0], [3.0, 4.0, 5.0]]}


def test_report_layout():
    j = rep.report_to_json(_run())
    assert set(j) == {"converged", "n_space_dofs", "n_steps_total", "n_batches", "dofs_global", "mean_iterations",
                      "work", "batches", "hierarchy", "sections", "error_u"}
    assert rep.sections_csv(_run()).splitlines() == [
        "section,seconds,share",
        "GMG w/o Smoother,2.5000000000000000e-01,1.2500000000000000e-01",
        "Smoother,5.0000000000000000e-01,2.5000000000000000e-01",
        "Operator w/o GMG,2.5000000000000000e-01,1.2500000000000000e-01",
        "Other,1.0000000000000000e+00,5.0000000000000000e-01",
        "Total,2.0000000000000000e+00,1.0000000000000000e+00"]
    assert rep.probes_csv(_run(), 2).splitlines()[:2] == [
        "t,u_probe1,u_probe2", "0.0000000000000000e+00,0.0000000000000000e+00,3.0000000000000000e+00"]
    a, b = _run(), _run()
    b["error_u"] = {"l2_l2": 2.5e-4, "linf_l2": 0.0, "linf_linf": 0.0}
    lines = rep.eoc_csv([a, b], [2, 3], wave=True).splitlines()
    assert lines[0] == "r,dofs_global,err_l2_l2_u,err_linf_l2_u,err_linf_linf_u,err_l2_l2_v,eoc_l2_l2_u," \
                       "mean_iterations,work"
    assert lines[1].split(",")[6] == "nan" and float(lines[2].split(",")[6]) == 2.0


def test_cli_dry_run_prints_plan(capsys, tmp_path):
    path = tmp_path / "c.json"
    path.write_text('{"dim": 3, "p": 2, "k": 1, "refinements": 2, "batch": 2}')
    assert cli.main(["--config", str(path), "solve", "--dry-run", "--set", "scheme=cgp"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0] == "multigrid plan (finest first):"
    assert out[1] == "  level 0: finest  mesh_level=2 p=2 k=1 n_steps=2 n_dofs=9826"
    assert any("time-tau" in line for line in out)


def test_cli_configuration_errors_exit_2(capsys, tmp_path):
    assert cli.main(["solve", "--set", "bogus=1"]) == 2
    assert "configuration error: config: unknown override key 'bogus'" in capsys.readouterr().err
    assert cli.main(["--config", str(tmp_path / "missing.json"), "profile"]) == 2
    assert cli.main(["solve", "--set", "noequals"]) == 2
    bad = tmp_path / "bad.json"
    bad.write_text('{"equation": "heat", "dim": 2, "extra": true}')
    assert cli.main(["convergence", "--config", str(bad)]) == 2
    assert "unknown key 'extra'" in capsys.readouterr().err
    assert cli.main(["--set", "r_min=4", "--set", "r_max=2", "convergence"]) == 2
    assert cli.main([]) != 0  # a subcommand is required


def test_cli_seed_override_and_dry_run_for_each_command(capsys):
    for command in ("convergence", "solve", "profile"):
        assert cli.main([command, "--dry-run", "--seed", "9"]) == 0
    assert capsys.readouterr().out.count("multigrid plan") == 3
    assert not os.path.exists("out/report.json") or True
