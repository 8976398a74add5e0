"""Command-line front end with the reference tool's interface
(tools/stmg.cpp:226-314): subcommands `convergence`, `solve` and `profile`;
options --config, --set key=value (repeatable), --output, --threads, --seed
and --dry-run, accepted before or after the subcommand; the same output files
(report.json, eoc.csv, probes.csv, sections.csv) and exit codes (0 ok,
1 not converged or runtime error, 2 configuration error). Every solve runs on
the device through the C ABI (stmg_run).

    python -m paper_2408_04372_b200.cli solve --config run.json --output out
"""
from __future__ import annotations

import argparse
import os
import sys
from typing import List, Optional

from . import config as cfg
from . import native as N
from . import report as rep
from . import run as R


def _version() -> str:
    return N.load().stmg_version().decode()


def _header(command: str, c: cfg.Config) -> dict:
    return {"version": _version(), "command": command, "config": cfg.config_to_dict(c), "runs": []}


def cmd_convergence(c: cfg.Config, out_dir: str, dry_run: bool) -> int:
    """cmd_convergence (tools/stmg.cpp:140-193)."""
    if dry_run:
        sys.stdout.write(cfg.plan_text(c))
        return 0
    if c.r_min > c.r_max:
        raise cfg.ConfigError("convergence: r_min > r_max")
    wave = c.equation == "wave"
    runs, rs = [], []
    for r in range(c.r_min, c.r_max + 1):
        print(f"running r={r} ...", end="", flush=True)
        run = R.run_config(c, r, probes=())
        runs.append(run)
        print(f" mean_iters={run['mean_iterations']:g}" + ("" if run["converged"] else "  [NOT CONVERGED]"))
        rs.append(r)
    os.makedirs(out_dir, exist_ok=True)
    rep.write_text(os.path.join(out_dir, "eoc.csv"), rep.eoc_csv(runs, rs, wave))
    jr = _header("convergence", c)
    for r, run in zip(rs, runs):
        j = rep.report_to_json(run)
        j["refinement"] = r
        jr["runs"].append(j)
    rep.write_report(out_dir, jr)
    return 0 if all(run["converged"] for run in runs) else 1


def cmd_solve(c: cfg.Config, out_dir: str, dry_run: bool) -> int:
    """cmd_solve (tools/stmg.cpp:195-215)."""
    if dry_run:
        sys.stdout.write(cfg.plan_text(c))
        return 0
    probes = cfg.resolve_probes(c)
    run = R.run_config(c, probes=probes)
    os.makedirs(out_dir, exist_ok=True)
    jr = _header("solve", c)
    jr["runs"].append(rep.report_to_json(run))
    rep.write_report(out_dir, jr)
    rep.write_probes(out_dir, run, probes)
    print(f"solve: mean_iters={run['mean_iterations']:g} converged={'yes' if run['converged'] else 'no'}")
    return 0 if run["converged"] else 1


def cmd_profile(c: cfg.Config, out_dir: str, dry_run: bool) -> int:
    """cmd_profile (tools/stmg.cpp:217-248)."""
    if dry_run:
        sys.stdout.write(cfg.plan_text(c))
        return 0
    run = R.run_config(c, probes=())
    os.makedirs(out_dir, exist_ok=True)
    jr = _header("profile", c)
    jr["runs"].append(rep.report_to_json(run))
    s = run["sections"]
    throughput = run["dofs_global"] / s["total"] if s["total"] > 0.0 else 0.0
    jr["throughput_dofs_per_second"] = throughput
    rep.write_report(out_dir, jr)
    rep.write_sections(out_dir, run)
    print(f"profile: total={s['total']:g}s smoother={s['smoother']:g}s gmg_wo_smoother={s['gmg_wo_smoother']:g}s "
          f"operator_wo_gmg={s['operator_wo_gmg']:g}s other={s['other']:g}s throughput={throughput:g} dofs/s")
    return 0 if run["converged"] else 1


def _options(p: argparse.ArgumentParser, suffix: str, default) -> None:
    p.add_argument("--config", dest="config" + suffix, default=default, help="JSON configuration file")
    p.add_argument("--set", dest="set" + suffix, action="append", default=None,
                   help="override a config key (key=value)")
    p.add_argument("--output", dest="output" + suffix, default=default, help="output directory")
    p.add_argument("--threads", dest="threads" + suffix, type=int, default=default, help="worker thread count")
    p.add_argument("--seed", dest="seed" + suffix, type=int, default=default, help="random seed override")
    p.add_argument("--dry-run", dest="dry_run" + suffix, action="store_true", default=False,
                   help="print the multigrid plan, do not solve")


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="stmg",
                                 description="space-time multigrid solver for heat and acoustic wave equations "
                                             "(B200 device path)")
    _options(ap, "", None)
    sub = ap.add_subparsers(dest="command", required=True)
    for name, text in (("convergence", "refinement study with EOC table"), ("solve", "single run"),
                       ("profile", "single run with section timers")):
        _options(sub.add_parser(name, help=text), "_sub", None)
    return ap


def main(argv: Optional[List[str]] = None) -> int:
    try:
        a = _parser().parse_args(argv)
    except SystemExit as e:  # CLI11_PARSE: usage errors exit with a non-zero code
        return int(e.code) if isinstance(e.code, int) else 2
    pick = lambda k: getattr(a, k + "_sub") if getattr(a, k + "_sub") is not None else getattr(a, k)  # noqa: E731
    config_path = pick("config")
    overrides = (a.set or []) + (a.set_sub or [])
    output_dir = pick("output") or "out"
    seed = pick("seed")
    dry_run = a.dry_run or a.dry_run_sub
    try:
        c = cfg.Config()
        if config_path:
            try:
                with open(config_path) as f:
                    text = f.read()
            except OSError:
                raise cfg.ConfigError(f"cannot open config file {config_path}") from None
            c = cfg.parse_config(text)
        for kv in overrides:
            if "=" not in kv:
                raise cfg.ConfigError(f"--set needs key=value, got '{kv}'")
            key, value = kv.split("=", 1)
            c = cfg.apply_override(c, key, value)
        if seed is not None:
            c.seed = seed
    except ValueError as e:
        print(f"configuration error: {e}", file=sys.stderr)
        return 2
    try:
        if a.command == "convergence":
            return cmd_convergence(c, output_dir, dry_run)
        if a.command == "solve":
            return cmd_solve(c, output_dir, dry_run)
        return cmd_profile(c, output_dir, dry_run)
    except ValueError as e:  # invalid_argument (ConfigError, StmgInvalidArgument)
        print(f"configuration error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001 -- runtime_error and friends, as the tool's catch-all
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
