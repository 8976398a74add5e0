"""Configured runs on the device: march(spec, probes) behind the C ABI
(stmg_run), and the reference's Python entry points over it
(proj/python/stmg/__init__.py, proj/python/module.cpp:81-132): solve(),
convergence() and temporal_weights() with dict configs and dict reports."""
from __future__ import annotations

import ctypes as C
from typing import Any, Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import config as cfg
from . import native as N
from . import report as rep


def march(problem: N.Problem, probes: Sequence[Tuple[float, float, float]] = ()) -> Dict[str, Any]:
    """One run of a resolved problem: the RunReport fields as a dict, with the
    probe series (probe_times, probe_values per probe)."""
    lib = N.load()
    n_steps_total, n_batches, n_samples = C.c_int(0), C.c_int(0), C.c_longlong(0)
    N.check(lib.stmg_problem_sizes(C.byref(problem), C.byref(n_steps_total), C.byref(n_batches),
                                   C.byref(n_samples)))
    nb = n_batches.value
    npb = len(probes)
    ns = n_samples.value if npb else 0
    it = np.zeros(nb, dtype=np.int32)
    res = np.zeros(nb)
    conv = np.zeros(nb, dtype=np.int32)
    cap_l = 64
    lints = np.zeros(5 * cap_l, dtype=np.int32)
    ldofs = np.zeros(cap_l, dtype=np.int64)
    lomega = np.zeros(cap_l)
    xyz = np.ascontiguousarray(np.asarray(probes, dtype=np.float64).reshape(-1)) if npb else np.zeros(3)
    ptimes = np.zeros(max(ns, 1))
    pvals = np.zeros(max(ns * npb, 1))
    r = N.RunReport()
    ip = lambda a: a.ctypes.data_as(N.c_int_p)  # noqa: E731
    dp = lambda a: a.ctypes.data_as(N.c_double_p)  # noqa: E731
    N.check(lib.stmg_run(C.byref(problem), npb, dp(xyz), C.byref(r), nb, ip(it), dp(res), ip(conv), cap_l, ip(lints),
                         ldofs.ctypes.data_as(N.c_ll_p), dp(lomega), ns, dp(ptimes), dp(pvals)))
    nrun = r.n_batches_run
    hierarchy = []
    for l in range(min(r.n_levels, cap_l)):
        code, ml, pp, kk, nst = (int(x) for x in lints[5 * l:5 * l + 5])
        hierarchy.append({"coarsening": "finest" if code < 0 else cfg.COARSENINGS[code], "mesh_level": ml, "p": pp,
                          "k": kk, "n_steps": nst, "n_dofs": int(ldofs[l]), "omega": float(lomega[l])})
    err = lambda a: {"l2_l2": a[0], "linf_l2": a[1], "linf_linf": a[2]}  # noqa: E731
    nsr = int(r.n_probe_samples) if npb else 0
    return {
        "converged": bool(r.converged),
        "n_space_dofs": int(r.n_space_dofs),
        "n_steps_total": int(r.n_steps_total),
        "n_batches": int(r.n_batches),
        "dofs_global": int(r.dofs_global),
        "mean_iterations": float(r.mean_iterations),
        "work": float(r.work),
        "batches": [{"iterations": int(it[b]), "final_residual": float(res[b]), "converged": bool(conv[b])}
                    for b in range(nrun)],
        "hierarchy": hierarchy,
        "sections": dict(zip(("total", "smoother", "gmg_wo_smoother", "operator_wo_gmg", "other"),
                             (float(x) for x in r.sections))),
        "error_u": err(list(r.error_u)) if r.has_error_u else None,
        "error_v": err(list(r.error_v)) if r.has_error_v else None,
        "probe_times": [float(t) for t in ptimes[:nsr]],
        "probe_values": [[float(v) for v in pvals[p * ns:p * ns + nsr]] for p in range(npb)],
    }


def run_config(c: cfg.Config, refinement: Optional[int] = None, probes: Optional[Sequence] = None) -> Dict[str, Any]:
    r = c.refinements if refinement is None else refinement
    return march(cfg.make_problem(c, r), cfg.resolve_probes(c) if probes is None else probes)


def _with_probes(run: Dict[str, Any]) -> Dict[str, Any]:
    j = rep.report_to_json(run)
    if run["probe_times"]:
        j["probe_times"] = run["probe_times"]
        j["probe_values"] = run["probe_values"]
    return j


def solve(config: Optional[Dict[str, Any]] = None, **overrides) -> Dict[str, Any]:
    """Single run at config.refinements; the report dict (module.cpp:96-110)."""
    c = cfg.merge(config, overrides)
    run = run_config(c)
    return {"command": "solve", "config": cfg.config_to_dict(c), "runs": [_with_probes(run)]}


def convergence(config: Optional[Dict[str, Any]] = None, **overrides) -> Dict[str, Any]:
    """Refinement study over r_min..r_max (module.cpp:112-130)."""
    c = cfg.merge(config, overrides)
    if c.r_min > c.r_max:
        raise cfg.ConfigError("convergence: r_min > r_max")
    runs: List[Dict[str, Any]] = []
    for r in range(c.r_min, c.r_max + 1):
        j = rep.report_to_json(run_config(c, r, probes=()))
        j["refinement"] = r
        runs.append(j)
    return {"command": "convergence", "config": cfg.config_to_dict(c), "runs": runs}


def temporal_weights(scheme: str, k: int) -> Dict[str, Any]:
    """Temporal weight matrices of DG(k) or CGP(k) on the unit interval
    (module.cpp:65-79, 84-94)."""
    if scheme not in cfg.SCHEMES:
        raise ValueError("scheme must be 'dg' or 'cgp'")
    sch = cfg.SCHEMES.index(scheme)
    nt = k + 1 if sch == 0 else k
    if nt < 1:
        raise ValueError("temporal_weights: invalid k")
    m, a = np.zeros(nt * nt), np.zeros(nt * nt)
    alpha, beta, nodes = np.zeros(nt), np.zeros(nt), np.zeros(nt)
    dp = lambda x: x.ctypes.data_as(N.c_double_p)  # noqa: E731
    N.check(N.load().stmg_temporal_weights(sch, k, dp(m), dp(a), dp(alpha), dp(beta), dp(nodes)))
    return {"scheme": scheme, "k": k, "n_t": nt, "m_tau": m.reshape(nt, nt), "a_tau": a.reshape(nt, nt),
            "alpha": alpha, "beta": beta, "nodes": nodes}
