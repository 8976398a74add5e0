"""Declarative run configuration: the reference's flat JSON schema, --set
overrides and problem construction (include/stmg/config.hpp:11-45,
src/config.cpp:12-215), resolving a config into the C-ABI's stmg_problem.

Semantics follow the reference: unknown keys are rejected by name, values are
type-checked the way nlohmann's get_to checks them (numbers for numeric keys,
booleans for `precondition`, strings for the enums), `--set key=value` parses
the value as JSON and falls back to a bare string, and the "shm" problem
rewrites the domain, time span, mesh and tolerance as shm_problem does
(src/driver.cpp:295-316) unless the config overrides them."""
from __future__ import annotations

import dataclasses
import json
from typing import Any, Dict, List, Sequence, Tuple

from . import native as N

EQUATIONS = ("heat", "wave")
SCHEMES = ("dg", "cgp")
PROBLEMS = ("manufactured", "shm", "zero")
COARSENINGS = ("space-h", "space-p", "time-tau", "time-k")  # Coarsening codes 0..3 (multigrid.hpp:14)


class ConfigError(ValueError):
    """invalid_argument raised by the configuration layer."""


@dataclasses.dataclass
class Config:
    equation: str = "heat"
    scheme: str = "dg"
    problem: str = "manufactured"
    k: int = 1
    p: int = 1
    dim: int = 2
    t_final: float = 1.0
    base_cells: int = 2
    base_time_intervals: int = 1
    refinements: int = 2
    r_min: int = 2
    r_max: int = 4
    batch: int = 2
    frequency: float = 2.0
    shm_s: float = 0.3
    perturb: float = 0.0
    rho_random_lo: float = 0.0
    rho_random_hi: float = 0.0
    seed: int = 42
    abs_tol: float = 1e-12
    rel_tol: float = 1e-12
    max_iters: int = 1000
    restart: int = 100
    n_smooth: int = 1
    precondition: bool = True
    probe_samples_per_step: int = 16
    strategy: List[str] = dataclasses.field(default_factory=list)
    probes: List[Tuple[float, float, float]] = dataclasses.field(default_factory=list)


_FIELDS = {f.name: f for f in dataclasses.fields(Config)}
_INT_KEYS = {n for n, f in _FIELDS.items() if f.type in ("int", int)}
_FLOAT_KEYS = {n for n, f in _FIELDS.items() if f.type in ("float", float)}
_STR_KEYS = {"equation", "scheme", "problem"}


def _number(key: str, v: Any, integral: bool):
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        raise ConfigError(f"config: bad value for '{key}': type must be number")
    if integral:
        if key == "seed" and v < 0:
            raise ConfigError(f"config: bad value for '{key}': seed must be >= 0")
        return int(v)
    return float(v)


def config_from_dict(j: Dict[str, Any]) -> Config:
    """config_from_json (src/config.cpp:12-84)."""
    if not isinstance(j, dict):
        raise ConfigError("config: top level must be an object")
    for key in j:
        if key not in _FIELDS:
            raise ConfigError(f"config: unknown key '{key}'")
    c = Config()
    for key, v in j.items():
        if key in _INT_KEYS:
            setattr(c, key, _number(key, v, True))
        elif key in _FLOAT_KEYS:
            setattr(c, key, _number(key, v, False))
        elif key in _STR_KEYS:
            if not isinstance(v, str):
                raise ConfigError(f"config: bad value for '{key}': type must be string")
            setattr(c, key, v)
        elif key == "precondition":
            if not isinstance(v, bool):
                raise ConfigError("config: bad value for 'precondition': type must be boolean")
            c.precondition = v
        elif key == "strategy":
            if not isinstance(v, list) or not all(isinstance(s, str) for s in v):
                raise ConfigError("config: bad value for 'strategy': type must be an array of strings")
            c.strategy = list(v)
        elif key == "probes":
            pts = []
            if not isinstance(v, list):
                raise ConfigError("config: bad value for 'probes': type must be array")
            for row in v:
                if not isinstance(row, list) or len(row) > 3:
                    raise ConfigError("config: probe must be an array of <= 3 reals")
                x = [0.0, 0.0, 0.0]
                for a, xa in enumerate(row):
                    x[a] = _number("probes", xa, False)
                pts.append(tuple(x))
            c.probes = pts
    if c.equation not in EQUATIONS:
        raise ConfigError("config: equation must be heat|wave")
    if c.scheme not in SCHEMES:
        raise ConfigError("config: scheme must be dg|cgp")
    if c.problem not in PROBLEMS:
        raise ConfigError("config: problem must be manufactured|shm|zero")
    return c


def parse_config(text: str) -> Config:
    """parse_config (src/config.cpp:88-100)."""
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise ConfigError(f"config: JSON parse error: {e}") from None
    if not isinstance(j, dict):
        raise ConfigError("config: top level must be an object")
    return config_from_dict(j)


def config_to_dict(c: Config) -> Dict[str, Any]:
    """config_to_json (src/config.cpp:102-132): lossless round trip."""
    d = dataclasses.asdict(c)
    d["probes"] = [list(p) for p in c.probes]
    d["strategy"] = list(c.strategy)
    return d


def apply_override(c: Config, key: str, value: str) -> Config:
    """apply_override (src/config.cpp:134-153): JSON value or bare string."""
    j = config_to_dict(c)
    if key not in j:
        raise ConfigError(f"config: unknown override key '{key}'")
    try:
        v = json.loads(value)
    except json.JSONDecodeError:
        v = value
    j[key] = v
    return config_from_dict(j)


def resolve_probes(c: Config) -> List[Tuple[float, float, float]]:
    """resolve_probes (src/config.cpp:155-161) with the demo defaults
    (shm_default_probes, src/driver.cpp:318-320)."""
    if c.probes:
        return list(c.probes)
    if c.problem == "shm":
        return [(0.75, 0.0, 0.0), (0.0, 0.0, 0.75), (0.75, 0.1, 0.75)]
    return []


def make_problem(c: Config, refinement: int) -> N.Problem:
    """make_problem (src/config.cpp:163-215) into the C-ABI problem record."""
    p = N.Problem()
    p.equation = EQUATIONS.index(c.equation)
    p.scheme = SCHEMES.index(c.scheme)
    p.problem = PROBLEMS.index(c.problem)
    p.k, p.p, p.dim = c.k, c.p, c.dim
    for a in range(3):
        p.lo[a], p.hi[a] = 0.0, 1.0
    p.t_final = c.t_final
    p.refinements = refinement
    p.base_cells = c.base_cells
    p.base_time_intervals = c.base_time_intervals
    p.batch = c.batch
    p.frequency = c.frequency
    p.shm_s = c.shm_s
    p.perturb = c.perturb
    p.seed = c.seed
    p.rho_random_lo, p.rho_random_hi = c.rho_random_lo, c.rho_random_hi
    p.abs_tol, p.rel_tol = c.abs_tol, c.rel_tol
    p.max_iters, p.restart, p.n_smooth = c.max_iters, c.restart, c.n_smooth
    p.precondition = 1 if c.precondition else 0
    p.probe_samples_per_step = c.probe_samples_per_step
    if len(c.strategy) > 32:
        raise ConfigError("config: strategy has more than 32 entries")
    for i, s in enumerate(c.strategy):
        if s not in COARSENINGS:
            raise ConfigError(f"config: unknown coarsening '{s}'")
        p.strategy[i] = COARSENINGS.index(s)
    p.n_strategy = len(c.strategy)
    p.timers = 1
    if c.problem == "shm":
        if c.equation != "wave":
            raise ConfigError("config: shm problem requires equation=wave")
        for a in range(3):
            p.lo[a], p.hi[a] = -1.0, 1.0
        p.abs_tol = 1e-10
        p.t_final = c.t_final if c.t_final != 1.0 else 2.0
        p.base_cells = c.base_cells if c.base_cells != 2 else 5
        p.base_time_intervals = c.base_time_intervals if c.base_time_intervals != 1 else 5
    return p


def level_plan(p: N.Problem) -> List[dict]:
    """The multigrid plan of a resolved problem (print_plan,
    tools/stmg.cpp:106-137): finest first."""
    lib = N.load()
    n_steps_total = p.base_time_intervals << (p.refinements + 1)
    tau = p.t_final / n_steps_total
    strat = (N.C.c_int * 32)(*p.strategy)
    n_levels = N.C.c_int(0)
    ints = (N.C.c_int * (5 * 64))()
    taus = (N.C.c_double * 64)()
    N.check(lib.stmg_level_plan(p.scheme, p.refinements, p.p, p.k, p.batch, tau,
                                p.n_strategy if p.n_strategy > 0 else -1, strat, 64, N.C.byref(n_levels), ints, taus))
    nt_of = (lambda k: k + 1) if p.scheme == 0 else (lambda k: k)
    out = []
    for l in range(n_levels.value):
        code, ml, pp, kk, ns = ints[5 * l:5 * l + 5]
        nx = 1
        for _ in range(p.dim):
            nx *= (p.base_cells << ml) * pp + 1
        out.append({"coarsening": "finest" if code < 0 else COARSENINGS[code], "mesh_level": ml, "p": pp, "k": kk,
                    "n_steps": ns, "tau": taus[l], "n_dofs": ns * nt_of(kk) * nx})
    return out


def plan_text(c: Config) -> str:
    lines = ["multigrid plan (finest first):"]
    for l, s in enumerate(level_plan(make_problem(c, c.refinements))):
        lines.append(f"  level {l}: {s['coarsening']}  mesh_level={s['mesh_level']} p={s['p']} k={s['k']} "
                     f"n_steps={s['n_steps']} n_dofs={s['n_dofs']}")
    return "\n".join(lines) + "\n"


def merge(config: Dict[str, Any] = None, overrides: Dict[str, Any] = None) -> Config:
    d = dict(config or {})
    d.update(overrides or {})
    return config_from_dict(d)


__all__: Sequence[str] = ["Config", "ConfigError", "parse_config", "config_from_dict", "config_to_dict",
                          "apply_override", "resolve_probes", "make_problem", "level_plan", "plan_text", "merge"]
