"""ctypes binding of oracle/_ref/libstmg_ref.so: the reference's own C++
(/root/reference/proj/src, compiled unmodified against oracle/shim by
oracle/Makefile) behind the C harness in oracle/ref_harness.cpp.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py as the checker, never by the
product package."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "libstmg_ref.so")
REF_SRC = "/root/reference/proj"

dp = C.POINTER(C.c_double)


class RefDesc(C.Structure):
    _fields_ = [("dim", C.c_int), ("equation", C.c_int), ("scheme", C.c_int), ("k", C.c_int), ("p", C.c_int),
                ("n_steps", C.c_int), ("tau", C.c_double), ("base_cells", C.c_int), ("refinements", C.c_int),
                ("lo", C.c_double * 3), ("hi", C.c_double * 3), ("vertices", dp), ("cell_scale", dp),
                ("perturb_magnitude", C.c_double), ("perturb_seed", C.c_uint64), ("with_mg", C.c_int),
                ("n_strategy", C.c_int), ("strategy", C.POINTER(C.c_int)), ("n_smooth", C.c_int),
                ("direct_coarse_max", C.c_long), ("coarse_rel_tol", C.c_double), ("coarse_max_iters", C.c_int),
                ("eig_iters", C.c_int), ("mg_seed", C.c_uint64)]


_lib = None


def build() -> None:
    """Compile the oracle from the reference sources (needs /root/reference)."""
    if not os.path.isdir(REF_SRC):
        raise RuntimeError("reference sources not mounted; use the prebuilt oracle/_ref")
    subprocess.run(["make", "-C", HERE, "-j8", "all"], check=True, stdout=subprocess.DEVNULL)


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        build()
    lib = C.CDLL(LIB)
    lib.ref_last_error.restype = C.c_char_p
    lib.ref_create.restype = C.c_void_p
    lib.ref_create.argtypes = [C.POINTER(RefDesc)]
    lib.ref_destroy.argtypes = [C.c_void_p]
    lib.ref_n_dofs.restype = C.c_long
    lib.ref_n_dofs.argtypes = [C.c_void_p]
    lib.ref_n_space.restype = C.c_long
    lib.ref_n_space.argtypes = [C.c_void_p]
    for name in ["ref_apply", "ref_vcycle_apply"]:
        getattr(lib, name).argtypes = [C.c_void_p, dp, dp]
    lib.ref_spatial_apply.argtypes = [C.c_void_p, C.c_int, dp, dp]
    lib.ref_mg_levels.argtypes = [C.c_void_p]
    lib.ref_level_info.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_long), dp]
    lib.ref_level_tau.restype = C.c_double
    lib.ref_level_tau.argtypes = [C.c_void_p, C.c_int]
    for name in ["ref_level_apply", "ref_asm_add_correction", "ref_prolong", "ref_restrict", "ref_smooth"]:
        getattr(lib, name).argtypes = [C.c_void_p, C.c_int, dp, dp]
    lib.ref_asm_overlap_counts.argtypes = [C.c_void_p, C.c_int, dp]
    lib.ref_omega.restype = C.c_double
    lib.ref_omega.argtypes = [C.c_void_p, C.c_int]
    lib.ref_set_omega.argtypes = [C.c_void_p, C.c_int, C.c_double]
    lib.ref_gmres.argtypes = [C.c_void_p, dp, dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                              C.POINTER(C.c_int), dp, dp, dp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    lib.ref_assemble_rhs.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, dp, dp, dp]
    lib.ref_extract_final.argtypes = [C.c_void_p, dp, dp, dp, dp, dp]
    lib.ref_error_norms.argtypes = [C.c_void_p, dp, dp, C.c_double, C.c_double, dp]
    lib.ref_probe_value.argtypes = [C.c_void_p, dp, dp, C.c_int, C.c_double, dp, dp]
    lib.ref_interpolate_gaussian.argtypes = [C.c_void_p, dp, C.c_double, dp]
    lib.ref_vertices.argtypes = [C.c_void_p, C.c_int, dp]
    lib.ref_temporal_weights.argtypes = [C.c_int, C.c_int, dp, dp, dp, dp, dp]
    lib.ref_quadrature.argtypes = [C.c_int, C.c_int, dp, dp]
    lib.ref_block_coefficients.argtypes = [C.c_void_p, C.c_int, C.c_int, dp, dp]
    lib.ref_run_json.argtypes = [C.c_char_p, C.c_int, C.c_char_p, C.c_long]
    lib.ref_config_json.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_char_p), C.c_char_p,
                                    C.c_long]
    lib.ref_perturbed_vertices.argtypes = [C.c_int, dp, dp, C.c_int, C.c_int, C.c_double, C.c_uint64, dp]
    _lib = lib
    return lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(dp)


def _chk(rc: int) -> None:
    if rc != 0:
        raise RuntimeError("reference: " + load().ref_last_error().decode())


class Reference:
    """One discretised slab system built with the reference's classes: the
    finest SpaceTimeOperator and, with with_mg, the SpaceTimeMultigrid."""

    def __init__(self, cfg, with_mg: bool = False, strategy: Optional[Sequence[int]] = None, n_smooth: int = 1,
                 direct_coarse_max: int = 20000, eig_iters: int = 20, mg_seed: int = 42, vertices=None,
                 perturb_magnitude: float = 0.0, perturb_seed: int = 42):
        lib = load()
        d = RefDesc()
        d.dim, d.equation, d.scheme, d.k, d.p, d.n_steps = cfg.dim, cfg.equation, cfg.scheme, cfg.k, cfg.p, cfg.n_steps
        d.tau, d.base_cells, d.refinements = cfg.tau, cfg.base_cells, cfg.refinements
        d.lo[:] = [0.0, 0.0, 0.0]
        d.hi[:] = [1.0, 1.0, 1.0]
        self._keep = []
        v = vertices if vertices is not None else cfg.vertices()
        if v is not None:
            v = np.ascontiguousarray(v, dtype=np.float64)
            self._keep.append(v)
            d.vertices = _p(v)
        if cfg.rho is not None:
            r = np.ascontiguousarray(cfg.rho, dtype=np.float64)
            self._keep.append(r)
            d.cell_scale = _p(r)
        d.perturb_magnitude, d.perturb_seed = perturb_magnitude, perturb_seed
        d.with_mg = 1 if with_mg else 0
        if strategy is None:
            d.n_strategy = -1
        else:
            s = (C.c_int * max(len(strategy), 1))(*strategy)
            self._keep.append(s)
            d.n_strategy, d.strategy = len(strategy), s
        d.n_smooth, d.direct_coarse_max, d.coarse_rel_tol, d.coarse_max_iters = n_smooth, direct_coarse_max, 1e-3, 2000
        d.eig_iters, d.mg_seed = eig_iters, mg_seed
        h = lib.ref_create(C.byref(d))
        if not h:
            raise RuntimeError("reference: " + lib.ref_last_error().decode())
        self.h = C.c_void_p(h)
        self.n_dofs = lib.ref_n_dofs(self.h)
        self.n_space = lib.ref_n_space(self.h)
        self.n_levels = lib.ref_mg_levels(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            load().ref_destroy(self.h)
            self.h = None

    def apply(self, u: np.ndarray) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.float64)
        y = np.empty(self.n_dofs)
        _chk(load().ref_apply(self.h, _p(u), _p(y)))
        return y

    def spatial_apply(self, kind: int, u: np.ndarray) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.float64)
        y = np.empty(self.n_space)
        _chk(load().ref_spatial_apply(self.h, kind, _p(u), _p(y)))
        return y

    def block_coefficients(self, s: int, j: int, n_t: int):
        cm, ca = np.zeros(n_t * n_t), np.zeros(n_t * n_t)
        _chk(load().ref_block_coefficients(self.h, s, j, _p(cm), _p(ca)))
        return cm.reshape(n_t, n_t), ca.reshape(n_t, n_t)

    def level_info(self):
        out = []
        for l in range(self.n_levels):
            ints = (C.c_int * 5)()
            n = C.c_long()
            w = C.c_double()
            _chk(load().ref_level_info(self.h, l, ints, C.byref(n), C.byref(w)))
            out.append({"mesh_level": ints[0], "p": ints[1], "k": ints[2], "n_steps": ints[3],
                        "coarsening": ints[4], "n_dofs": n.value, "omega": w.value,
                        "tau": load().ref_level_tau(self.h, l)})
        return out

    def level_apply(self, l: int, u: np.ndarray) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.float64)
        y = np.empty_like(u)
        _chk(load().ref_level_apply(self.h, l, _p(u), _p(y)))
        return y

    def asm_add_correction(self, l: int, r: np.ndarray, z: np.ndarray) -> np.ndarray:
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.array(z, dtype=np.float64)
        _chk(load().ref_asm_add_correction(self.h, l, _p(r), _p(z)))
        return z

    def overlap_counts(self, l: int, n: int) -> np.ndarray:
        c = np.empty(n)
        _chk(load().ref_asm_overlap_counts(self.h, l, _p(c)))
        return c

    def prolong(self, l: int, c: np.ndarray, n_fine: int) -> np.ndarray:
        c = np.ascontiguousarray(c, dtype=np.float64)
        f = np.empty(n_fine)
        _chk(load().ref_prolong(self.h, l, _p(c), _p(f)))
        return f

    def restrict_(self, l: int, f: np.ndarray, n_coarse: int) -> np.ndarray:
        f = np.ascontiguousarray(f, dtype=np.float64)
        c = np.empty(n_coarse)
        _chk(load().ref_restrict(self.h, l, _p(f), _p(c)))
        return c

    def omega(self, l: int) -> float:
        return load().ref_omega(self.h, l)

    def set_omega(self, l: int, w: float) -> None:
        load().ref_set_omega(self.h, l, w)

    def smooth(self, l: int, f: np.ndarray, u: np.ndarray) -> np.ndarray:
        f = np.ascontiguousarray(f, dtype=np.float64)
        u = np.array(u, dtype=np.float64)
        _chk(load().ref_smooth(self.h, l, _p(f), _p(u)))
        return u

    def vcycle(self, r: np.ndarray) -> np.ndarray:
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.empty(self.n_dofs)
        _chk(load().ref_vcycle_apply(self.h, _p(r), _p(z)))
        return z

    def gmres(self, b: np.ndarray, x0: Optional[np.ndarray] = None, max_iters: int = 1000, restart: int = 100,
              rel_tol: float = 1e-10, abs_tol: float = 0.0, precond: bool = True, history_cap: int = 1100):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(self.n_dofs) if x0 is None else np.array(x0, dtype=np.float64)
        it, conv, hl = C.c_int(), C.c_int(), C.c_int()
        fr, ir = C.c_double(), C.c_double()
        hist = np.zeros(history_cap)
        _chk(load().ref_gmres(self.h, _p(b), _p(x), max_iters, restart, rel_tol, abs_tol, 1 if precond else 0,
                              C.byref(it), C.byref(fr), C.byref(ir), _p(hist), history_cap, C.byref(hl),
                              C.byref(conv)))
        return x, {"iterations": it.value, "final_residual": fr.value, "initial_residual": ir.value,
                   "converged": bool(conv.value), "residual_history": hist[:min(hl.value, history_cap)].tolist()}

    def assemble_rhs(self, source_kind: int = 1, frequency: float = 0.5, t0: float = 0.0,
                     u0: Optional[np.ndarray] = None, v0: Optional[np.ndarray] = None) -> np.ndarray:
        u0 = np.zeros(self.n_space) if u0 is None else np.ascontiguousarray(u0, dtype=np.float64)
        v0 = np.zeros(self.n_space) if v0 is None else np.ascontiguousarray(v0, dtype=np.float64)
        rhs = np.empty(self.n_dofs)
        _chk(load().ref_assemble_rhs(self.h, source_kind, frequency, t0, _p(u0), _p(v0), _p(rhs)))
        return rhs

    def extract_final(self, u: np.ndarray, u0: np.ndarray, v0: Optional[np.ndarray] = None):
        u = np.ascontiguousarray(u, dtype=np.float64)
        u0 = np.ascontiguousarray(u0, dtype=np.float64)
        v0 = np.zeros(self.n_space) if v0 is None else np.ascontiguousarray(v0, dtype=np.float64)
        uf, vf = np.empty(self.n_space), np.empty(self.n_space)
        _chk(load().ref_extract_final(self.h, _p(u), _p(u0), _p(v0), _p(uf), _p(vf)))
        return uf, vf

    def error_norms(self, u: np.ndarray, u0: np.ndarray, frequency: float = 0.5, t0: float = 0.0):
        """error_norms (driver.cpp:83-92) of one batch vs the manufactured
        solution: (L2(L2), Linf(L2), Linf(Linf))."""
        out = np.zeros(3)
        _chk(load().ref_error_norms(self.h, _p(np.ascontiguousarray(u, dtype=np.float64)),
                                    _p(np.ascontiguousarray(u0, dtype=np.float64)), frequency, t0, _p(out)))
        return tuple(out)

    def probe_value(self, u: np.ndarray, u0: np.ndarray, step: int, t_ref: float, x) -> float:
        """value_at + evaluate_fe at locate_point(x) (the march() probe sample)."""
        out = np.zeros(1)
        _chk(load().ref_probe_value(self.h, _p(np.ascontiguousarray(u, dtype=np.float64)),
                                    _p(np.ascontiguousarray(u0, dtype=np.float64)), step, t_ref,
                                    _p(np.ascontiguousarray(x, dtype=np.float64)), _p(out)))
        return float(out[0])

    def interpolate_gaussian(self, centre=(0.5, 0.5, 0.5), width: float = 0.05) -> np.ndarray:
        c = np.ascontiguousarray(centre, dtype=np.float64)
        u = np.empty(self.n_space)
        _chk(load().ref_interpolate_gaussian(self.h, _p(c), width, _p(u)))
        return u


def temporal_weights(scheme: int, k: int):
    nt = k + 1 if scheme == 0 else k
    m, a = np.zeros(nt * nt), np.zeros(nt * nt)
    al, be, nodes = np.zeros(nt), np.zeros(nt), np.zeros(nt)
    _chk(load().ref_temporal_weights(scheme, k, _p(m), _p(a), _p(al), _p(be), _p(nodes)))
    return {"m": m.reshape(nt, nt), "a": a.reshape(nt, nt), "alpha": al, "beta": be, "nodes": nodes}


def quadrature(kind: int, n: int):
    p, w = np.zeros(n), np.zeros(n)
    _chk(load().ref_quadrature(kind, n, _p(p), _p(w)))
    return p, w


def run_json(config: dict, refinement: int = -1) -> dict:
    """The reference's march over a config (parse_config, make_problem,
    resolve_probes; src/config.cpp, src/driver.cpp:95-262) as a report dict."""
    import json
    buf = C.create_string_buffer(1 << 24)
    _chk(load().ref_run_json(json.dumps(config).encode(), refinement, buf, len(buf)))
    return json.loads(buf.value.decode())


def config_json(config_text: str, overrides=()) -> dict:
    """parse_config + apply_override + config_to_json of the reference;
    raises ValueError with the reference's message on invalid input."""
    import json
    keys = (C.c_char_p * max(1, len(overrides)))(*[k.encode() for k, _ in overrides])
    vals = (C.c_char_p * max(1, len(overrides)))(*[v.encode() for _, v in overrides])
    buf = C.create_string_buffer(1 << 16)
    rc = load().ref_config_json(config_text.encode(), len(overrides), keys, vals, buf, len(buf))
    if rc != 0:
        raise ValueError(load().ref_last_error().decode())
    return json.loads(buf.value.decode())


def perturbed_vertices(dim: int, lo, hi, base_cells: int, refinements: int, magnitude: float, seed: int):
    n = (base_cells << refinements) + 1
    nv = n ** dim
    out = np.zeros(3 * nv)
    lo_a = np.asarray(lo, dtype=np.float64)
    hi_a = np.asarray(hi, dtype=np.float64)
    _chk(load().ref_perturbed_vertices(dim, _p(lo_a), _p(hi_a), base_cells, refinements, magnitude, seed, _p(out)))
    return out.reshape(nv, 3)
