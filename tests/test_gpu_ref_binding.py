"""The reference-side binding of INTEGRATION.md, compiled and run: the
reference's OWN gmres() (src/gmres.cpp:8-115, compiled unmodified into
oracle/_ref) drives the B200 operator and V-cycle through the LinearMap
adapter b200_operator / b200_vcycle (oracle/b200_backend.cpp, host buffers
through stmg_st_operator_apply_host / stmg_multigrid_apply_host), the way
march() plugs in its CPU maps (src/driver.cpp:193-203); and the one-call
device solve b200_solve (stmg_solve_host). Both must match the all-CPU
reference: GMRES iterations within +-1, solution relative difference
<= 1e-8 (north_star)."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2408_04372_b200 import problems

pytestmark = pytest.mark.gpu

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "libb200_backend.so")
dp = C.POINTER(C.c_double)


def _lib():
    lib = C.CDLL(LIB)
    lib.b200_backend_last_error.restype = C.c_char_p
    lib.b200_backend_gmres.argtypes = [C.c_int] * 6 + [C.c_double, C.c_int, C.c_int, dp, dp, C.c_int, C.c_uint64,
                                                       C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, dp, dp,
                                                       C.POINTER(C.c_int), C.POINTER(C.c_int)]
    return lib


def _p(a):
    return None if a is None else a.ctypes.data_as(dp)


@pytest.mark.parametrize("name,r", [("C1", None), ("C2", 2), ("C5-8", None)])
@pytest.mark.parametrize("mode", [0, 1])
def test_reference_gmres_with_b200_linear_maps(cuda, ref, name, r, mode):
    cfg = problems.config(name, r)
    R = ref.Reference(cfg, with_mg=True)
    b = R.assemble_rhs(1, 0.5, 0.0)
    x_ref, info_ref = R.gmres(b, rel_tol=1e-10, abs_tol=0.0)
    lib = _lib()
    v = cfg.vertices()
    v = None if v is None else np.ascontiguousarray(v, dtype=np.float64)
    rho = None if cfg.rho is None else np.ascontiguousarray(cfg.rho, dtype=np.float64)
    x = np.zeros_like(b)
    it, conv = C.c_int(), C.c_int()
    rc = lib.b200_backend_gmres(cfg.dim, cfg.equation, cfg.scheme, cfg.p, cfg.k, cfg.n_steps, cfg.tau,
                                cfg.base_cells, cfg.refinements, _p(v), _p(rho), 1, 42, mode, 1e-10, 0.0, 100, 1000,
                                _p(b), _p(x), C.byref(it), C.byref(conv))
    assert rc == 0, lib.b200_backend_last_error().decode()
    assert conv.value == 1 and info_ref["converged"]
    assert abs(it.value - info_ref["iterations"]) <= 1, (it.value, info_ref["iterations"])
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 1e-8
