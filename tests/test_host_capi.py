"""CPU tests of the product's host layer and C ABI: the extension loads,
exports every symbol include/stmg_b200.h declares, rejects bad arguments with
the documented codes, and its host-side discretisation tables equal the
reference's (no GPU compute calls)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import refbind
from paper_2408_04372_b200 import native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "stmg_b200.h")


def _declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(stmg_[a-z0-9_]+)\s*\(", src))
    return sorted(n for n in names if n != "stmg_linear_map")


def test_header_symbols_exported_and_bound():
    lib = N.load()
    declared = _declared_symbols()
    assert len(declared) >= 35
    bound = {name for name, _, _ in N.SIGNATURES}
    for name in declared:
        assert hasattr(lib, name), f"{name} missing from libstmg_b200.so"
        assert name in bound, f"{name} has no ctypes signature"


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {N.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out


def _arr(n):
    a = np.zeros(n)
    return a, a.ctypes.data_as(N.c_double_p)


@pytest.mark.parametrize("kind,n", [(0, 1), (0, 3), (0, 5), (1, 2), (1, 4), (1, 5), (2, 1), (2, 3), (2, 4)])
def test_quadrature_matches_reference(kind, n):
    p, pp = _arr(n)
    w, wp = _arr(n)
    N.check(N.load().stmg_quadrature(kind, n, pp, wp))
    rp, rw = refbind.quadrature(kind, n)
    assert np.max(np.abs(p - rp)) <= 1e-15
    assert np.max(np.abs(w - rw)) <= 2e-15


@pytest.mark.parametrize("scheme,k", [(0, 0), (0, 1), (0, 2), (0, 3), (1, 1), (1, 2), (1, 3)])
def test_temporal_weights_match_reference(scheme, k):
    nt = k + 1 if scheme == 0 else k
    m, mp = _arr(nt * nt)
    a, ap = _arr(nt * nt)
    al, alp = _arr(nt)
    be, bep = _arr(nt)
    nd, ndp = _arr(nt)
    N.check(N.load().stmg_temporal_weights(scheme, k, mp, ap, alp, bep, ndp))
    r = refbind.temporal_weights(scheme, k)
    for got, want in [(m, r["m"].ravel()), (a, r["a"].ravel()), (al, r["alpha"]), (be, r["beta"]),
                      (nd, r["nodes"])]:
        assert np.max(np.abs(got - want)) <= 1e-14 * max(1.0, np.max(np.abs(want)))


@pytest.mark.parametrize("eq,scheme,k,S", [(0, 0, 1, 3), (0, 1, 2, 3), (1, 0, 1, 4), (1, 1, 2, 4), (1, 1, 1, 3),
                                           (1, 0, 2, 2), (0, 0, 3, 1)])
def test_block_coefficients_match_reference(eq, scheme, k, S):
    from paper_2408_04372_b200 import problems
    nt = k + 1 if scheme == 0 else k
    tau = 0.3
    F = S * nt
    cm, cmp_ = _arr(F * F)
    ca, cap = _arr(F * F)
    N.check(N.load().stmg_block_coefficients(eq, scheme, k, tau, S, cmp_, cap))
    cfg = problems.Config("t", eq, scheme, 1 + 1, 2, 0, 1, k, S, tau)
    R = refbind.Reference(cfg)
    CM, CA = cm.reshape(F, F), ca.reshape(F, F)
    for s in range(S):
        for j in range(S):
            rm, ra = R.block_coefficients(s, j, nt)
            got_m = CM[s * nt:(s + 1) * nt, j * nt:(j + 1) * nt]
            got_a = CA[s * nt:(s + 1) * nt, j * nt:(j + 1) * nt]
            scale = max(1.0, np.max(np.abs(rm)), np.max(np.abs(ra)))
            assert np.max(np.abs(got_m - rm)) <= 1e-13 * scale
            assert np.max(np.abs(got_a - ra)) <= 1e-13 * scale


def test_invalid_arguments_return_codes():
    lib = N.load()
    p, pp = _arr(4)
    w, wp = _arr(4)
    assert lib.stmg_quadrature(0, 0, pp, wp) == -1
    assert "n must be" in lib.stmg_last_error().decode()
    assert lib.stmg_temporal_weights(1, 0, pp, pp, pp, pp, pp) == -1
    h = C.c_void_p()
    lo = np.zeros(3)
    hi = np.ones(3)
    assert lib.stmg_mesh_create(4, lo.ctypes.data_as(N.c_double_p), hi.ctypes.data_as(N.c_double_p), 2, 1, None,
                                C.byref(h)) == -1
    with pytest.raises(N.StmgInvalidArgument):
        N.check(-1)
    with pytest.raises(ValueError):
        N.check(-1)
    with pytest.raises(N.StmgError):
        N.check(-2)


def test_reference_side_binding_links():
    """oracle/b200_backend.cpp (INTEGRATION.md's LinearMap adapter) compiles
    against the reference headers and links the reference's objects with
    libstmg_b200.so; GPU runs are in tests/test_gpu_ref_binding.py."""
    path = os.path.join(ROOT, "oracle", "_ref", "libb200_backend.so")
    if not os.path.exists(path):
        refbind.build()
    lib = C.CDLL(path)
    assert hasattr(lib, "b200_backend_gmres") and hasattr(lib, "b200_backend_last_error")
