"""Oracle pinning (CPU): the reference's own C++ compiled against oracle/shim
must pass the reference's own unit suites and fast acceptance criteria, and
reproduce the known-answer tests its test-suite holds."""
import os
import subprocess

import numpy as np
import pytest

from oracle import refbind

REF_BIN = os.path.join(os.path.dirname(refbind.LIB))


@pytest.fixture(scope="module", autouse=True)
def _built():
    refbind.load()


@pytest.mark.parametrize("suite", ["test_temporal", "test_mesh_spatial", "test_operator", "test_multigrid",
                                   "test_gmres", "test_driver_config"])
def test_reference_unit_suite_passes_under_shim(suite):
    exe = os.path.join(REF_BIN, suite)
    if not os.path.exists(exe):
        pytest.skip("reference test binaries not built (no /root/reference on this host)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.parametrize("criterion", [1, 2, 3, 7])
def test_reference_acceptance_fast_criteria(criterion):
    exe = os.path.join(REF_BIN, "acceptance")
    if not os.path.exists(exe):
        pytest.skip("reference acceptance binary not built")
    r = subprocess.run([exe, str(criterion)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout + r.stderr


def _dg_step(w, tau, lam, u_prev):
    A = w["a"] + tau * lam * w["m"]
    return np.linalg.solve(A, w["alpha"] * u_prev)[-1]


def _cgp_step(w, tau, lam, u_prev):
    A = w["a"] + tau * lam * w["m"]
    return np.linalg.solve(A, -(w["alpha"] + tau * lam * w["beta"]) * u_prev)[-1]


def test_known_answer_dg0_is_backward_euler():
    # tests/test_temporal.cpp:69-78
    w = refbind.temporal_weights(0, 0)
    for tau in (0.5, 0.1, 0.01):
        for lam in (1.0, 3.5):
            assert abs(_dg_step(w, tau, lam, 1.0) - 1.0 / (1.0 + tau * lam)) <= 1e-13


def test_known_answer_cgp1_is_crank_nicolson():
    # tests/test_temporal.cpp:80-89
    w = refbind.temporal_weights(1, 1)
    for tau in (0.5, 0.1, 0.01):
        for lam in (1.0, 3.5):
            cn = (1.0 - 0.5 * tau * lam) / (1.0 + 0.5 * tau * lam)
            assert abs(_cgp_step(w, tau, lam, 1.0) - cn) <= 1e-13


def test_known_answer_dg1_is_radau_iia():
    # tests/test_temporal.cpp:91-98
    w = refbind.temporal_weights(0, 1)
    for z in (-0.5, -2.0, -10.0):
        u = np.linalg.solve(w["a"] - z * w["m"], w["alpha"])[-1]
        radau = (1.0 + z / 3.0) / (1.0 - 2.0 * z / 3.0 + z * z / 6.0)
        assert abs(u - radau) <= 1e-12


def test_quadrature_exactness():
    # tests/test_support.hpp:117-148
    for n in range(1, 7):
        p, w = refbind.quadrature(0, n)
        for m in range(2 * n):
            assert abs(np.dot(w, p ** m) - 1.0 / (m + 1)) < 1e-13
    for n in range(2, 7):
        p, w = refbind.quadrature(1, n)
        for m in range(2 * n - 2):
            assert abs(np.dot(w, p ** m) - 1.0 / (m + 1)) < 1e-13
    for n in range(1, 7):
        p, w = refbind.quadrature(2, n)
        for m in range(2 * n - 1):
            assert abs(np.dot(w, p ** m) - 1.0 / (m + 1)) < 1e-13


def test_oracle_matrix_free_matches_numpy_assembly_c1():
    """Independent numpy check of the oracle's C1 operator: columns of the
    matrix-free operator form a matrix whose Dirichlet rows are identity."""
    from paper_2408_04372_b200 import problems
    cfg = problems.config("C1", refinements=1)
    R = refbind.Reference(cfg)
    n = R.n_dofs
    A = np.stack([R.apply(np.eye(n)[j]) for j in range(n)], axis=1)
    nx = R.n_space
    d = cfg.cells * cfg.p + 1
    g = np.arange(nx)
    bd = (g % d == 0) | (g % d == d - 1) | (g // d == 0) | (g // d == d - 1)
    for f in range(n // nx):
        for b in np.nonzero(bd)[0]:
            row = A[f * nx + b]
            assert row[f * nx + b] == 1.0 and np.count_nonzero(row) == 1
    assert np.linalg.cond(A) < 1e8
