"""Pin the numpy restatement (oracle/stmg_np.py) against the reference's own
C++ (oracle/_ref) on the same seeded inputs (CPU)."""
import numpy as np
import pytest

from oracle import refbind, stmg_np
from paper_2408_04372_b200 import problems


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("kind,fn", [(0, stmg_np.gauss), (1, stmg_np.gauss_lobatto), (2, stmg_np.gauss_radau_right)])
def test_quadrature(kind, fn):
    for n in range(2 if kind == 1 else 1, 7):
        p, w = fn(n)
        rp, rw = refbind.quadrature(kind, n)
        assert np.max(np.abs(p - rp)) < 1e-15 and np.max(np.abs(w - rw)) < 1e-14


@pytest.mark.parametrize("scheme,k", [(0, 0), (0, 1), (0, 2), (0, 3), (1, 1), (1, 2), (1, 3)])
def test_weights(scheme, k):
    w = stmg_np.dg_weights(k) if scheme == 0 else stmg_np.cgp_weights(k)
    r = refbind.temporal_weights(scheme, k)
    for a, b in [(w.m, r["m"]), (w.a, r["a"]), (w.alpha, r["alpha"]), (w.beta, r["beta"]), (w.unknown_nodes, r["nodes"])]:
        assert np.max(np.abs(a - b)) < 1e-13


CFGS = [("C1", None), ("C2", 1), ("C3", 0), ("C4", 0), ("C5-4", None)]


@pytest.mark.parametrize("name,r", CFGS)
def test_apply(name, r):
    cfg = problems.config(name, r)
    op, _ = stmg_np.build(cfg)
    R = refbind.Reference(cfg)
    u = problems.uniform_vector(R.n_dofs, seed=8)
    assert _rel(op.apply(u), R.apply(u)) < 1e-13


@pytest.mark.parametrize("name,r", [("C1", 2), ("C2", 1), ("C3", 0)])
def test_multigrid_components(name, r):
    cfg = problems.config(name, r)
    _, M = stmg_np.build(cfg, with_mg=True)
    R = refbind.Reference(cfg, with_mg=True)
    info = R.level_info()
    assert [o.n_dofs for o in M.ops] == [l["n_dofs"] for l in info]
    for l, li in enumerate(info):
        assert abs(M.omega[l] - li["omega"]) < 1e-8
    for l in range(len(info) - 1):
        nf, nc = info[l]["n_dofs"], info[l + 1]["n_dofs"]
        c = problems.uniform_vector(nc, seed=l)
        f = problems.uniform_vector(nf, seed=50 + l)
        assert _rel(M.transfers[l].prolong(c), R.prolong(l, c, nf)) < 1e-13
        assert _rel(M.transfers[l].restrict(f), R.restrict_(l, f, nc)) < 1e-13
        res = problems.uniform_vector(nf, seed=90 + l)
        z = M.smoothers[l].add_correction(res, np.zeros(nf))
        assert _rel(z, R.asm_add_correction(l, res, np.zeros(nf))) < 1e-11
    res = problems.uniform_vector(R.n_dofs, seed=3)
    assert _rel(M.apply(res), R.vcycle(res)) < 1e-11


@pytest.mark.parametrize("name,r", [("C1", None), ("C2", 1)])
def test_gmres_solve(name, r):
    cfg = problems.config(name, r)
    op, M = stmg_np.build(cfg, with_mg=True)
    R = refbind.Reference(cfg, with_mg=True)
    b = R.assemble_rhs(1, 0.5, 0.0)
    x, info = stmg_np.gmres(op.apply, b, np.zeros_like(b), rel_tol=1e-10, abs_tol=0.0, precond=M.apply)
    xr, ir = R.gmres(b, rel_tol=1e-10, abs_tol=0.0)
    assert info["iterations"] == ir["iterations"]
    assert _rel(x, xr) < 1e-9
