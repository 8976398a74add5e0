"""GPU parity of wide batches -- S * n_t > 8 time-step fields per slab system,
which the reference's march allows for any batch size (driver.cpp:105-109):
the operator composes 2F single-field applications (st_apply_wide), the
smoother sweeps groups of whole steps, the temporal transfers read the fields
straight from memory. Oracle: the reference's SpaceTimeOperator,
ASMSmoother, Transfer, V-cycle and GMRES on the same system. Bars as the
narrow path: vmult 1e-12, smoother 1e-9, transfers 1e-13, V-cycle 1e-9,
GMRES iterations +-1 and solution 1e-8."""
import numpy as np
import pytest

from paper_2408_04372_b200 import api, problems

pytestmark = pytest.mark.gpu

# (equation, scheme, dim, base, r, p, k, S): F = S * n_t = 12, 16, 10, 9
WIDE = [(0, 0, 2, 2, 2, 2, 2, 4), (1, 1, 2, 2, 2, 2, 2, 8), (0, 0, 3, 2, 1, 2, 1, 5), (1, 1, 3, 2, 1, 1, 3, 3)]
# the default plan halves S (time-tau), so the multigrid cases have even S
WIDE_MG = [(0, 0, 2, 2, 2, 2, 2, 4), (1, 1, 2, 2, 2, 2, 2, 8), (0, 0, 3, 2, 1, 2, 2, 4), (1, 1, 3, 2, 1, 1, 3, 4)]


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _cfg(case, perturb=0.0):
    eq, scheme, dim, base, r, p, k, S = case
    cfg = problems.Config("wide", eq, scheme, dim, base, r, p, k, S, 0.1)
    cfg.perturb = perturb
    return cfg


def _dev(cuda, a):
    return cuda.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("case", WIDE)
@pytest.mark.parametrize("perturb", [0.0, 0.15])
def test_wide_vmult_and_residual(cuda, ref, case, perturb):
    cfg = _cfg(case, perturb)
    assert cfg.n_steps * cfg.n_t > 8
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    op = api.SpaceTimeOperator(mesh, cfg.refinements, cfg.p, cfg.equation, cfg.scheme, cfg.k, cfg.tau, cfg.n_steps,
                               cfg.rho)
    R = ref.Reference(cfg)
    u = problems.uniform_vector(op.n_dofs, seed=5)
    f = problems.uniform_vector(op.n_dofs, seed=6)
    want = R.apply(u)
    assert _rel(op.apply(_dev(cuda, u)).cpu().numpy(), want) <= 1e-12
    assert _rel(op.residual(_dev(cuda, f), _dev(cuda, u)).cpu().numpy(), f - want) <= 1e-12


@pytest.mark.parametrize("case", WIDE_MG)
def test_wide_multigrid_components_and_gmres(cuda, ref, case):
    cfg = _cfg(case)
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    M = api.SpaceTimeMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                               cfg.tau)
    R = ref.Reference(cfg, with_mg=True)
    info = R.level_info()
    assert [(g["mesh_level"], g["p"], g["k"], g["n_steps"]) for g in M.level_info()] == \
           [(w["mesh_level"], w["p"], w["k"], w["n_steps"]) for w in info]
    for l in range(M.n_levels - 1):
        n, nc = info[l]["n_dofs"], info[l + 1]["n_dofs"]
        res = problems.uniform_vector(n, seed=30 + l)
        z0 = problems.uniform_vector(n, seed=40 + l)
        got = M.asm_add_correction(l, _dev(cuda, res), _dev(cuda, z0)).cpu().numpy()
        assert _rel(got - z0, R.asm_add_correction(l, res, z0) - z0) <= 1e-9, f"asm level {l}"
        c = problems.uniform_vector(nc, seed=50 + l)
        assert _rel(M.prolong(l, _dev(cuda, c)).cpu().numpy(), R.prolong(l, c, n)) <= 1e-13, f"prolong {l}"
        assert _rel(M.restrict_(l, _dev(cuda, res)).cpu().numpy(), R.restrict_(l, res, nc)) <= 1e-13, f"restrict {l}"
    for l in range(M.n_levels):
        M.set_omega(l, R.omega(l))
    r = problems.uniform_vector(cfg.n_dofs, seed=60)
    assert _rel(M.apply(_dev(cuda, r)).cpu().numpy(), R.vcycle(r)) <= 1e-9
    b = R.assemble_rhs(1, 0.5, 0.0)
    x_ref, info_ref = R.gmres(b, rel_tol=1e-10, abs_tol=0.0)
    x = cuda.zeros(cfg.n_dofs, dtype=cuda.float64, device="cuda")
    res_info = M.solve(_dev(cuda, b), x, rel_tol=1e-10, abs_tol=0.0)
    assert res_info["converged"] and abs(res_info["iterations"] - info_ref["iterations"]) <= 1
    assert _rel(x.cpu().numpy(), x_ref) <= 1e-8
