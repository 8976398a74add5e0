"""GPU parity of the slab right-hand side, state transfer and nodal
interpolation (reference: space_time_operator.cpp:138-248,
spatial_operator.cpp:437-449) against the compiled reference."""
import numpy as np
import pytest

from paper_2408_04372_b200 import api, problems

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _pair(cfg, ref):
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    op = api.SpaceTimeOperator(mesh, cfg.refinements, cfg.p, cfg.equation, cfg.scheme, cfg.k, cfg.tau, cfg.n_steps,
                               cfg.rho)
    return mesh, op, ref.Reference(cfg)


@pytest.mark.parametrize("name,r", [("C1", None), ("C2", 2), ("C3", 1), ("C4", 0), ("C5-4", None)])
def test_assemble_rhs_manufactured(cuda, ref, name, r):
    cfg = problems.config(name, r)
    mesh, op, R = _pair(cfg, ref)
    u0 = problems.uniform_vector(op.n_space, seed=21)
    v0 = problems.uniform_vector(op.n_space, seed=22)
    want = R.assemble_rhs(1, 0.5, 0.125, u0, v0)
    got = op.assemble_rhs(1, 0.5, 0.125, cuda.from_numpy(u0).cuda(),
                          cuda.from_numpy(v0).cuda() if cfg.equation == 1 else None).cpu().numpy()
    assert _rel(got, want) <= 1e-12


@pytest.mark.parametrize("name,r", [("C1", None), ("C3", 1), ("C4", 0)])
def test_extract_final(cuda, ref, name, r):
    cfg = problems.config(name, r)
    mesh, op, R = _pair(cfg, ref)
    u = problems.uniform_vector(op.n_dofs, seed=31)
    u0 = problems.uniform_vector(op.n_space, seed=32)
    v0 = problems.uniform_vector(op.n_space, seed=33)
    uf_ref, vf_ref = R.extract_final(u, u0, v0)
    wave = cfg.equation == 1
    uf, vf = op.extract_final(cuda.from_numpy(u).cuda(), cuda.from_numpy(u0).cuda(),
                              cuda.from_numpy(v0).cuda() if wave else None)
    assert _rel(uf.cpu().numpy(), uf_ref) <= 1e-14
    if wave:
        assert _rel(vf.cpu().numpy(), vf_ref) <= 1e-12


@pytest.mark.parametrize("name,r", [("C2", 2), ("C4", 0)])
def test_gaussian_interpolation(cuda, ref, name, r):
    cfg = problems.config(name, r)
    mesh, op, R = _pair(cfg, ref)
    want = R.interpolate_gaussian((0.5, 0.5, 0.5), 0.05)
    got = op.interpolate(2, centre=(0.5, 0.5, 0.5), width=0.05).cpu().numpy()
    assert _rel(got, want) <= 1e-13


def test_fused_residual_matches_apply(cuda):
    cfg = problems.config("C2", 2)
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    op = api.SpaceTimeOperator(mesh, cfg.refinements, cfg.p, cfg.equation, cfg.scheme, cfg.k, cfg.tau, cfg.n_steps)
    g = cuda.Generator(device="cuda").manual_seed(3)
    u = cuda.rand(op.n_dofs, dtype=cuda.float64, device="cuda", generator=g)
    f = cuda.rand(op.n_dofs, dtype=cuda.float64, device="cuda", generator=g)
    r = op.residual(f, u)
    assert float(((r - (f - op.apply(u))).norm() / r.norm())) <= 1e-14
