"""GPU parity of the z-slab partitioned solve run as
several parts in ONE process on one GPU -- the same partitioned algorithm
(interface sums, owner rules, replicated coarse tail) the multi-rank run
executes, with in-process interface sums instead of NCCL exchanges.

Oracle: the unpartitioned device path, itself pinned against the reference
(test_gpu_operator.py, test_gpu_multigrid.py), and the reference's GMRES for
the solve. Bars: operator and smoother 1e-12 / 1e-11 (only the summation order
at interface planes differs), V-cycle 1e-10, relaxation factors 1e-8, GMRES
iterations within +-1 of the reference and solution 1e-8."""
import numpy as np
import pytest

from paper_2408_04372_b200 import api, problems

pytestmark = pytest.mark.gpu

CASES = [("C2", 2, 2), ("C2", 3, 2), ("C2", 3, 4), ("C3", 1, 2), ("C3", 1, 4), ("C5-8", None, 2)]


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _pair(cfg, n_parts):
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    G = api.SpaceTimeMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                               cfg.tau)
    S = api.SlabMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                          cfg.tau, n_parts)
    return mesh, G, S


def _full(cuda, a):
    return cuda.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("name,r,parts", CASES)
def test_slab_operator_matches_global(cuda, name, r, parts):
    cfg = problems.config(name, r)
    mesh, G, S = _pair(cfg, parts)
    assert S.dist_levels >= 1 and len(S.parts) == parts
    u = _full(cuda, problems.uniform_vector(cfg.n_dofs, seed=21))
    want = G.operator_at(0).apply(u)
    yl = S.apply(S.scatter(u))
    got = S.gather(yl, cuda.zeros_like(u))
    assert _rel(got.cpu().numpy(), want.cpu().numpy()) <= 1e-12
    # both copies of every interface plane hold the assembled value
    again = S.scatter(got)
    assert _rel(again.cpu().numpy(), yl.cpu().numpy()) <= 1e-13


@pytest.mark.parametrize("name,r,parts", CASES)
def test_slab_smoother_matches_global(cuda, name, r, parts):
    cfg = problems.config(name, r)
    mesh, G, S = _pair(cfg, parts)
    res = _full(cuda, problems.uniform_vector(cfg.n_dofs, seed=22))
    z0 = _full(cuda, problems.uniform_vector(cfg.n_dofs, seed=23))
    want = G.asm_add_correction(0, res, z0.clone())
    zl = S.asm_add_correction(S.scatter(res), S.scatter(z0))
    got = S.gather(zl, cuda.zeros_like(res))
    assert _rel((got - z0).cpu().numpy(), (want - z0).cpu().numpy()) <= 1e-11


@pytest.mark.parametrize("name,r,parts", CASES)
def test_slab_relaxation_and_vcycle_match_global(cuda, name, r, parts):
    cfg = problems.config(name, r)
    mesh, G, S = _pair(cfg, parts)
    for l in range(G.n_levels):
        assert abs(S.omega_at(l) - G.omega_at(l)) <= 1e-8 * G.omega_at(l), f"omega level {l}"
        S.set_omega(l, G.omega_at(l))
    res = _full(cuda, problems.uniform_vector(cfg.n_dofs, seed=24))
    want = G.apply(res)
    got = S.gather(S.vcycle(S.scatter(res)), cuda.zeros_like(res))
    assert _rel(got.cpu().numpy(), want.cpu().numpy()) <= 1e-10


@pytest.mark.parametrize("name,r,parts", [("C2", 3, 2), ("C2", 3, 4), ("C3", 1, 4)])
def test_slab_gmres_matches_reference(cuda, ref, name, r, parts):
    cfg = problems.config(name, r)
    mesh, G, S = _pair(cfg, parts)
    R = ref.Reference(cfg, with_mg=True)
    b = R.assemble_rhs(1, 0.5, 0.0)
    x_ref, info_ref = R.gmres(b, rel_tol=1e-10, abs_tol=0.0)
    bl = S.scatter(_full(cuda, b))
    xl = cuda.zeros(S.n_local, dtype=cuda.float64, device="cuda")
    info = S.solve(bl, xl, rel_tol=1e-10, abs_tol=0.0)
    assert info["converged"] and abs(info["iterations"] - info_ref["iterations"]) <= 1
    x = S.gather(xl, cuda.zeros(cfg.n_dofs, dtype=cuda.float64, device="cuda")).cpu().numpy()
    assert _rel(x, x_ref) <= 1e-8


def test_slab_dot_counts_interfaces_once(cuda):
    cfg = problems.config("C2", 3)
    mesh, G, S = _pair(cfg, 4)
    a = problems.uniform_vector(cfg.n_dofs, seed=25)
    b = problems.uniform_vector(cfg.n_dofs, seed=26)
    got = S.dot(S.scatter(_full(cuda, a)), S.scatter(_full(cuda, b)))
    assert abs(got - float(a @ b)) <= 1e-12 * abs(float(np.abs(a) @ np.abs(b)))


def test_slab_rejects_uneven_partition(cuda):
    cfg = problems.config("C2", 2)  # 4 cell layers
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    with pytest.raises(ValueError):
        api.SlabMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                          cfg.tau, 3)


def test_slab_with_nccl_comm_world1(cuda):
    """The NCCL communicator path (dlopen'd libnccl, world 1: exchanges and
    allreduces are no-ops) gives the single-process result."""
    cfg = problems.config("C2", 1)
    uid = api.Comm.unique_id()
    assert len(uid) == 128
    comm = api.Comm(1, 0, uid)
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    G = api.SpaceTimeMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                               cfg.tau)
    S = api.SlabMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                          cfg.tau, 1, first_part=0, local_parts=1, comm=comm)
    u = _full(cuda, problems.uniform_vector(cfg.n_dofs, seed=27))
    assert _rel(S.apply(u).cpu().numpy(), G.operator_at(0).apply(u).cpu().numpy()) <= 1e-12
    assert S.dot(u, u) == pytest.approx(float((u * u).sum()), rel=1e-12)


def test_weak_scaling_box_partition(cuda):
    """The N = 2 weak-scaling box of bench.py (C5: Q4 dG(3), box mesh of
    1 x 1 x 2 base cells; here refined to 64 x 64 x 128 cells, 1.36e8 ST dofs,
    so that the unpartitioned and the partitioned hierarchies fit one GPU
    together) cut into two z-slabs held by this process: operator and V-cycle
    against the unpartitioned solve of the same box mesh (1e-12 / 1e-10)."""
    from paper_2408_04372_b200 import dist as sdist
    base = problems.config("C5-64")
    box = sdist.weak_box(2)
    mesh = api.Mesh(3, (0, 0, 0), tuple(float(b) for b in box), box, base.refinements)
    G = api.SpaceTimeMultigrid(base.equation, base.scheme, mesh, None, base.refinements, base.p, base.k,
                               base.n_steps, base.tau)
    S = api.SlabMultigrid(base.equation, base.scheme, mesh, None, base.refinements, base.p, base.k, base.n_steps,
                          base.tau, 2)
    assert S.dist_levels >= 2
    for l in range(G.n_levels):
        assert abs(S.omega_at(l) - G.omega_at(l)) <= 1e-8 * G.omega_at(l)
        S.set_omega(l, G.omega_at(l))
    n = G.operator_at(0).n_dofs
    g = cuda.Generator(device="cuda").manual_seed(8)
    u = cuda.rand(n, dtype=cuda.float64, device="cuda", generator=g) * 2 - 1
    want = G.operator_at(0).apply(u)
    got = S.gather(S.apply(S.scatter(u)), cuda.zeros_like(u))
    assert float((got - want).norm() / want.norm()) <= 1e-12
    del want, got
    want = G.apply(u)
    got = S.gather(S.vcycle(S.scatter(u)), cuda.zeros_like(u))
    assert float((got - want).norm() / want.norm()) <= 1e-10
