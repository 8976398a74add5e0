"""GPU march (driver.cpp:95-260) and error norms (driver.cpp:18-92,
spatial_operator.cpp:526-557) against the reference: the reference's march
loop is composed from its own assemble_rhs / gmres / error_norms /
extract_final on the same mesh and slab operator (march() itself builds its
mesh from a ProblemSpec and cannot take the BASELINE perturbation), then
compared batch by batch: GMRES iterations within +-1, error norms 1e-6
relative (they differ only through the solves' rounding), final state 1e-8."""
import numpy as np
import pytest

from paper_2408_04372_b200 import api, problems

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _ref_march(R, n_batches, u0, v0, frequency, source_kind, wave, slab_time):
    its, acc = [], np.zeros(3)
    l2sq = 0.0
    u, v = u0.copy(), (v0.copy() if wave else None)
    for b in range(n_batches):
        t0 = b * slab_time
        rhs = R.assemble_rhs(source_kind, frequency, t0, u, v)
        x, info = R.gmres(rhs, rel_tol=1e-10, abs_tol=0.0)
        its.append(info["iterations"])
        if not wave:
            e = R.error_norms(x, u, frequency, t0)
            l2sq += e[0] ** 2
            acc[1] = max(acc[1], e[1])
            acc[2] = max(acc[2], e[2])
        u, vf = R.extract_final(x, u, v)
        v = vf if wave else None
    acc[0] = np.sqrt(l2sq)
    return its, acc, u, v


@pytest.mark.parametrize("name,r,n_batches", [("C1", None, 3), ("C1", 2, 4), ("C2", 2, 2), ("C3", 0, 2)])
def test_march_heat_matches_reference(cuda, ref, name, r, n_batches):
    cfg = problems.config(name, r)
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    M = api.SpaceTimeMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                               cfg.tau)
    R = ref.Reference(cfg, with_mg=True)
    n_space = M.operator_at(0).n_space
    its_ref, err_ref, uf_ref, _ = _ref_march(R, n_batches, np.zeros(n_space), None, 0.5, 1, False,
                                              cfg.n_steps * cfg.tau)
    u = cuda.zeros(n_space, dtype=cuda.float64, device="cuda")
    out = M.march(n_batches, u, source_kind=1, frequency=0.5, rel_tol=1e-10, abs_tol=0.0)
    assert all(abs(a - b) <= 1 for a, b in zip(out["iterations"], its_ref)), (out["iterations"], its_ref)
    for got, want in zip(out["error_u"], err_ref):
        assert abs(got - want) <= 1e-6 * want + 1e-14
    assert _rel(u.cpu().numpy(), uf_ref) <= 1e-8


def test_march_wave_gaussian_matches_reference(cuda, ref):
    """C4 shape (wave, CGP(2), 4 steps per slab, Q4, layered rho) at the
    coarsest mesh with the Gaussian pulse: iterations and final state."""
    cfg = problems.config("C4", 0)
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    M = api.SpaceTimeMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                               cfg.tau)
    R = ref.Reference(cfg, with_mg=True)
    u0 = R.interpolate_gaussian((0.5, 0.5, 0.5), 0.05)
    v0 = np.zeros_like(u0)
    its_ref, _, uf_ref, vf_ref = _ref_march(R, 2, u0, v0, 0.5, 0, True, cfg.n_steps * cfg.tau)
    u = cuda.from_numpy(u0.copy()).cuda()
    v = cuda.zeros_like(u)
    out = M.march(2, u, v, source_kind=0, errors=False, rel_tol=1e-10, abs_tol=0.0)
    assert all(abs(a - b) <= 1 for a, b in zip(out["iterations"], its_ref)), (out["iterations"], its_ref)
    assert _rel(u.cpu().numpy(), uf_ref) <= 1e-8
    assert _rel(v.cpu().numpy(), vf_ref) <= 1e-8


@pytest.mark.parametrize("name,r", [("C1", 2), ("C2", 2)])
def test_error_norms_match_reference(cuda, ref, name, r):
    """error_norms of one and the same batch vector (the reference's own
    solution) on the device vs the reference: 1e-10 relative."""
    cfg = problems.config(name, r)
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    op = api.SpaceTimeOperator(mesh, cfg.refinements, cfg.p, cfg.equation, cfg.scheme, cfg.k, cfg.tau, cfg.n_steps)
    R = ref.Reference(cfg, with_mg=True)
    u0 = np.zeros(op.n_space)
    x, _ = R.gmres(R.assemble_rhs(1, 0.5, 0.0, u0), rel_tol=1e-10, abs_tol=0.0)
    want = R.error_norms(x, u0, 0.5, 0.0)
    got = op.error_norms(cuda.from_numpy(x).cuda(), cuda.from_numpy(u0).cuda(), 0.5, 0.0)
    for g, w in zip(got, want):
        assert abs(g - w) <= 1e-10 * w + 1e-15


def test_march_heat_converges_at_the_expected_order(cuda):
    """Heat 2D Q2 dG(1) manufactured solution over t in [0, 1]: refining h
    and tau together, the L2(L2) error converges at order min(p+1, k+1) = 2
    (checked >= 1.8 per refinement)."""
    errs = []
    for r in (2, 3, 4):
        cfg = problems.Config("eoc", problems.HEAT, problems.DG, 2, 1, r, 2, 1, 1, 0.5 / (1 << r))
        mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements)
        M = api.SpaceTimeMultigrid(cfg.equation, cfg.scheme, mesh, None, cfg.refinements, cfg.p, cfg.k, 1, cfg.tau)
        u = cuda.zeros(M.operator_at(0).n_space, dtype=cuda.float64, device="cuda")
        out = M.march(1 << (r + 1), u, source_kind=1, frequency=0.5, rel_tol=1e-12, abs_tol=0.0)
        errs.append(out["error_u"][0])
    rates = [np.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert all(rt >= 1.8 for rt in rates), (errs, rates)


@pytest.mark.parametrize("name,r,n_batches", [("C1", 2, 3), ("C2", 2, 2)])
def test_march_probes_match_reference(cuda, ref, name, r, n_batches):
    """Probe time series (locate_point + value_at + evaluate_fe at every
    sample, driver.cpp:146-236) of the device march vs the reference's own
    functions on the reference's batch solutions: 1e-8 of the series' scale."""
    cfg = problems.config(name, r)
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    M = api.SpaceTimeMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                               cfg.tau)
    R = ref.Reference(cfg, with_mg=True)
    pts = np.array([[0.31, 0.47, 0.5], [0.73, 0.22, 0.61], [0.5, 0.5, 0.5]])
    if cfg.dim == 2:
        pts[:, 2] = 0.0
    ns = 4
    u = cuda.zeros(M.operator_at(0).n_space, dtype=cuda.float64, device="cuda")
    out = M.march_probes(n_batches, u, pts, samples_per_step=ns, rel_tol=1e-10, abs_tol=0.0)
    # the reference series on its own march loop
    n_space = M.operator_at(0).n_space
    uu = np.zeros(n_space)
    want = [[0.0] for _ in pts]  # the entering state u(0) = 0
    times = [0.0]
    for b in range(n_batches):
        t0 = b * cfg.n_steps * cfg.tau
        x, _ = R.gmres(R.assemble_rhs(1, 0.5, t0, uu), rel_tol=1e-10, abs_tol=0.0)
        for st in range(cfg.n_steps):
            for j in range(1, ns + 1):
                for pi, xp in enumerate(pts):
                    want[pi].append(R.probe_value(x, uu, st, j / ns, xp))
                times.append(t0 + (st + j / ns) * cfg.tau)
        uu, _ = R.extract_final(x, uu)
    want = np.array(want)
    assert np.allclose(out["times"], times, rtol=0, atol=1e-14)
    scale = float(np.abs(want).max())
    assert scale > 0
    assert float(np.abs(out["values"] - want).max()) <= 1e-8 * scale
