"""GPU parity of the fused space-time operator (SpaceTimeOperator::apply,
space_time_operator.cpp:45-130) against the reference oracle, through the C
ABI. Tolerance (north_star): relative L2 difference <= 1e-12."""
import numpy as np
import pytest

from paper_2408_04372_b200 import api, problems

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _pair(cfg, ref):
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    op = api.SpaceTimeOperator(mesh, cfg.refinements, cfg.p, cfg.equation, cfg.scheme, cfg.k, cfg.tau, cfg.n_steps,
                               cfg.rho)
    R = ref.Reference(cfg)
    assert op.n_dofs == R.n_dofs == cfg.n_dofs
    return mesh, op, R


@pytest.mark.parametrize("name,r", [("C1", None), ("C2", 2), ("C3", 1), ("C4", 0), ("C5-8", None)])
def test_config_vmult_parity(cuda, ref, name, r):
    cfg = problems.config(name, r)
    mesh, op, R = _pair(cfg, ref)
    u = problems.uniform_vector(op.n_dofs, seed=42)
    y = op.apply(cuda.from_numpy(u).cuda()).cpu().numpy()
    want = R.apply(u)
    assert _rel(y, want) <= TOL


CASES = []
for dim in (2, 3):
    for p in (1, 2, 3, 4):
        for eq in (0, 1):
            for scheme, k in ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2)):
                for S in (1, 2, 3):
                    nt = k + 1 if scheme == 0 else k
                    if S * nt > 8 or (dim == 3 and p == 4 and S > 1):
                        continue
                    CASES.append((dim, p, eq, scheme, k, S))


@pytest.mark.parametrize("dim,p,eq,scheme,k,S", CASES[::3])
@pytest.mark.parametrize("geom", ["cartesian", "cartesian+rho", "perturbed+rho"])
def test_vmult_parity_sweep(cuda, ref, dim, p, eq, scheme, k, S, geom):
    """Cartesian levels run the element-matrix kernel (st_cart.cuh), perturbed
    ones the quadrature form (st_lines.cuh / st_operator.cuh)."""
    base, refine = (2, 1) if dim == 3 else (3, 1)
    cfg = problems.Config("sweep", eq, scheme, dim, base, refine, p, k, S, 0.3)
    if geom.startswith("perturbed"):
        cfg.perturb = 0.15
    if geom.endswith("rho"):
        rng = np.random.default_rng(7)
        cfg.rho = rng.uniform(0.5, 3.0, base ** dim)
    mesh, op, R = _pair(cfg, ref)
    u = problems.uniform_vector(op.n_dofs, seed=3)
    y = op.apply(cuda.from_numpy(u).cuda()).cpu().numpy()
    assert _rel(y, R.apply(u)) <= TOL


# every field count of the Cartesian element-matrix kernel, both thread-group
# layouts (one group per line, and two when N * F > 20), heat and wave
CART_FIELDS = [(p, eq, scheme, k, S) for p in (1, 2, 3, 4)
               for eq, scheme, k, S in ((0, 0, 0, 1), (0, 0, 1, 1), (0, 0, 2, 1), (0, 0, 1, 2), (1, 1, 1, 5),
                                        (0, 0, 2, 2), (1, 1, 2, 7 // 2), (0, 0, 0, 7), (1, 1, 2, 4))]


@pytest.mark.parametrize("p,eq,scheme,k,S", CART_FIELDS)
def test_cartesian_vmult_every_field_count(cuda, ref, p, eq, scheme, k, S):
    cfg = problems.Config("cart", eq, scheme, 3, 3, 0, p, k, S, 0.2)
    rng = np.random.default_rng(p * 100 + S)
    cfg.rho = rng.uniform(0.5, 3.0, 27)
    mesh, op, R = _pair(cfg, ref)
    u = problems.uniform_vector(op.n_dofs, seed=5)
    y = op.apply(cuda.from_numpy(u).cuda()).cpu().numpy()
    assert _rel(y, R.apply(u)) <= TOL


@pytest.mark.parametrize("kind", [0, 1])
def test_spatial_operator_parity(cuda, ref, kind):
    cfg = problems.config("C2", 2)
    cfg.rho = np.array([2.5])
    mesh, op, R = _pair(cfg, ref)
    u = problems.uniform_vector(op.n_space, seed=11)
    y = op.spatial_apply(kind, cuda.from_numpy(u).cuda()).cpu().numpy()
    assert _rel(y, R.spatial_apply(kind, u)) <= TOL


def test_host_buffer_apply_and_linearity(cuda, ref):
    cfg = problems.config("C2", 2)
    mesh, op, R = _pair(cfg, ref)
    u = problems.uniform_vector(op.n_dofs, seed=5)
    v = problems.uniform_vector(op.n_dofs, seed=6)
    yu = op.apply_host(u)
    assert _rel(yu, R.apply(u)) <= TOL
    yuv = op.apply_host(2.0 * u - 3.0 * v)
    assert _rel(yuv, 2.0 * yu - 3.0 * op.apply_host(v)) <= 1e-13


def test_size_mismatch_raises(cuda):
    cfg = problems.config("C1", 1)
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements)
    op = api.SpaceTimeOperator(mesh, cfg.refinements, cfg.p, cfg.equation, cfg.scheme, cfg.k, cfg.tau, cfg.n_steps)
    with pytest.raises(ValueError):
        op.apply(cuda.zeros(op.n_dofs + 1, dtype=cuda.float64, device="cuda"))


def test_full_size_c2_properties(cuda):
    """C2 at full size (21.6M ST dofs): identity on Dirichlet rows, linearity
    and determinism-to-rounding across two applications."""
    cfg = problems.config("C2")
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    op = api.SpaceTimeOperator(mesh, cfg.refinements, cfg.p, cfg.equation, cfg.scheme, cfg.k, cfg.tau, cfg.n_steps)
    g = cuda.Generator(device="cuda").manual_seed(1)
    u = cuda.rand(op.n_dofs, dtype=cuda.float64, device="cuda", generator=g) * 2 - 1
    y1 = op.apply(u)
    y2 = op.apply(u)
    assert float((y1 - y2).norm() / y1.norm()) <= 1e-14
    d = cfg.cells * cfg.p + 1
    yv = y1.view(-1, d, d, d)
    uv = u.view(-1, d, d, d)
    assert cuda.equal(yv[:, 0], uv[:, 0]) and cuda.equal(yv[:, :, :, -1], uv[:, :, :, -1])
    y3 = op.apply(2.0 * u)
    assert float((y3 - 2.0 * y1).norm() / y1.norm()) <= 1e-14


def test_full_size_c5_256_translation_invariance(cuda):
    """C5 at 256^3 cells (4.31e9 ST dofs, vector indices beyond 2^32): the
    Cartesian constant-coefficient operator is translation invariant away
    from the boundary, so the same nodal bump placed near the start and near
    the end of the lattice must give the same output pattern in every
    temporal field -- any 32-bit index wrap would break it."""
    cfg = problems.config("C5-256")
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements)
    op = api.SpaceTimeOperator(mesh, cfg.refinements, cfg.p, cfg.equation, cfg.scheme, cfg.k, cfg.tau, cfg.n_steps)
    d = cfg.cells * cfg.p + 1
    F = cfg.n_steps * cfg.n_t
    u = cuda.zeros(op.n_dofs, dtype=cuda.float64, device="cuda")
    uv = u.view(F, d, d, d)
    g = cuda.Generator(device="cuda").manual_seed(3)
    bump = cuda.rand((F, 5, 5, 5), dtype=cuda.float64, device="cuda", generator=g)
    lo = 40  # both far from the boundary, hi near the end of the lattice, same offset mod p
    hi = (d - 60) - ((d - 60 - lo) % cfg.p)
    uv[:, lo:lo + 5, lo:lo + 5, lo:lo + 5] = bump
    uv[:, hi:hi + 5, hi:hi + 5, hi:hi + 5] = bump
    y = op.apply(u)
    del u, uv
    yv = y.view(F, d, d, d)
    w = 12  # window covering the bump's support (cells of width p)
    a = yv[:, lo - w:lo + 5 + w, lo - w:lo + 5 + w, lo - w:lo + 5 + w]
    b = yv[:, hi - w:hi + 5 + w, hi - w:hi + 5 + w, hi - w:hi + 5 + w]
    assert float(a.norm()) > 0
    assert float((a - b).norm() / a.norm()) <= 1e-13
    del y
    cuda.cuda.empty_cache()


# the owner-computes Cartesian kernel (st_brick.cu) runs every Cartesian level
# whose coefficient is constant on each z layer (C4, C5): p in {1, 2, 4}, every
# field count, tiles that end exactly on the lattice's end plane (12 cells)
# and partial tiles (10 cells), several z chunks
BRICK = [(p, eq, scheme, k, S, base, refine) for p in (1, 2, 4)
         for eq, scheme, k, S in ((0, 0, 0, 1), (0, 0, 1, 1), (0, 0, 2, 1), (0, 0, 3, 1), (1, 1, 1, 5),
                                  (1, 1, 2, 3), (0, 0, 0, 7), (0, 0, 1, 4))
         for base, refine in ((3, 2), (5, 1))]


def _layered_rho(base, seed):
    rng = np.random.default_rng(seed)
    layer = rng.uniform(0.5, 4.0, base)
    return np.repeat(layer, base * base)


@pytest.mark.parametrize("p,eq,scheme,k,S,base,refine", BRICK)
def test_brick_vmult_and_residual_parity(cuda, ref, p, eq, scheme, k, S, base, refine):
    cfg = problems.Config("brick", eq, scheme, 3, base, refine, p, k, S, 0.2)
    cfg.rho = _layered_rho(base, p * 10 + S)
    mesh, op, R = _pair(cfg, ref)
    u = problems.uniform_vector(op.n_dofs, seed=5)
    f = problems.uniform_vector(op.n_dofs, seed=6)
    want = R.apply(u)
    ud = cuda.from_numpy(u).cuda()
    y = op.apply(ud).cpu().numpy()
    assert _rel(y, want) <= TOL
    r = op.residual(cuda.from_numpy(f).cuda(), ud).cpu().numpy()
    assert _rel(r, f - want) <= TOL


def test_brick_c5_64_parity(cuda, ref):
    """C5 at 64^3 cells (67.9 M ST dofs, 4 x 4 tiles of 16^2 nodes x z chunks)
    against the reference's own apply."""
    cfg = problems.config("C5-64")
    mesh, op, R = _pair(cfg, ref)
    u = problems.uniform_vector(op.n_dofs, seed=42)
    y = op.apply(cuda.from_numpy(u).cuda()).cpu().numpy()
    assert _rel(y, R.apply(u)) <= TOL
