"""Spatial h-transfers at sizes where the fused z-marching kernels run
(csrc/transfer.cu xyz_restrict_kernel / xyz_prolong_kernel: equal p on all
axes, fine planes of >= 2^16 nodes and >= 64 of them), against
oracle/stmg_np.Transfer -- the restatement of the reference's Transfer
(transfer.cpp:58-190), pinned against the compiled reference in
tests/test_oracle_np.py -- at C5-64 (1e-13), plus full-size properties at
C5-128 and C4 (adjointness <R f, c> = <f, P c>, the reference's own transfer
property, and exact prolongation of a per-cell polynomial), and the z-slab
partitioned V-cycle at C5-128 (its slab interface options run through the
fused kernels) against the unpartitioned one."""
import types

import numpy as np
import pytest

from oracle import stmg_np
from paper_2408_04372_b200 import api, problems

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _level(cfg, cells, p, F):
    d = cells * p + 1
    idx = np.indices((d, d, d)).reshape(3, -1)[::-1]  # x fastest
    bdry = np.any((idx == 0) | (idx == d - 1), axis=0)
    sp = types.SimpleNamespace(p=p, dim=3, dofs=d, bdry=bdry)
    return types.SimpleNamespace(sp=sp, nx=d ** 3, S=1, w=None)


def _mg(cfg):
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    M = api.SpaceTimeMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                               cfg.tau)
    return mesh, M


def test_fused_transfers_match_restatement_c5_64(cuda):
    cfg = problems.config("C5-64")
    mesh, M = _mg(cfg)
    info = M.level_info()
    F = cfg.n_steps * cfg.n_t
    fine, coarse = _level(cfg, 64, cfg.p, F), _level(cfg, 32, cfg.p, F)
    T = stmg_np.Transfer(fine, coarse, 64, 32)
    c = problems.uniform_vector(info[1]["n_dofs"], seed=5)
    f = problems.uniform_vector(info[0]["n_dofs"], seed=6)
    pf = M.prolong(0, cuda.from_numpy(c).cuda()).cpu().numpy()
    rc = M.restrict_(0, cuda.from_numpy(f).cuda()).cpu().numpy()
    assert _rel(pf, T.prolong(c)) <= 1e-13
    assert _rel(rc, T.restrict(f)) <= 1e-13


@pytest.mark.parametrize("name", ["C5-128", "C4"])
def test_fused_transfers_full_size_properties(cuda, name):
    cfg = problems.config(name)
    mesh, M = _mg(cfg)
    info = M.level_info()
    nf, nc = info[0]["n_dofs"], info[1]["n_dofs"]
    g = cuda.Generator(device="cuda").manual_seed(3)
    f = cuda.rand(nf, dtype=cuda.float64, device="cuda", generator=g) * 2 - 1
    c = cuda.rand(nc, dtype=cuda.float64, device="cuda", generator=g) * 2 - 1
    lhs = float(cuda.dot(M.restrict_(0, f), c))
    pc = M.prolong(0, c)
    rhs = float(cuda.dot(f, pc))
    scale = float(f.norm() * pc.norm())
    assert abs(lhs - rhs) <= 1e-12 * scale
    # exactness: the coarse nodal values of q(x,y,z) = x(1-x) y(1-y) z(1-z)
    # (degree 2 per axis <= p, zero on the boundary) prolongate to the fine
    # nodal values of q in every field
    F = cfg.n_steps * cfg.n_t
    p = cfg.p

    def nodal(cells):
        gl = stmg_np.gauss_lobatto(p + 1)[0]
        x = np.concatenate([(np.arange(cells)[:, None] + gl[None, :p]).ravel(), [cells]]) / cells
        q = x * (1 - x)
        v = (q[None, None, :] * q[None, :, None] * q[:, None, None]).ravel()
        return np.tile(v, F)
    nce = cfg.cells // 2
    cq = cuda.from_numpy(nodal(nce)).cuda()
    fq = M.prolong(0, cq).cpu().numpy()
    want = nodal(cfg.cells)
    assert _rel(fq, want) <= 1e-13


def test_slab_vcycle_full_c5_128(cuda):
    cfg = problems.config("C5-128")
    mesh, G = _mg(cfg)
    S = api.SlabMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                          cfg.tau, 2)
    for l in range(G.n_levels):
        S.set_omega(l, G.omega_at(l))
    g = cuda.Generator(device="cuda").manual_seed(4)
    r = cuda.rand(G.operator_at(0).n_dofs, dtype=cuda.float64, device="cuda", generator=g) * 2 - 1
    want = G.apply(r)
    got = S.gather(S.vcycle(S.scatter(r)), cuda.zeros_like(r))
    assert float((got - want).norm() / want.norm()) <= 1e-10
