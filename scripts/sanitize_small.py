"""Small vmult + smoother sweep for compute-sanitizer (racecheck/memcheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_04372_b200 import api, problems  # noqa: E402

for name, r in (("C2", 1), ("C3", 0)):
    cfg = problems.config(name, r)
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    M = api.SpaceTimeMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                               cfg.tau)
    op = M.operator_at(0)
    u = torch.rand(op.n_dofs, dtype=torch.float64, device="cuda")
    y = op.apply(u)
    z = torch.zeros_like(u)
    M.asm_add_correction(0, u, z)
    torch.cuda.synchronize()
    print(name, float(y.norm()), float(z.norm()))
