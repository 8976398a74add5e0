"""One warm STMG-GMRES solve inside a cudaProfilerStart/Stop range (ncu --profile-from-start off)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_04372_b200 import api, problems  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = problems.config(name)
mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
M = api.SpaceTimeMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                           cfg.tau)
op = M.operator_at(0)
b = op.assemble_rhs(1, 0.5, 0.0, torch.zeros(op.n_space, dtype=torch.float64, device="cuda"), None)
x = torch.zeros_like(b)
M.solve(b, x, rel_tol=1e-10, abs_tol=0.0)
x.zero_()
torch.cuda.synchronize()
torch.cuda.profiler.start()
M.solve(b, x, rel_tol=1e-10, abs_tol=0.0)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
