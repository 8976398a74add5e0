"""Time one warm STMG-GMRES solve and its parts (for GMRES overhead analysis):
  python scripts/solve_profile.py C5-32"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_04372_b200 import api, native, problems  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5-32"
cfg = problems.config(name)
mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
M = api.SpaceTimeMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                           cfg.tau)
op = M.operator_at(0)
u0 = torch.zeros(op.n_space, dtype=torch.float64, device="cuda")
b = op.assemble_rhs(1, 0.5, 0.0, u0, None)
x = torch.zeros_like(b)
M.solve(b, x, rel_tol=1e-10, abs_tol=0.0)
lib = native.load()
for rep in range(2):
    x.zero_()
    torch.cuda.synchronize()
    l0 = lib.stmg_kernel_launches()
    t0 = time.perf_counter()
    info = M.solve(b, x, rel_tol=1e-10, abs_tol=0.0)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    print(f"solve: {info['iterations']} it, {1e3 * t:.1f} ms, launches {lib.stmg_kernel_launches() - l0}")
z = torch.empty_like(b)
y = torch.empty_like(b)
for fn, nm in ((lambda: M.apply(b, z), "vcycle"), (lambda: op.apply(b, y), "vmult")):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    print(f"{nm}: {1e2 * (time.perf_counter() - t0):.3f} ms (wall, 10 reps)")
