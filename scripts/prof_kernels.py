"""Small driver for ncu: builds a workload and runs the hot kernels inside a
cudaProfilerStart/Stop range (use ncu --profile-from-start off).

  python scripts/prof_kernels.py kernels [C2]   # vmult x3 + fine ASM x3
  python scripts/prof_kernels.py step [C2]      # 2 bench steps (V-cycle + vmult)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2408_04372_b200 import api, problems  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "kernels"
    name = sys.argv[2] if len(sys.argv) > 2 else "C2"
    cfg = problems.config(name)
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    g = torch.Generator(device="cuda").manual_seed(1)
    if mode == "kernels":
        op = api.SpaceTimeOperator(mesh, cfg.refinements, cfg.p, cfg.equation, cfg.scheme, cfg.k, cfg.tau,
                                   cfg.n_steps, cfg.rho)
        sm = api.ASMSmoother(op)
        u = torch.rand(op.n_dofs, dtype=torch.float64, device="cuda", generator=g)
        y = torch.empty_like(u)
        z = torch.zeros_like(u)
        op.apply(u, y)
        sm.add_correction(u, z)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        for _ in range(3):
            op.apply(u, y)
        for _ in range(3):
            sm.add_correction(u, z)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    else:
        M = api.SpaceTimeMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k,
                                   cfg.n_steps, cfg.tau)
        op = M.operator_at(0)
        r = torch.rand(op.n_dofs, dtype=torch.float64, device="cuda", generator=g)
        z, y = torch.empty_like(r), torch.empty_like(r)
        M.apply(r, z)
        op.apply(z, y)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        for _ in range(2):
            M.apply(r, z)
            op.apply(z, y)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    print("done")


if __name__ == "__main__":
    main()
