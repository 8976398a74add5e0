"""Times the operator apply / residual (and optionally the fine smoother) of
one or more workloads with CUDA events: python scripts/time_ops.py C5-128 C4 [--asm]"""
import os
import sys

ROOT = os.environ.get("STMG_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2408_04372_b200 import api, problems  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    names = [a for a in sys.argv[1:] if not a.startswith("--")]
    for name in names or ["C5-128"]:
        cfg = problems.config(name)
        mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
        op = api.SpaceTimeOperator(mesh, cfg.refinements, cfg.p, cfg.equation, cfg.scheme, cfg.k, cfg.tau,
                                   cfg.n_steps, cfg.rho)
        g = torch.Generator(device="cuda").manual_seed(1)
        u = torch.rand(op.n_dofs, dtype=torch.float64, device="cuda", generator=g)
        f = torch.rand(op.n_dofs, dtype=torch.float64, device="cuda", generator=g)
        y = torch.empty_like(u)
        ta = timed(lambda: op.apply(u, y))
        tr = timed(lambda: op.residual(f, u, y))
        N = op.n_dofs
        gbs = 16 * N / (ta * 1e-3) / 1e9
        line = f"{name}: N={N} apply {ta:.3f} ms ({gbs:.0f} GB/s alg, {N / ta / 1e6:.1f} GDoF/s) residual {tr:.3f} ms"
        if "--xfer" in sys.argv:
            M = api.SpaceTimeMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k,
                                       cfg.n_steps, cfg.tau)
            nc = M.level_info()[1]["n_dofs"]
            c = torch.rand(nc, dtype=torch.float64, device="cuda", generator=g)
            tr_ = timed(lambda: M.restrict_(0, u, c))
            tp_ = timed(lambda: M.prolong(0, c, y))
            tv_ = timed(lambda: M.apply(u, y), 5)
            line += f" restrict {tr_:.3f} ms prolong {tp_:.3f} ms vcycle {tv_:.3f} ms"
            del M, c
        if "--asm" in sys.argv:
            sm = api.ASMSmoother(op)
            z = torch.zeros_like(u)
            line += f" asm {timed(lambda: sm.add_correction(u, z), 5):.3f} ms"
        print(line, flush=True)
        del op, u, f, y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
