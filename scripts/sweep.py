"""Per-configuration throughput of the two metric kernels (BASELINE.json
configs C1-C5): operator vmult and one STMG V-cycle, device-timed with CUDA
events on the launching stream after warm-up, vectors resident in HBM.
Prints one JSON line per configuration (DoF/s, ms, HBM fraction of the vmult's
algorithmic bytes 16 N (+ 24 n_verts perturbed) against MEASURED_PEAKS.json).

  python scripts/sweep.py [C1 C2 C3 C4 C5-32 C5-64 C5-128 C5-256v]
  (suffix v: vmult only; suffix n: vmult and V-cycle, no solve -- the
   Krylov basis of C5-256 does not fit one GPU)
"""
import gc
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2408_04372_b200 import api, problems  # noqa: E402


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main(names):
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    for name in names:
        vonly = name.endswith("v")
        nosolve = name.endswith("n")
        cname = name[:-1] if (vonly or nosolve) else name
        cfg = problems.config(cname)
        t0 = time.perf_counter()
        mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
        if vonly:
            op = api.SpaceTimeOperator(mesh, cfg.refinements, cfg.p, cfg.equation, cfg.scheme, cfg.k, cfg.tau,
                                       cfg.n_steps, cfg.rho)
            M = None
        else:
            # C5-256 on one GPU: the 20-vector Arnoldi basis of the relaxation
            # estimate (multigrid.cpp:127-172) does not fit next to the level
            # vectors, so omega is fixed to 1 there (the estimate's value on
            # every C5 level at the sizes where it runs)
            opts = {"eig_iters": 0} if nosolve else {}
            M = api.SpaceTimeMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k,
                                       cfg.n_steps, cfg.tau, **opts)
            op = M.operator_at(0)
        torch.cuda.synchronize()
        setup = time.perf_counter() - t0
        N = op.n_dofs
        u = torch.rand(N, dtype=torch.float64, device="cuda").mul_(2).sub_(1)
        y = torch.empty_like(u)
        reps = 3 if N > 5e8 else 10
        op.apply(u, y)
        t_v = timed(lambda: op.apply(u, y), reps)
        nv = (cfg.cells + 1) ** cfg.dim
        vbytes = 16 * N + (24 * nv if cfg.perturb > 0 else 0)
        line = {"config": name, **cfg.describe(), "setup_s": round(setup, 2), "vmult_ms": t_v,
                "omegas": [li["omega"] for li in M.level_info()] if M is not None else None,
                "vmult_dofs_per_s": N / (t_v * 1e-3), "vmult_hbm_frac": vbytes / (t_v * 1e-3) / 1e9 / peak}
        if M is not None:
            z = y  # the vmult output is reused (C5-256: four fine vectors would not fit)
            M.apply(u, z)
            t_c = timed(lambda: M.apply(u, z), max(3, reps // 2))
            vc_bytes = M.vcycle_bytes()
            line.update({"vcycle_ms": t_c, "vcycle_dofs_per_s": N / (t_c * 1e-3), "mg_levels": M.n_levels,
                         "vcycle_algorithmic_bytes": vc_bytes,
                         "vcycle_hbm_frac": vc_bytes / (t_c * 1e-3) / 1e9 / peak,
                         "smoother_kind_fine": M.smoother_kind(0), "device_bytes": M.device_bytes()})
            if nosolve:
                print(json.dumps(line), flush=True)
                del M, op, u, y, mesh, z
                torch.cuda.empty_cache()
                continue
            # one full STMG-GMRES solve (manufactured source; C4: the Gaussian pulse, zero source)
            u0 = torch.zeros(op.n_space, dtype=torch.float64, device="cuda")
            wave = cfg.equation == problems.WAVE
            if wave:
                u0 = op.interpolate(2, 0.5, 0.0, (0.5, 0.5, 0.5), 0.05, zero_boundary=True)
            v0 = torch.zeros_like(u0) if wave else None
            b = op.assemble_rhs(0 if wave else 1, 0.5, 0.0, u0, v0)
            x = torch.zeros_like(b)
            M.solve(b, x, rel_tol=1e-10, abs_tol=0.0)  # warm-up: Krylov basis allocated once
            x.zero_()
            torch.cuda.synchronize()
            ts = time.perf_counter()
            info = M.solve(b, x, rel_tol=1e-10, abs_tol=0.0)
            torch.cuda.synchronize()
            t_s = time.perf_counter() - ts
            line.update({"solve_iterations": info["iterations"], "solve_ms": 1e3 * t_s, "solve_dofs_per_s": N / t_s})
            del b, x, u0, v0, z
        print(json.dumps(line), flush=True)
        # every device buffer of this configuration is released before the
        # next one (C4's solve vectors left C5-128 out of memory otherwise)
        del M, op, u, y, mesh
        gc.collect()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5-32", "C5-64", "C5-128", "C5-256n"])
