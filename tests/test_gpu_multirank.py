"""The per-rank path of the z-slab partitioned solve
with TWO processes: each rank holds one slab (first_part = rank,
local_parts = 1) and the interface exchanges / allreduces cross processes
through the host-staged communicator (api.Comm.host over a gloo process
group). This pool gives one GPU per call, so both ranks share cuda:0; the
NCCL communicator takes the same code path with device buffers.

Oracle: the unpartitioned device path of the same process (itself pinned
against the reference in test_gpu_operator.py / test_gpu_multigrid.py).
Bars: operator 1e-12 and smoother 1e-11 (interface summation order only),
V-cycle 1e-10, GMRES iterations +-1 and solution 1e-8."""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CASES = [("C5-8", None), ("C3", 1), ("C2", 3)]


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _rank(rank, world, port, name, r, out):
    import torch
    import torch.distributed as dist

    from paper_2408_04372_b200 import api, problems
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        cfg = problems.config(name, r)
        mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
        G = api.SpaceTimeMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k,
                                   cfg.n_steps, cfg.tau)
        comm = api.Comm.host()
        S = api.SlabMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                              cfg.tau, world, first_part=rank, local_parts=1, comm=comm)
        res = {"dist_levels": S.dist_levels}

        def full(a):
            return torch.from_numpy(np.ascontiguousarray(a)).cuda()

        def collect(local):
            """the owned planes of every rank's slab summed into one full vector"""
            f = S.gather(local, torch.zeros(cfg.n_dofs, dtype=torch.float64, device="cuda")).cpu()
            dist.all_reduce(f)
            return f.numpy()

        u = full(problems.uniform_vector(cfg.n_dofs, seed=21))
        res["apply"] = _rel(collect(S.apply(S.scatter(u))), G.operator_at(0).apply(u).cpu().numpy())
        z0 = full(problems.uniform_vector(cfg.n_dofs, seed=23))
        want = (G.asm_add_correction(0, u, z0.clone()) - z0).cpu().numpy()
        got = collect(S.asm_add_correction(S.scatter(u), S.scatter(z0))) - z0.cpu().numpy()
        res["asm"] = _rel(got, want)
        res["omega"] = max(abs(S.omega_at(l) - G.omega_at(l)) / G.omega_at(l) for l in range(G.n_levels))
        for l in range(G.n_levels):
            S.set_omega(l, G.omega_at(l))
        res["vcycle"] = _rel(collect(S.vcycle(S.scatter(u))), G.apply(u).cpu().numpy())
        op = G.operator_at(0)
        u0 = torch.zeros(op.n_space, dtype=torch.float64, device="cuda")
        v0 = torch.zeros_like(u0) if cfg.equation == problems.WAVE else None
        b = op.assemble_rhs(1, 0.5, 0.0, u0, v0)
        xg = torch.zeros_like(b)
        ig = G.solve(b, xg, rel_tol=1e-10, abs_tol=0.0)
        xl = torch.zeros(S.n_local, dtype=torch.float64, device="cuda")
        info = S.solve(S.scatter(b), xl, rel_tol=1e-10, abs_tol=0.0)
        res["iters"] = (info["iterations"], ig["iterations"], info["converged"])
        res["solution"] = _rel(collect(xl), xg.cpu().numpy())
        out[rank] = res
        del S, G, comm
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,r", CASES)
def test_two_rank_host_staged_partition(cuda, name, r):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = 29600 + (os.getpid() + len(name) * 7 + (r or 0)) % 300
    mp.start_processes(_rank, args=(2, port, name, r, out), nprocs=2, join=True, start_method="spawn")
    for rank in (0, 1):
        res = out[rank]
        assert res["dist_levels"] >= 1
        assert res["apply"] <= 1e-12, res
        assert res["asm"] <= 1e-11, res
        assert res["omega"] <= 1e-8, res
        assert res["vcycle"] <= 1e-10, res
        it, it_g, conv = res["iters"]
        assert conv and abs(it - it_g) <= 1, res
        assert res["solution"] <= 1e-8, res
