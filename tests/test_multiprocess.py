"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host logic:
max-over-ranks step timing and whole-job throughput of the replica bench, and
the z-slab partition of the lattice."""
import os

import pytest
import torch.multiprocessing as mp

from paper_2408_04372_b200 import dist as sdist


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ms_local = 10.0 + 5.0 * rank  # rank 1 is the slow one
        value, ms = sdist.aggregate_throughput(1000.0, ms_local)
        out[rank] = (value, ms)
    finally:
        dist.destroy_process_group()


def test_replica_aggregation_gloo_world2():
    mgr = mp.Manager()
    out = mgr.dict()
    port = 29500 + os.getpid() % 1000
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in (0, 1):
        value, ms = out[r]
        assert ms == 15.0  # max over ranks
        assert value == pytest.approx(2 * 1000.0 / 15e-3)


@pytest.mark.parametrize("layers,world,p", [(64, 1, 3), (64, 2, 3), (64, 8, 3), (96, 8, 4), (7, 3, 2)])
def test_slab_partition_covers_lattice_once(layers, world, p):
    planes = []
    cells = []
    for r in range(world):
        part = sdist.slab_partition(layers, world, r, p)
        planes.extend(range(*part["planes"]))
        cells.extend(range(*part["cells"]))
        assert part["halo_low"] == (r > 0) and part["halo_high"] == (r < world - 1)
    assert planes == list(range(layers * p + 1))
    assert cells == list(range(layers))


def test_slab_partition_rejects_too_many_ranks():
    with pytest.raises(ValueError):
        sdist.slab_partition(4, 8, 0, 2)


# ---- the partitioned solve's plan, from the C ABI (host only, no GPU)
@pytest.mark.parametrize("name,refine,parts,want", [
    ("C2", 6, 8, 3),   # 64 layers: 8/4/2 per part stay partitioned, 1 does not (next step is h)
    ("C2", 6, 2, 5),   # 32/16/8/4/2
    ("C2", 6, 1, 8),   # one part: everything but the coarsest level
    ("C3", 4, 8, 6),   # 128 layers: 16/8/4/2/1 on h levels, 1 stays for the tau step
    ("C4", 5, 8, 2),   # 96 layers: 12/6, then 3 is odd before another h step
])
def test_slab_plan_levels(name, refine, parts, want):
    from paper_2408_04372_b200 import api, problems
    cfg = problems.config(name, refine)
    d, n = api.slab_plan(cfg.scheme, cfg.refinements, cfg.p, cfg.k, cfg.n_steps, cfg.cells, parts)
    assert d == want and 1 <= d < n


def test_slab_plan_rejects_uneven_split():
    from paper_2408_04372_b200 import api, problems
    cfg = problems.config("C2", 6)
    with pytest.raises(ValueError):
        api.slab_plan(cfg.scheme, cfg.refinements, cfg.p, cfg.k, cfg.n_steps, cfg.cells, 3)


def _slab_worker(rank, world, port, out):
    """Each rank derives its parts of the partition the way bench.py does and
    the ranks agree (gloo all_gather) that the parts tile the finest lattice."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        part = sdist.slab_partition(64, world, rank, 3)
        t = torch.tensor([part["cells"][0], part["cells"][1], part["planes"][0], part["planes"][1]])
        allp = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allp, t)
        out[rank] = [a.tolist() for a in allp]
    finally:
        dist.destroy_process_group()


def test_slab_partition_agreed_over_gloo_world2():
    mgr = mp.Manager()
    out = mgr.dict()
    port = 29600 + os.getpid() % 1000
    mp.spawn(_slab_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] == out[1]
    (c0, c1, g0, g1), (d0, d1, h0, h1) = out[0]
    assert (c0, c1, d0, d1) == (0, 32, 32, 64) and (g0, g1, h0, h1) == (0, 96, 96, 193)
