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
