"""Multi-GPU plumbing for the STMG path (one process per GPU, torch.distributed).

The partitioned solve (csrc/slab_mg.cpp): the finest
mesh is cut into z-slabs, one per rank; NCCL (or the host-staged transport,
api.Comm.host) carries the interface-plane sums and the dot-product /
coarse-vector allreduces. Here: the rank environment, the slab bookkeeping,
the weak-scaling meshes of the C5 study and max-over-ranks timing helpers.
"""
from __future__ import annotations

from typing import Tuple


def env_rank() -> Tuple[int, int, int]:
    import os
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def weak_box(n_gpus: int) -> Tuple[int, int, int]:
    """Base cells per axis of the C5 weak-scaling mesh for n_gpus GPUs, each
    rank holding one 128^3 block after 7 refinements (128^3 on
    1 GPU -> 256^3 on 8): 1 -> 1x1x1, 2 -> 1x1x2, 4 -> 1x2x2, 8 -> 2x2x2,
    otherwise 1x1xN (z-slabs of 128 layers)."""
    return {1: (1, 1, 1), 2: (1, 1, 2), 4: (1, 2, 2), 8: (2, 2, 2)}.get(n_gpus, (1, 1, n_gpus))


def slab_partition(n_cell_layers: int, world: int, rank: int, p: int) -> dict:
    """Cell layers [c0, c1) and owned lattice planes [g0, g1) of `rank` for a
    z-slab split of `n_cell_layers` layers of degree-p cells: layers are dealt
    as evenly as possible; every rank owns the planes of its layers except the
    top interface plane, which belongs to the next rank (the last rank also
    owns the top boundary plane)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("slab_partition: bad world/rank")
    if n_cell_layers < world:
        raise ValueError("slab_partition: fewer cell layers than ranks (agglomerate the level instead)")
    base, extra = divmod(n_cell_layers, world)
    c0 = rank * base + min(rank, extra)
    c1 = c0 + base + (1 if rank < extra else 0)
    g0 = c0 * p
    g1 = c1 * p + (1 if rank == world - 1 else 0)
    return {"cells": (c0, c1), "planes": (g0, g1), "halo_low": rank > 0, "halo_high": rank < world - 1}


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (device-timed step times); identity
    without an initialised process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_throughput(units_per_rank: float, ms_local: float, device=None) -> Tuple[float, float]:
    """Whole-job throughput for weak-scaled replicas: (sum of units over ranks)
    / (max over ranks of the step time). Returns (value per second, max ms)."""
    import torch.distributed as dist
    world = dist.get_world_size() if (dist.is_available() and dist.is_initialized()) else 1
    ms = max_over_ranks(ms_local, device)
    return world * units_per_rank / (ms * 1e-3), ms
