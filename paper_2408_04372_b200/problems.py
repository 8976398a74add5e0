"""Workload definitions of BASELINE.json's configs (C1..C5) with seeded
synthetic inputs, shared by tests and bench.py. Each config fixes the mesh
hierarchy, discretisation, coefficient and the generators of its inputs.

Choices BASELINE leaves open (documented in DESIGN.md):
  * tau: C1 uses the stated slab [0, 0.5] (tau = 0.5); C2-C5 use tau = h
    (one cell width), i.e. the reference's convention of refining h and tau
    together.
  * C2 perturbation: interior vertices displaced i.i.d. uniform in
    [-0.2h, 0.2h] per coordinate from numpy PCG64(seed), drawn for all
    vertices in lexicographic order (x fastest), boundary vertices fixed.
  * C3: rho in {1, 1e4} on the 8^3 checkerboard of level-0 cells
    (1e4 where cx+cy+cz is odd).
  * C4: rho = c^2 with c in {1, 2, 4} for the three z-layers of the 3^3 base
    mesh; Gaussian pulse of width 0.05 at the centre of [0,1]^3.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

HEAT, WAVE = 0, 1
DG, CGP = 0, 1


def uniform_vector(n: int, seed: int = 42, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Seeded U[lo,hi] test vector (fast numpy PCG64 stream; parity tests feed
    the same array to the oracle and the GPU)."""
    return np.random.default_rng(seed).uniform(lo, hi, n)


def cartesian_vertices(dim: int, cells: int, lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0)) -> np.ndarray:
    n = cells + 1
    ax = [lo[a] + (hi[a] - lo[a]) * np.arange(n, dtype=np.float64) / cells for a in range(dim)]
    while len(ax) < 3:
        ax.append(np.zeros(1))
    z, y, x = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    return np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1)


def perturbed_vertices(dim: int, cells: int, magnitude: float = 0.2, seed: int = 42,
                       lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0)) -> np.ndarray:
    """Finest-level vertices with interior vertices displaced i.i.d. uniform in
    [-magnitude*h, magnitude*h] per coordinate (BASELINE C2)."""
    v = cartesian_vertices(dim, cells, lo, hi)
    n = cells + 1
    rng = np.random.Generator(np.random.PCG64(seed))
    h = np.array([(hi[a] - lo[a]) / cells for a in range(3)])
    d = rng.uniform(-1.0, 1.0, size=v.shape) * magnitude * h
    vi = np.arange(v.shape[0])
    idx = np.stack([vi % n, (vi // n) % n, vi // (n * n)], axis=1)
    interior = np.ones(v.shape[0], dtype=bool)
    for a in range(dim):
        interior &= (idx[:, a] > 0) & (idx[:, a] < n - 1)
    d[~interior] = 0.0
    d[:, dim:] = 0.0
    return v + d


@dataclasses.dataclass
class Config:
    name: str
    equation: int
    scheme: int
    dim: int
    base_cells: int
    refinements: int
    p: int
    k: int
    n_steps: int
    tau: float
    perturb: float = 0.0
    rho: Optional[np.ndarray] = None  # per level-0 cell
    seed: int = 42

    @property
    def cells(self) -> int:
        return self.base_cells << self.refinements

    @property
    def n_t(self) -> int:
        return self.k + 1 if self.scheme == DG else self.k

    @property
    def n_space(self) -> int:
        return (self.cells * self.p + 1) ** self.dim

    @property
    def n_dofs(self) -> int:
        return self.n_steps * self.n_t * self.n_space

    def vertices(self) -> Optional[np.ndarray]:
        if self.perturb <= 0.0:
            return None
        return perturbed_vertices(self.dim, self.cells, self.perturb, self.seed)

    def describe(self) -> dict:
        return {"equation": ["heat", "wave"][self.equation], "scheme": ["dg", "cgp"][self.scheme], "dim": self.dim,
                "cells": self.cells, "p": self.p, "k": self.k, "n_steps": self.n_steps, "tau": self.tau,
                "perturb": self.perturb, "rho": None if self.rho is None else "per-level-0-cell",
                "n_dofs": self.n_dofs}


def checkerboard(base: int, lo_val: float = 1.0, hi_val: float = 1e4) -> np.ndarray:
    c = np.arange(base)
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    return np.where((x + y + z) % 2 == 1, hi_val, lo_val).astype(np.float64).ravel()


def layered(base: int = 3, speeds=(1.0, 2.0, 4.0)) -> np.ndarray:
    c = np.arange(base)
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    s = np.asarray(speeds)[np.minimum(z * len(speeds) // base, len(speeds) - 1)]
    return (s * s).astype(np.float64).ravel()


def config(name: str, refinements: Optional[int] = None) -> Config:
    """C1..C5 at full size, or with fewer refinements (same base mesh) for
    oracle-reachable parity runs."""
    if name == "C1":
        r = 4 if refinements is None else refinements
        return Config("C1", HEAT, DG, 2, 1, r, 2, 1, 1, 0.5)
    if name == "C2":
        r = 6 if refinements is None else refinements
        return Config("C2", HEAT, DG, 3, 1, r, 3, 2, 1, 1.0 / (1 << r), perturb=0.2)
    if name == "C3":
        r = 4 if refinements is None else refinements
        return Config("C3", HEAT, CGP, 3, 8, r, 2, 2, 2, 1.0 / (8 << r), rho=checkerboard(8))
    if name == "C4":
        r = 5 if refinements is None else refinements
        return Config("C4", WAVE, CGP, 3, 3, r, 4, 2, 4, 1.0 / (3 << r), rho=layered(3))
    if name.startswith("C5"):
        # C5-32 / C5-64 / C5-128 / C5-256 (cells per axis)
        cells = int(name.split("-")[1]) if "-" in name else 128
        r = int(np.log2(cells)) if refinements is None else refinements
        return Config(name, HEAT, DG, 3, 1, r, 4, 3, 1, 1.0 / (1 << r))
    raise KeyError(name)
