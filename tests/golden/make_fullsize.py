"""Generates the full-size vmult fingerprints of the reference
(tests/golden/fullsize_<cfg>.npz): the reference's own
SpaceTimeOperator::apply (space_time_operator.cpp:45-130, compiled unmodified
into oracle/_ref by oracle/Makefile) on the seeded input
problems.uniform_vector(N, seed=42) at the FULL BASELINE sizes C2 (64^3),
C3 (128^3), C4 (96^3) and C5-128.

A 4.3 GB output cannot be committed, so the fixture holds size-independent
fingerprints of y = S u that the GPU test recomputes from its own output:
  * block_dot[b] = sum_{i in block b} y_i s_i over 4096 contiguous blocks,
    s = seeded random signs (first-order sensitive to any local error),
  * block_norm[b] = ||y_block||_2,
  * 20000 seeded sample entries (index, value),
  * ||y||_2 and n_dofs.
Run (CPU, needs /root/reference; ~40 GB RAM and ~15 min for C5-128):
  python tests/golden/make_fullsize.py [C2 C3 C4 C5-128]
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import refbind  # noqa: E402
from paper_2408_04372_b200 import problems  # noqa: E402

BLOCKS = 4096
SAMPLES = 20000


def signs(n):
    return (np.random.default_rng(99).integers(0, 2, n, dtype=np.int8) * 2 - 1).astype(np.int8)


def bounds(n):
    return (n * np.arange(BLOCKS + 1, dtype=np.int64)) // BLOCKS


def fingerprint(y):
    n = y.size
    s = signs(n)
    b = bounds(n)
    dots = np.add.reduceat(y * s, b[:-1])
    norms = np.sqrt(np.add.reduceat(y * y, b[:-1]))
    idx = np.unique(np.random.default_rng(7).integers(0, n, SAMPLES))
    return {"n_dofs": np.int64(n), "norm": np.float64(np.linalg.norm(y)), "block_dot": dots, "block_norm": norms,
            "sample_idx": idx, "sample_val": y[idx]}


def main(names):
    for name in names:
        cfg = problems.config(name)
        t0 = time.time()
        R = refbind.Reference(cfg)
        t1 = time.time()
        u = problems.uniform_vector(R.n_dofs, seed=42)
        y = R.apply(u)
        t2 = time.time()
        del u, R
        np.savez_compressed(os.path.join(HERE, f"fullsize_{name}.npz"), **fingerprint(y))
        print(f"{name}: N={y.size} setup {t1 - t0:.0f}s apply {t2 - t1:.0f}s", flush=True)
        del y


if __name__ == "__main__":
    main(sys.argv[1:] or ["C2", "C3", "C4", "C5-128"])
