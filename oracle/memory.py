"""Oracle: compressed-memory accounting ("memory requirement of
compressed tensors (i.e., core tensors and factor matrices)").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Element counts from the
rank formulas of SURVEY.md §8(c) c11; bytes = element_bytes x count
(8 for complex64, the hot-path storage).  Saving = 100 (1 - c/o) (the
reported numbers of Tables I/III are 1 - ratio).
"""
from __future__ import annotations

import numpy as np


def original_elems(n, ndir) -> int:
    return int(np.prod(n)) * int(ndir)


def tucker3d_elems(n, ranks_per_dir) -> int:
    return int(sum(np.prod(r) + sum(ni * ri for ni, ri in zip(n, r)) for r in ranks_per_dir))


def tucker4d_elems(n, ndir, r) -> int:
    dims = tuple(n) + (ndir,)
    return int(np.prod(r) + sum(ni * ri for ni, ri in zip(dims, r)))


def htucker_elems(n, ndir, r) -> int:
    """r = (r1, r2, r3, r4, r12, r34)."""
    dims = tuple(n) + (ndir,)
    r1, r2, r3, r4, r12, r34 = r
    return int(sum(ni * ri for ni, ri in zip(dims, (r1, r2, r3, r4)))
               + r1 * r2 * r12 + r3 * r4 * r34 + r12 * r34)


def tt3d_elems(n, ranks_per_dir) -> int:
    n1, n2, n3 = n
    return int(sum(n1 * r1 + r1 * n2 * r2 + n3 * r2 for (r1, r2) in ranks_per_dir))


def tt4d_elems(n, ndir, r) -> int:
    n1, n2, n3 = n
    r1, r2, r3 = r
    return int(n1 * r1 + r1 * n2 * r2 + r2 * n3 * r3 + ndir * r3)


def saving_percent(compressed: int, original: int) -> float:
    return 100.0 * (1.0 - compressed / original)
