"""Worker-count API of the reference (parallel.py:1-69), kept for drop-in compatibility.

On the B200 the CUDA grid replaces the reference's thread-pool span split
(parallel.py:43-69).  The reference's determinism contract -- results
bitwise independent of the worker count -- becomes "bitwise independent of
launch geometry for a fixed ReductionConfig", which the kernels guarantee by
construction (the lattice shape, not the grid, fixes every rounding).  The
worker count is therefore recorded but changes nothing.
"""

from __future__ import annotations

import os

_num_workers = 1


def set_num_workers(n: int) -> None:
    """parallel.py:17-25 (validation identical; no effect on GPU results)."""
    global _num_workers
    if n < 1:
        raise ValueError(f"worker count must be >= 1, got {n}")
    _num_workers = n


def num_workers() -> int:
    return _num_workers


def max_workers() -> int:
    return os.cpu_count() or 1


def split_range(n: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous (lo, hi) spans covering range(n), at most `parts` of them,
    lengths differing by at most one, longer spans first (parallel.py:43-53).

    Used by the multi-GPU partitioner (dist.py) to cut vectors into rank chunks.
    """
    k = max(1, min(parts, n))
    base, longer = divmod(n, k)
    edge = [i * base + min(i, longer) for i in range(k + 1)]
    return list(zip(edge[:-1], edge[1:]))
