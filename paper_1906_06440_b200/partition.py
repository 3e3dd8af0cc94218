"""Deterministic work splitting — drop-in for ``brkernels.partition``.

The reference distributes blocked work items over a CPU thread pool
(``partition.py:8-50``).  On the GPU the same item order (minibatch block
innermost, so consecutive items share a weight slice) is the tile order of
the persistent CTA scheduler; these helpers remain for API compatibility and
for host-side sharding across ranks (``dist.py``).
"""

from __future__ import annotations


def split_evenly(n_items: int, workers: int) -> list[range]:
    """Contiguous ranges covering [0, n_items), sizes differing by at most one."""
    if n_items < 0:
        raise ValueError(f"n_items must be >= 0, got {n_items}")
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    q, r = divmod(n_items, workers)
    bounds = [0]
    for w in range(workers):
        bounds.append(bounds[-1] + q + (w < r))
    return [range(bounds[w], bounds[w + 1]) for w in range(workers)]


def partition_work_2d(k_blocks: int, n_blocks: int, workers: int) -> list[range]:
    """Split the flat (ib_k * n_blocks + ib_n) item grid block-contiguously."""
    if k_blocks < 1 or n_blocks < 1:
        raise ValueError(f"grid extents must be >= 1, got ({k_blocks}, {n_blocks})")
    return split_evenly(k_blocks * n_blocks, workers)
