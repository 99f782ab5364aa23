"""Execution configuration (kbesolve/engine.py:28-63) on the device path.

The reference's engine is a CPU stand-in for the GPU hierarchy: k-shards,
a thread pool, block chunking and a deterministic tree reduce.  On B200 the
same roles are played natively:

* ``Schedule.n_shards``  <-> one process per GPU; k-shards of size n_k / world
  (validated exactly as engine.py:57-60);
* ``workers`` / ``WorkerPool``  -> accepted for API compatibility, ignored
  (one host thread per GPU; all device work is asynchronous on one stream);
* ``block_size`` / ``reduce_mode`` / ``fusion_enabled`` / ``index_mode``
  -> validated and advisory: CUDA blocks, warp reduce-scatter shuffles and
  on-the-fly index folding replace them, with a fixed reduction order so
  results are deterministic run to run.

``combine_shards`` / ``execute`` / ``plan`` are kept as host utilities for
callers of the reference API.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .errors import ConfigError
from .kgrid import KGrid

INDEX_MODES = ("on-the-fly", "lookup")
REDUCE_MODES = ("tree", "sequential")


@dataclass(frozen=True)
class Schedule:
    """Same fields, defaults and validation as engine.py:28-63."""

    n_shards: int = 1
    workers: int = 1
    block_size: int = 128
    batch_enabled: bool = True
    fusion_enabled: bool = True
    index_mode: str = "on-the-fly"
    reduce_mode: str = "tree"

    def validate(self, n_k: int | None = None) -> None:
        if self.n_shards < 1:
            raise ConfigError(f"n_shards must be >= 1, got {self.n_shards}")
        if self.workers < 1:
            raise ConfigError(f"workers must be >= 1, got {self.workers}")
        if self.block_size < 1:
            raise ConfigError(f"block_size must be >= 1, got {self.block_size}")
        if self.index_mode not in INDEX_MODES:
            raise ConfigError(f"index_mode must be one of {INDEX_MODES}, got {self.index_mode!r}")
        if self.reduce_mode not in REDUCE_MODES:
            raise ConfigError(f"reduce_mode must be one of {REDUCE_MODES}, got {self.reduce_mode!r}")
        if n_k is not None and n_k % self.n_shards != 0:
            raise ConfigError(f"n_shards: {self.n_shards} does not divide n_k={n_k}")

    def with_workers(self, workers: int) -> "Schedule":
        return replace(self, workers=workers)


@dataclass(frozen=True)
class WorkPlan:
    shard_ranges: tuple
    pair_count: int
    inner_size: int
    chunk_count: int


def plan(grid: KGrid, n_t: int, schedule: Schedule) -> WorkPlan:
    """Partition of one frontier evaluation (engine.py:80-97)."""
    schedule.validate(grid.n_k)
    my_nk = grid.n_k // schedule.n_shards
    ranges = tuple((s * my_nk, (s + 1) * my_nk) for s in range(schedule.n_shards))
    inner = grid.n_k * grid.n_k
    chunks = -(-inner // schedule.block_size) if schedule.fusion_enabled else grid.n_k
    return WorkPlan(ranges, 2 * n_t + 1, inner, chunks)


class WorkerPool:
    """Accepted for API compatibility (engine.py:100-124); device work is not threaded."""

    def __init__(self, workers: int = 1):
        if workers < 1:
            raise ConfigError(f"workers must be >= 1, got {workers}")
        self.workers = workers

    def map(self, fn, items):
        return [fn(item) for item in items]

    def close(self) -> None:
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def execute(kernel, items, pool: WorkerPool | None = None) -> list:
    """Evaluate a pure callable over items in order (engine.py:127-138)."""
    return [kernel(item) for item in items]


def combine_shards(pieces, axis: int = 0) -> np.ndarray:
    """Concatenate per-shard outputs by global k offset (engine.py:210-224)."""
    ordered = sorted(pieces, key=lambda p: p[0])
    expect = ordered[0][0]
    for off, arr in ordered:
        if off != expect:
            raise ValueError(f"shard pieces not contiguous at k-offset {off}")
        expect = off + arr.shape[axis]
    if len(ordered) == 1:
        return ordered[0][1]
    return np.concatenate([arr for _, arr in ordered], axis=axis)


def shard_range(n_k: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous k-range owned by one GPU (the reference's shard s = rank)."""
    if world < 1 or n_k % world != 0:
        raise ConfigError(f"n_shards: {world} does not divide n_k={n_k}")
    my = n_k // world
    return rank * my, (rank + 1) * my
