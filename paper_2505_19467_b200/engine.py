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


# ---- fixed-order reducers (engine.py:141-207) ------------------------------------------
# Host utilities for callers of the reference API.  On the device these orders are
# realised by the kernels themselves (warp reduce-scatter, fixed chunk order in K3);
# nothing on the step path calls these functions.

def chunk_partial_sums(terms, block_size: int, axis: int = -1) -> np.ndarray:
    """Sums over consecutive blocks of ``block_size`` along ``axis`` (engine.py:141-166).

    ceil(m / block_size) chunks, the last one possibly short; each chunk is summed by
    numpy along the innermost memory axis, so the in-chunk order depends only on the
    block size."""
    if block_size < 1:
        raise ConfigError(f"block_size must be >= 1, got {block_size}")
    x = np.ascontiguousarray(np.moveaxis(np.asarray(terms), axis, -1))
    m = x.shape[-1]
    lead = x.shape[:-1]
    if m == 0:
        return np.moveaxis(np.zeros(lead + (0,), dtype=x.dtype), -1, axis)
    n_full, rest = divmod(m, block_size)
    pieces = []
    if n_full:
        pieces.append(x[..., : n_full * block_size].reshape(lead + (n_full, block_size)).sum(axis=-1))
    if rest:
        pieces.append(x[..., n_full * block_size:].sum(axis=-1)[..., None])
    sums = np.concatenate(pieces, axis=-1) if len(pieces) > 1 else pieces[0]
    return np.moveaxis(sums, -1, axis)


def tree_reduce(parts, axis: int = -1, return_rounds: bool = False):
    """Offset-doubling pairwise reduction (engine.py:169-191): round r adds element
    i + 2^r into i for i a multiple of 2^(r+1); ceil(log2 m) rounds."""
    x = np.moveaxis(np.asarray(parts), axis, -1).copy()
    m = x.shape[-1]
    if m == 0:
        raise ValueError("cannot reduce zero partial sums")
    stride, rounds = 1, 0
    while stride < m:
        src = x[..., stride::2 * stride]
        x[..., 0: src.shape[-1] * 2 * stride: 2 * stride] += src
        stride <<= 1
        rounds += 1
    total = x[..., 0]
    return (total, rounds) if return_rounds else total


def sequential_reduce(parts, axis: int = -1) -> np.ndarray:
    """Left-to-right sum of the partials (engine.py:194-202)."""
    x = np.moveaxis(np.asarray(parts), axis, -1)
    if x.shape[-1] == 0:
        raise ValueError("cannot reduce zero partial sums")
    acc = np.array(x[..., 0], copy=True)
    for i in range(1, x.shape[-1]):
        acc += x[..., i]
    return acc


def reduce_partials(parts, schedule: Schedule | None, axis: int = -1) -> np.ndarray:
    """tree_reduce unless the schedule asks for sequential (engine.py:205-207)."""
    if schedule is not None and schedule.reduce_mode == "sequential":
        return sequential_reduce(parts, axis=axis)
    return tree_reduce(parts, axis=axis)
