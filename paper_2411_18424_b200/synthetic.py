"""Synthetic swap plans for measurement: seeded
block tables and run layouts.  Inputs only — `bench.py` and `tools/` build
their plans here so that nothing on a measured path imports `oracle/`
(which restates the path to check it)."""

from __future__ import annotations

from typing import Optional, Sequence

import numpy as np


def random_runs(rng: np.random.Generator, total_blocks: int, group: int, gpu_pool: int,
                cpu_pool: int) -> np.ndarray:
    """Config 2: `total_blocks` in runs of `group` blocks at random,
    non-overlapping positions on both sides, in a random logical order;
    int64 [n, 3] = (blocks, gpu_start, cpu_start)."""
    n_runs = -(-total_blocks // group)
    sizes = [group] * n_runs
    sizes[-1] = total_blocks - group * (n_runs - 1)

    def starts(pool: int) -> list[int]:
        slots = pool // group
        if slots < n_runs:
            raise ValueError(f"pool of {pool} blocks cannot hold {n_runs} runs of {group}")
        return [int(x) * group for x in np.sort(rng.choice(slots, size=n_runs, replace=False))]

    gpu, cpu = starts(gpu_pool), starts(cpu_pool)
    order, host_order = rng.permutation(n_runs), rng.permutation(n_runs)
    return np.asarray([(sizes[i], gpu[j], cpu[k]) for i, (j, k) in
                       enumerate(zip(order, host_order))], dtype=np.int64)


def random_block_table(rng: np.random.Generator, blocks: int, pool: int,
                       used: Optional[np.ndarray] = None) -> np.ndarray:
    """Config 1: `blocks` distinct random blocks of a pool (fragmented table)."""
    free = np.ones(pool, dtype=bool)
    if used is not None:
        free[used] = False
    return rng.choice(np.flatnonzero(free), size=blocks, replace=False).astype(np.int64)


def pair_tables(gpu_table: Sequence[int], cpu_table: Sequence[int]) -> np.ndarray:
    """Two per-logical-block tables -> maximal (blocks, gpu_start, cpu_start)
    runs, split wherever either side stops being contiguous."""
    g = np.asarray(gpu_table, dtype=np.int64)
    c = np.asarray(cpu_table, dtype=np.int64)
    if len(g) == 0:
        return np.zeros((0, 3), dtype=np.int64)
    brk = np.flatnonzero((np.diff(g) != 1) | (np.diff(c) != 1)) + 1
    starts = np.concatenate([[0], brk])
    ends = np.concatenate([brk, [len(g)]])
    return np.stack([ends - starts, g[starts], c[starts]], axis=1)
