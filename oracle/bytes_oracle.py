"""ORACLE — test infrastructure only.  CPU restatement of the swap path's bytes.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module, and only as the checker (or the timed
CPU baseline) — never as the product path.

Parity status: the reference (kvswitch) moves no bytes (SPEC.md:8,
SPEC.md:74 "a block is an opaque fixed-size byte extent"), so byte parity is
anchored on the reference's TransferOp semantics and pinned by the golden
fixtures in tests/golden/ (plans recorded from the reference itself):

* TransferOp(blocks, gpu_start, cpu_start) copies `blocks` consecutive GPU
  blocks starting at gpu_start to/from `blocks` consecutive host blocks
  starting at cpu_start (cpu_store.py:73-79, built by _pair_extents
  cpu_store.py:95-120 from the GPU block table engine.py:317-325 and the
  copy's host extents cpu_store.py:169-191).
* The baseline ablation splits each op into single-block ops
  (swap.py:170-179); `split_single` restates it and must move identical bytes.
* A block spans every KV plane (all layers of the rank); the host image is
  block-major [cpu_block][plane][chunk].
"""

from __future__ import annotations

from typing import Iterable, Sequence

import numpy as np


def as_ops(ops) -> np.ndarray:
    if isinstance(ops, np.ndarray):
        return np.ascontiguousarray(ops, dtype=np.int64).reshape(-1, 3)
    rows = []
    for op in ops:
        if hasattr(op, "blocks"):
            rows.append((op.blocks, op.gpu_start, op.cpu_start))
        else:
            rows.append(tuple(op))
    return np.asarray(rows, dtype=np.int64).reshape(-1, 3)


def split_single(ops) -> np.ndarray:
    """swap.py:170-179: one op per block, same (gpu, cpu) pairing."""
    out = []
    for b, g, c in as_ops(ops):
        for i in range(int(b)):
            out.append((1, g + i, c + i))
    return np.asarray(out, dtype=np.int64).reshape(-1, 3)


def block_pairs(ops) -> np.ndarray:
    """[(gpu_block, cpu_block)] in plan order — the op list's bijection."""
    pairs = []
    for b, g, c in as_ops(ops):
        idx = np.arange(int(b), dtype=np.int64)
        pairs.append(np.stack([g + idx, c + idx], axis=1))
    if not pairs:
        return np.zeros((0, 2), dtype=np.int64)
    return np.concatenate(pairs)


def apply_plan(direction: str, planes: np.ndarray, host: np.ndarray, ops) -> None:
    """Apply one SwapPlan in place.

    planes: uint8 [P, num_gpu_blocks, chunk]   (GPU KV planes)
    host:   uint8 [num_cpu_blocks, P * chunk]  (block-major host pool)
    """
    P, G, chunk = planes.shape
    if host.shape[1] != P * chunk:
        raise ValueError("host block size != planes * chunk")
    for b, g, c in as_ops(ops):
        b, g, c = int(b), int(g), int(c)
        if b < 1 or g < 0 or c < 0 or g + b > G or c + b > host.shape[0]:
            raise IndexError(f"op ({b}, {g}, {c}) outside the pools")
        if direction == "out":
            host[c:c + b].reshape(b, P, chunk)[:] = planes[:, g:g + b, :].transpose(1, 0, 2)
        elif direction == "in":
            planes[:, g:g + b, :] = host[c:c + b].reshape(b, P, chunk).transpose(1, 0, 2)
        else:
            raise ValueError(f"direction must be 'out' or 'in', got {direction!r}")


def _fmix32(x: np.ndarray) -> np.ndarray:
    x = x ^ (x >> np.uint32(16))
    x = x * np.uint32(0x85EBCA6B)
    x = x ^ (x >> np.uint32(13))
    x = x * np.uint32(0xC2B2AE35)
    return x ^ (x >> np.uint32(16))


def kv_pattern(seed: int, num_planes: int, num_blocks: int, chunk: int) -> np.ndarray:
    """Counter-hash KV bytes: word (plane, block, i) = fmix32(seed, plane, block, i).

    Any misplaced or stale 4-byte word is detectable.
    """
    if chunk % 4:
        raise ValueError("chunk must be a multiple of 4")
    words = chunk // 4
    with np.errstate(over="ignore"):
        p = np.arange(num_planes, dtype=np.uint32)[:, None, None]
        b = np.arange(num_blocks, dtype=np.uint32)[None, :, None]
        i = np.arange(words, dtype=np.uint32)[None, None, :]
        key = (np.uint32(seed & 0xFFFFFFFF) * np.uint32(0x9E3779B1)) ^ (
            p * np.uint32(0x27D4EB2F)) ^ (b * np.uint32(0x165667B1)) ^ i
        vals = _fmix32(key.astype(np.uint32))
    return np.ascontiguousarray(vals).view(np.uint8).reshape(num_planes, num_blocks, chunk)


def random_runs(rng: np.random.Generator, total_blocks: int, group: int, gpu_pool: int,
                cpu_pool: int) -> np.ndarray:
    """Config-2 synthetic plan: `total_blocks` split into runs of `group`
    blocks at random non-overlapping positions on both sides."""
    n_runs = -(-total_blocks // group)
    sizes = [group] * n_runs
    sizes[-1] = total_blocks - group * (n_runs - 1)

    def place(pool: int) -> list[int]:
        slots = pool // group
        if slots < n_runs:
            raise ValueError(f"pool of {pool} blocks cannot hold {n_runs} runs of {group}")
        chosen = np.sort(rng.choice(slots, size=n_runs, replace=False))
        return [int(s) * group for s in chosen]

    gpu = place(gpu_pool)
    cpu = place(cpu_pool)
    order = rng.permutation(n_runs)  # logical order != address order
    return np.asarray([(sizes[i], gpu[j], cpu[k]) for i, (j, k) in
                       enumerate(zip(order, rng.permutation(n_runs)))], dtype=np.int64)


def random_block_table(rng: np.random.Generator, blocks: int, pool: int,
                       used: np.ndarray | None = None) -> np.ndarray:
    """Config-1 fragmented table: `blocks` distinct random pool blocks."""
    free = np.ones(pool, dtype=bool)
    if used is not None:
        free[used] = False
    cand = np.flatnonzero(free)
    return rng.choice(cand, size=blocks, replace=False).astype(np.int64)


def table_to_ops(gpu_table: Sequence[int], cpu_table: Sequence[int]) -> np.ndarray:
    """Zip two per-logical-block tables into maximal TransferOps (the
    _pair_extents rule: break wherever either side loses contiguity)."""
    ops = []
    for g, c in zip(gpu_table, cpu_table):
        g, c = int(g), int(c)
        if ops and ops[-1][1] + ops[-1][0] == g and ops[-1][2] + ops[-1][0] == c:
            ops[-1][0] += 1
        else:
            ops.append([1, g, c])
    return np.asarray(ops, dtype=np.int64).reshape(-1, 3)
