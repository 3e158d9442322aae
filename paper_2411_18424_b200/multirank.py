"""Multi-GPU plumbing for the swap path.

Tensor parallelism shards KV heads: rank r of a TP group owns heads
[r*H/TP, (r+1)*H/TP) of every layer, so its per-block bytes are 1/TP of the
model's.  Every rank runs the *identical* control plane (the engine is
deterministic) and executes the identical TransferOp list against its own KV
shard, over its own PCIe link, into its own pinned host pool — there is no
exchange step, hence no collective on the data path.  The only collectives
are control/measurement plumbing:

* `agree(digest)`     — all ranks dispatched the same plan stream (tiny
                        all_gather of a sha256; the multi-process analogue of
                        the reference's single decision stream);
* `max_over_ranks(t)` — job time = slowest rank (bench timing rule).
"""

from __future__ import annotations

import hashlib
import os
from typing import Optional

from .geometry import KVGeometry


def env() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(geometry: KVGeometry, tp: int) -> KVGeometry:
    """Per-rank geometry of a TP-sharded KV cache (block bytes / tp)."""
    return geometry.with_tp(tp)


class PlanDigest:
    """Running sha256 of every dispatched SwapPlan (ops + direction + request)."""

    def __init__(self) -> None:
        self._h = hashlib.sha256()
        self.plans = 0

    def add(self, iteration: int, plan) -> None:
        ops = ";".join(f"{o.blocks},{o.gpu_start},{o.cpu_start}" for o in plan.all_ops())
        self._h.update(f"{iteration}|{plan.request}|{plan.direction}|{ops}\n".encode())
        self.plans += 1

    def attach(self, manager) -> "PlanDigest":
        orig = manager.dispatch

        def dispatch(clock, iteration, plan, not_before=0):
            self.add(iteration, plan)
            return orig(clock, iteration, plan, not_before)

        manager.dispatch = dispatch
        return self

    def hexdigest(self) -> str:
        return self._h.hexdigest()


def agree(digest: str, group=None) -> bool:
    """True iff every rank reports the same digest (all_gather_object)."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return True
    out: list[Optional[str]] = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, digest, group=group)
    return all(d == digest for d in out)


def max_over_ranks(value: float, device=None, group=None) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(value: float, device=None, group=None) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())
