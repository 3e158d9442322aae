"""Run configuration, per-request state and the metrics the swap path is
judged by (the data types of kvswitch/engine.py:34-203, regrouped).

`MetricsReport` keeps the reference's 33 field names so `to_json()` /
`to_csv()` (both key-sorted) are byte-identical with the reference's reports
for the same run — tests/test_golden.py relies on that.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import Optional

from .alloc import PoolConfig
from .core import BlockSpec, RequestId, SimTime
from .costmodel import InferParams, TransferParams
from .scheduler import PriorityTrace, SchedulerConfig
from .workload import Conversation

# --------------------------------------------------------------------- ablations

# name -> (group_alloc, reuse, adaptive): each step adds one FastSwitch feature
_ABLATIONS = {
    "baseline": (False, False, False),
    "blockgroup": (True, False, False),
    "blockgroup_reuse": (True, True, False),
    "full": (True, True, True),
}
ABLATION_MODES = tuple(_ABLATIONS)


@dataclass(frozen=True)
class AblationMode:
    name: str
    group_alloc: bool  # block-group transfers (else one op per block)
    reuse: bool  # CPU-copy reuse across turns
    adaptive: bool  # adaptive sync/async swap-in (else always sync)


def ablation_modes() -> dict[str, AblationMode]:
    return {name: AblationMode(name, *flags) for name, flags in _ABLATIONS.items()}


# ------------------------------------------------------------------ percentiles

def _rank_index(n: int, q: float) -> int:
    """0-based nearest-rank index ceil(q*n)-1, robust to q*n landing a hair
    above an integer."""
    return max(1, math.ceil(q * n - 1e-9)) - 1


def percentile(samples: list, q: float):
    """Nearest-rank percentile (engine.py:77-89)."""
    if not samples:
        raise ValueError("percentile of empty sample set")
    if q <= 0.0 or q > 1.0:
        raise ValueError(f"q must be in (0, 1], got {q}")
    return sorted(samples)[_rank_index(len(samples), q)]


def tail_percentile(samples: list, q: float):
    """Nearest-rank counted from the largest sample down (engine.py:92-101):
    tail_percentile(efficiencies, 0.99) is the worst-1% efficiency."""
    if not samples:
        raise ValueError("tail percentile of empty sample set")
    return sorted(samples, reverse=True)[_rank_index(len(samples), q)]


# ------------------------------------------------------------------ configuration

def _gpu_pool_default() -> PoolConfig:
    return PoolConfig(total_blocks=512)


@dataclass(frozen=True)
class EngineConfig:
    block: BlockSpec = field(default_factory=BlockSpec)
    gpu_pool: PoolConfig = field(default_factory=_gpu_pool_default)
    cpu_pool_blocks: int = 491520  # 60 GiB at the reference's 128 KiB block
    transfer: TransferParams = field(default_factory=TransferParams)
    inference: InferParams = field(default_factory=InferParams)
    scheduler: SchedulerConfig = field(default_factory=SchedulerConfig)
    trace: PriorityTrace = field(default_factory=PriorityTrace)
    ablation: str = "full"
    sync_threshold_ratio: float = 0.5
    short_request_blocks: int = 16
    prealloc_min_blocks: int = 8
    prealloc_max_blocks: int = 256
    release_copy_on_swap_in: bool = False

    def __post_init__(self) -> None:
        problems = [
            (self.ablation not in _ABLATIONS, f"ablation must be one of {ABLATION_MODES}"),
            (self.cpu_pool_blocks < 1, "cpu_pool_blocks must be >= 1"),
            (not self.sync_threshold_ratio > 0, "sync_threshold_ratio must be positive"),
        ]
        for bad, msg in problems:
            if bad:
                raise ValueError(msg)

    @property
    def mode(self) -> AblationMode:
        return ablation_modes()[self.ablation]


# ------------------------------------------------------------------ per request

@dataclass
class RequestState:
    conv: Conversation
    phase: str = "pending"
    turn_idx: int = 0
    context_tokens: int = 0  # tokens whose KV exists
    pending_input: int = 0  # this turn's prompt, not yet prefilled
    remaining_output: int = 0
    turn_arrival: SimTime = 0
    turn_start_blocks: int = 0
    prev_token_at: Optional[SimTime] = None
    recompute_tokens: int = 0  # KV dropped or contaminated, owed as prefill
    last_out_done: SimTime = 0  # completion of this request's latest swap-out

    @property
    def req(self) -> RequestId:
        return self.conv.id


# ------------------------------------------------------------------ metrics

@dataclass
class IterationRecord:
    index: int
    start: SimTime
    end: SimTime
    prefill_tokens: int
    decode_tokens: int
    stall_sync: SimTime
    stall_conflict: SimTime
    stall_yield: SimTime
    stall_recompute: SimTime
    tokens_emitted: int

    @property
    def stall_total(self) -> SimTime:
        return self.stall_sync + self.stall_conflict + self.stall_yield + self.stall_recompute


@dataclass
class MetricsReport:
    # latency (us)
    ttft_p95_us: int
    ttft_p99_us: int
    ttft_p999_us: int
    tbt_p999_us: int
    # throughput / efficiency
    throughput_tokens_per_s: float
    efficiency_p50: float
    efficiency_p90: float
    efficiency_p99: float
    efficiency_p999: float
    # where the time went (us)
    overhead_ratio: float
    stall_sync_us: int
    stall_conflict_us: int
    stall_yield_us: int
    stall_recompute_us: int
    stall_total_us: int
    busy_time_us: int
    # swap traffic
    avg_granularity_blocks: float
    swap_out_blocks: int
    swap_out_ops: int
    swap_in_blocks: int
    swap_in_ops: int
    reused_blocks: int
    peak_cpu_blocks: int
    # run bookkeeping
    total_tokens: int
    expected_tokens: int
    iterations: int
    sim_end_us: int
    conversations: int
    turns_completed: int
    conflicts: int
    sync_stalls: int
    epochs: int
    granularity_histogram: dict = field(default_factory=dict)

    def to_dict(self) -> dict:
        out = dict(vars(self))
        out["granularity_histogram"] = {
            str(size): n for size, n in sorted(self.granularity_histogram.items())}
        return out

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), sort_keys=True, indent=2)

    def to_csv(self) -> str:
        rows = [f"{k},{v}" for k, v in sorted(self.to_dict().items())
                if k != "granularity_histogram"]
        return "\n".join(["metric,value", *rows]) + "\n"


def build_report(eng, stalls: dict[str, int], effs: list[float],
                 first_arrival: SimTime) -> MetricsReport:
    """Summarise a finished engine run (engine.py:828-876)."""
    busy = sum(r.end - r.start for r in eng.records)
    stall_total = sum(stalls.values())
    gran = eng.pool.granularity_stats()
    avg_gran, hist = gran if gran is not None else (0.0, {})

    def pct(xs, q):
        return percentile(xs, q) if xs else 0

    mgr = eng.manager
    return MetricsReport(
        ttft_p95_us=pct(eng.ttft_samples, 0.95),
        ttft_p99_us=pct(eng.ttft_samples, 0.99),
        ttft_p999_us=pct(eng.ttft_samples, 0.999),
        tbt_p999_us=pct(eng.tbt_samples, 0.999),
        throughput_tokens_per_s=eng.total_tokens * 1_000_000 / max(1, eng.clock - first_arrival),
        efficiency_p50=tail_percentile(effs, 0.50),
        efficiency_p90=tail_percentile(effs, 0.90),
        efficiency_p99=tail_percentile(effs, 0.99),
        efficiency_p999=tail_percentile(effs, 0.999),
        overhead_ratio=stall_total / busy if busy else 0.0,
        stall_sync_us=stalls["sync"],
        stall_conflict_us=stalls["conflict"],
        stall_yield_us=stalls["yield"],
        stall_recompute_us=stalls["recompute"],
        stall_total_us=stall_total,
        busy_time_us=busy,
        avg_granularity_blocks=avg_gran,
        swap_out_blocks=mgr.total_blocks["out"],
        swap_out_ops=mgr.total_ops["out"],
        swap_in_blocks=mgr.total_blocks["in"],
        swap_in_ops=mgr.total_ops["in"],
        reused_blocks=eng.reused_blocks,
        peak_cpu_blocks=eng.store.peak_used_blocks,
        total_tokens=eng.total_tokens,
        expected_tokens=sum(b for conv in eng.conversations for _, b in conv.turns),
        iterations=eng.iteration,
        sim_end_us=eng.clock,
        conversations=len(eng.conversations),
        turns_completed=eng.turns_completed,
        conflicts=eng.conflict_count,
        sync_stalls=eng.sync_stall_count,
        epochs=eng.epoch,
        granularity_histogram=hist,
    )
