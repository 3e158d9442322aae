"""JSON run documents -> EngineConfig / WorkloadConfig (mirror of the subset
of kvswitch/config.py the swap path's callers need: config.py:35-144 schema
and defaults, config.py:220-319 seed fan-out).  One top-level seed feeds the
allocator RNG, the priority trace and the workload generator.
"""

from __future__ import annotations

import copy
from typing import Any

from .alloc import PoolConfig
from .core import BlockSpec
from .costmodel import InferParams, TransferParams
from .engine import ABLATION_MODES, EngineConfig
from .scheduler import PriorityTrace, SchedulerConfig
from .workload import LengthDist, WorkloadConfig


class ConfigError(ValueError):
    def __init__(self, key: str, message: str) -> None:
        self.key = key
        super().__init__(f"config key '{key}': {message}")


def default_config() -> dict:
    return {
        "seed": 42,
        "ablation": "full",
        "block": {"block_size_tokens": 16, "bytes_per_block": 131072},
        "gpu_pool": {"total_blocks": 512, "initial_group_blocks": 60, "victim_policy": "random"},
        "cpu_pool": {"total_blocks": 491520},
        "transfer": {"dispatch_per_op_us": 12, "bandwidth_bytes_per_us": 32000,
                     "per_op_latency_floor_us": 2, "sync_batch": 8},
        "inference": {"decode_base_us": 2000, "decode_per_token_us": 25,
                      "prefill_per_token_us": 50},
        "scheduler": {"max_running": None, "preemption_mode": "swap",
                      "max_prefill_tokens": None},
        "workload": {"num_conversations": 200, "arrival_rate_per_s": 1.0, "mean_turns": 5.5,
                     "input_tokens": {"median": 96.0, "sigma": 0.9, "max": 1024},
                     "output_tokens": {"median": 112.0, "sigma": 0.7, "max": 512},
                     "think_time_mean_s": 10.0, "max_context_tokens": 3072,
                     "trace_path": None},
        "trace": {"pattern": "markov", "frequency": 0.02, "p_keep": 0.8,
                  "vtc_wp": 1, "vtc_wq": 2},
        "swap_policy": {"sync_threshold_ratio": 0.5, "short_request_blocks": 16},
        "reuse": {"prealloc_min_blocks": 8, "prealloc_max_blocks": 256,
                  "release_copy_on_swap_in": False},
        "output": {"report_json": None, "report_csv": None, "iteration_log": None},
    }


def _merge(base: dict, over: dict, prefix: str = "") -> dict:
    out = copy.deepcopy(base)
    for k, v in over.items():
        path = f"{prefix}.{k}" if prefix else k
        if k not in out:
            raise ConfigError(path, "unknown key")
        if isinstance(out[k], dict):
            if not isinstance(v, dict):
                raise ConfigError(path, f"expected an object, got {type(v).__name__}")
            out[k] = _merge(out[k], v, path)
        else:
            out[k] = v
    return out


def build(doc: dict) -> tuple[EngineConfig, WorkloadConfig, dict]:
    """Validate `doc` over the defaults; return (engine, workload, full document)."""
    full = _merge(default_config(), doc or {})
    seed = full["seed"]
    t, w, inf = full["transfer"], full["workload"], full["inference"]
    if full["ablation"] not in ABLATION_MODES:
        raise ConfigError("ablation", f"must be one of {ABLATION_MODES}")
    try:
        engine = EngineConfig(
            block=BlockSpec(**full["block"]),
            gpu_pool=PoolConfig(rng_seed=seed, **full["gpu_pool"]),
            cpu_pool_blocks=full["cpu_pool"]["total_blocks"],
            transfer=TransferParams(dispatch_per_op=t["dispatch_per_op_us"],
                                    bandwidth=t["bandwidth_bytes_per_us"],
                                    per_op_latency_floor=t["per_op_latency_floor_us"],
                                    sync_batch=t["sync_batch"]),
            inference=InferParams(decode_base=inf["decode_base_us"],
                                  decode_per_token=inf["decode_per_token_us"],
                                  prefill_per_token=inf["prefill_per_token_us"]),
            scheduler=SchedulerConfig(**full["scheduler"]),
            trace=PriorityTrace(seed=seed, **full["trace"]),
            ablation=full["ablation"],
            sync_threshold_ratio=full["swap_policy"]["sync_threshold_ratio"],
            short_request_blocks=full["swap_policy"]["short_request_blocks"],
            prealloc_min_blocks=full["reuse"]["prealloc_min_blocks"],
            prealloc_max_blocks=full["reuse"]["prealloc_max_blocks"],
            release_copy_on_swap_in=full["reuse"]["release_copy_on_swap_in"],
        )
        workload = WorkloadConfig(
            num_conversations=w["num_conversations"],
            arrival_rate_per_s=w["arrival_rate_per_s"],
            mean_turns=w["mean_turns"],
            input_tokens=LengthDist(w["input_tokens"]["median"], w["input_tokens"]["sigma"],
                                    w["input_tokens"]["max"]),
            output_tokens=LengthDist(w["output_tokens"]["median"], w["output_tokens"]["sigma"],
                                     w["output_tokens"]["max"]),
            think_time_mean_s=w["think_time_mean_s"],
            max_context_tokens=w["max_context_tokens"],
            seed=seed,
        )
    except ValueError as exc:
        raise ConfigError("<document>", str(exc)) from exc
    return engine, workload, full


def set_by_path(doc: dict, dotted: str, value: Any) -> None:
    node = doc
    parts = dotted.split(".")
    for p in parts[:-1]:
        node = node.setdefault(p, {})
    node[parts[-1]] = value
