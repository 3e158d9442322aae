"""KV-cache geometry per tensor-parallel rank.

The reference reduces a block to an opaque byte count, `BlockSpec.bytes_per_block`
(core.py:27-38, default 131072, which matches none of the BASELINE shapes —
SURVEY §0 finding 7).  Here the count is derived from the model's KV shape so
the simulated timing (replay mode) and the real bytes agree:

    chunk  = 2 (K,V) * block_tokens * kv_heads_per_rank * head_dim * dtype_bytes
    block  = num_layers * chunk          (all layers, one rank)

GPU layout: per layer one plane [num_blocks, 2, block_tokens, H_rank, d]
(FlashInfer / vLLM-v1 style); a run of g blocks is one contiguous g*chunk
extent per layer.  `split_kv=True` models the vLLM-v0 [2, num_blocks, ...]
layout as two planes per layer.  Host layout: block-major
[cpu_block][plane][chunk], so a host block group is one contiguous range.
"""

from __future__ import annotations

from dataclasses import dataclass

# ----------------------------------------------------------------------------
# Scalars the whole swap path shares (mirror of kvswitch/core.py:11-65):
# simulated time is an int count of microseconds, so replay-mode decisions are
# bit-exact with the reference; real transfers are timed by CUDA events.
# kvswitch.core's import path is kept by core.py, which re-exports these.
# ----------------------------------------------------------------------------

SimTime = int
RequestId = int
TurnId = int
GroupId = int

US_PER_S = 1_000_000


def elapsed(later: SimTime, earlier: SimTime) -> SimTime:
    """Non-negative difference: a clock never runs backwards (core.py:22-24)."""
    return max(later - earlier, 0)


def _at_least_one(owner: object, *names: str) -> None:
    for n in names:
        v = getattr(owner, n)
        if v < 1:
            raise ValueError(f"{n} must be >= 1, got {v}")


@dataclass(frozen=True)
class BlockSpec:
    """Tokens per KV block, and the bytes a block moves in one swap."""

    block_size_tokens: int = 16
    bytes_per_block: int = 131072  # the reference default; KVGeometry.block_spec() sets it per model

    def __post_init__(self) -> None:
        _at_least_one(self, "block_size_tokens", "bytes_per_block")


def blocks_needed(tokens: int, spec: BlockSpec) -> int:
    """Blocks that hold `tokens` tokens: ceil(tokens / block_size_tokens)."""
    if tokens < 0:
        raise ValueError(f"tokens must be >= 0, got {tokens}")
    return (tokens + spec.block_size_tokens - 1) // spec.block_size_tokens


def group_bytes(num_blocks: int, spec: BlockSpec) -> int:
    """Bytes a run of `num_blocks` consecutive blocks moves."""
    if num_blocks < 0:
        raise ValueError(f"num_blocks must be >= 0, got {num_blocks}")
    return spec.bytes_per_block * num_blocks


@dataclass(frozen=True, order=True)
class Priority:
    """Scheduling order: lower rank first, then lower request id."""

    rank: int
    request_id: RequestId


def priority_key(rank: int, request_id: RequestId) -> tuple[int, RequestId]:
    return rank, request_id


# ----------------------------------------------------------------------------
# Model KV shapes per tensor-parallel rank
# ----------------------------------------------------------------------------


@dataclass(frozen=True)
class KVGeometry:
    name: str
    num_layers: int
    num_kv_heads: int
    head_dim: int
    block_tokens: int = 16
    dtype_bytes: int = 2
    tp: int = 1
    split_kv: bool = False

    def __post_init__(self) -> None:
        for field_name in ("num_layers", "num_kv_heads", "head_dim", "block_tokens",
                           "dtype_bytes", "tp"):
            if getattr(self, field_name) < 1:
                raise ValueError(f"{field_name} must be >= 1")
        if self.num_kv_heads % self.tp:
            raise ValueError(
                f"tp={self.tp} does not divide num_kv_heads={self.num_kv_heads}"
            )
        if self.plane_chunk_bytes % 16:
            raise ValueError("per-plane chunk must be a multiple of 16 bytes")

    @property
    def heads_per_rank(self) -> int:
        return self.num_kv_heads // self.tp

    @property
    def num_planes(self) -> int:
        return self.num_layers * (2 if self.split_kv else 1)

    @property
    def layer_chunk_bytes(self) -> int:
        """K+V bytes of one block in one layer on this rank."""
        return 2 * self.block_tokens * self.heads_per_rank * self.head_dim * self.dtype_bytes

    @property
    def plane_chunk_bytes(self) -> int:
        return self.layer_chunk_bytes // (2 if self.split_kv else 1)

    @property
    def block_bytes(self) -> int:
        """All-layer bytes of one block on one rank (the BlockSpec figure)."""
        return self.num_planes * self.plane_chunk_bytes

    def block_spec(self) -> BlockSpec:
        return BlockSpec(block_size_tokens=self.block_tokens, bytes_per_block=self.block_bytes)

    def with_tp(self, tp: int) -> "KVGeometry":
        return KVGeometry(self.name, self.num_layers, self.num_kv_heads, self.head_dim,
                          self.block_tokens, self.dtype_bytes, tp, self.split_kv)

    def head_slice(self, rank: int) -> tuple[int, int]:
        """KV heads [lo, hi) that TP rank `rank` owns."""
        if not 0 <= rank < self.tp:
            raise ValueError(f"rank {rank} outside tp={self.tp}")
        h = self.heads_per_rank
        return rank * h, (rank + 1) * h


# BASELINE.json shapes (16-token blocks, fp16, d=128, 8 KV heads).
LLAMA3_8B = KVGeometry("llama3-8b", num_layers=32, num_kv_heads=8, head_dim=128)
QWEN25_32B = KVGeometry("qwen2.5-32b", num_layers=64, num_kv_heads=8, head_dim=128)
LLAMA3_70B = KVGeometry("llama3-70b", num_layers=80, num_kv_heads=8, head_dim=128)

PRESETS = {g.name: g for g in (LLAMA3_8B, QWEN25_32B, LLAMA3_70B)}
