"""B200-native FastSwitch KV-swap hot path (arXiv 2411.18424).

Drop-in for the kvswitch reference's block-manager / CPU-store / swap-manager
API, with the bytes moved by sm_100a gather/scatter kernels in libkvswap.so.
"""

from .core import BlockSpec, blocks_needed, group_bytes
from .geometry import KVGeometry, LLAMA3_8B, LLAMA3_70B, QWEN25_32B, PRESETS

__all__ = [
    "BlockSpec",
    "blocks_needed",
    "group_bytes",
    "KVGeometry",
    "LLAMA3_8B",
    "QWEN25_32B",
    "LLAMA3_70B",
    "PRESETS",
]
