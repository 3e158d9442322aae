"""Real-bytes runtime attached to an Engine (replay mode).

The engine keeps making the reference's decisions on its simulated clock;
this object gives those decisions real consequences on one GPU:

* every SwapPlan is executed by libkvswap on per-direction streams
  (StreamExecutor, swap.py) — one kernel launch per plan;
* the compute stream writes, for each iteration, the KV of every token the
  iteration produces into the token's paged slot (block table from
  Engine._gpu_extents, engine.py:317-325) after waiting for any transfer
  still touching those blocks (the conflict stall of engine.py:411-414 and
  the swap-in completion of engine.py:376-384, enforced with CUDA events);
* optionally, when a swap-in lands, the request's whole KV is read back and
  compared with the deterministic token pattern: a byte-level end-to-end
  check of block tables, reuse, dirty-tail refresh and stream ordering.

KV slot layout inside a plane chunk (one layer, FlashInfer-style):
[2 (K,V)][block_tokens][heads_per_rank * head_dim * dtype_bytes].
"""

from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from .dataplane import HostKVPool, PagedKVCache, SwapDataPlane
from .geometry import KVGeometry
from .swap import StreamExecutor


class KVIntegrityError(AssertionError):
    """A swapped-in request's KV bytes differ from what its tokens wrote."""


class Runtime:
    def __init__(self, geometry: KVGeometry, gpu_blocks: int, cpu_blocks: int,
                 device="cuda:0", copy_impl: str = "kernel", write_kv: bool = True,
                 verify: bool = False, timing: bool = False,
                 duplex_policy: str = "latency") -> None:
        if geometry.split_kv:
            raise ValueError("runtime token writes assume fused K/V planes")
        self.geometry = geometry
        self.cache = PagedKVCache(geometry, gpu_blocks, device=device)
        self.host = HostKVPool(cpu_blocks, geometry.block_bytes)
        self.dataplane = SwapDataPlane(self.cache, self.host)
        self.executor = StreamExecutor(self.dataplane, copy_impl=copy_impl, timing=timing,
                                       duplex_policy=duplex_policy)
        self.write_kv = write_kv
        self.verify = verify
        self.verified = 0
        self.tokens_written = 0
        self.barrier_waits = 0
        T = geometry.block_tokens
        row = geometry.heads_per_rank * geometry.head_dim * geometry.dtype_bytes
        if row % 4:
            raise ValueError("token row must be a multiple of 4 bytes")
        self._words = row // 4
        # [P, G, 2, T, words] int32 view of the planes
        self._slots = self.cache.planes.view(torch.int32).view(
            geometry.num_planes, gpu_blocks, 2, T, self._words)
        dev = self.cache.device
        self._plane_term = (torch.arange(geometry.num_planes, device=dev, dtype=torch.int64)
                            * 0x9E3779B1).view(1, -1, 1, 1)
        self._kv_term = (torch.arange(2, device=dev, dtype=torch.int64) * 0x7F4A7C15).view(
            1, 1, -1, 1)
        self._word_term = torch.arange(self._words, device=dev, dtype=torch.int64).view(
            1, 1, 1, -1)

    # -- token KV pattern -----------------------------------------------------

    def _pattern(self, reqs: torch.Tensor, tokens: torch.Tensor) -> torch.Tensor:
        """int32 [n, P, 2, words]: deterministic KV of each (request, token)."""
        base = (tokens * 0x01000193 + reqs * 0x5BD1E995).view(-1, 1, 1, 1)
        v = (base + self._plane_term + self._kv_term + self._word_term) & 0xFFFFFFFF
        return (v - ((v >> 31) << 32)).to(torch.int32)

    def _slots_of(self, engine, spans):
        """Flattened (request, token, physical block, slot) for token spans."""
        T = self.geometry.block_tokens
        reqs, toks, phys = [], [], []
        for req, lo, hi in spans:
            if hi <= lo:
                continue
            table = np.concatenate([np.arange(s, s + n) for s, n in engine._gpu_extents(req)])
            t = np.arange(lo, hi, dtype=np.int64)
            reqs.append(np.full(hi - lo, req, dtype=np.int64))
            toks.append(t)
            phys.append(table[t // T])
        if not toks:
            return None
        dev = self.cache.device
        r = torch.from_numpy(np.concatenate(reqs)).to(dev, non_blocking=True)
        t = torch.from_numpy(np.concatenate(toks)).to(dev, non_blocking=True)
        p = torch.from_numpy(np.concatenate(phys)).to(dev, non_blocking=True)
        return r, t, p, t % T

    # -- engine hooks ------------------------------------------------------------

    def compute(self, engine, spans) -> None:
        """One iteration's compute on the compute stream: wait for conflicting
        transfers, then write the KV of every produced token (one scatter)."""
        extents = []
        for req, _, _ in spans:
            extents.extend(engine._gpu_extents(req))
        self.barrier_waits += self.executor.compute_barrier(extents)
        if not self.write_kv:
            return
        with torch.cuda.stream(self.executor.compute):
            got = self._slots_of(engine, spans)
            if got is None:
                return
            r, t, p, slot = got
            self._slots[:, p, :, slot, :] = self._pattern(r, t)
            self.tokens_written += int(t.numel())

    def swap_in_landed(self, engine, req: int) -> None:
        if not self.verify:
            return
        st = engine.states[req]
        valid = st.context_tokens - st.recompute_tokens
        if valid <= 0:
            return
        self.executor.compute_barrier(engine._gpu_extents(req))
        with torch.cuda.stream(self.executor.compute):
            r, t, p, slot = self._slots_of(engine, [(req, 0, valid)])
            got = self._slots[:, p, :, slot, :]
            bad = int((got != self._pattern(r, t)).any(dim=(1, 2, 3)).sum().item())
        if bad:
            raise KVIntegrityError(
                f"request {req}: {bad} of {valid} tokens' KV differ after swap-in "
                f"(iteration {engine.iteration})")
        self.verified += 1

    def forget(self, req: int) -> None:
        pass

    def synchronize(self) -> None:
        self.executor.synchronize()

    def stats(self) -> dict:
        ex = self.executor
        return {"bytes_out": ex.bytes["out"], "bytes_in": ex.bytes["in"],
                "refresh_bytes": ex.refresh_bytes, "kernel_launches": ex.launches,
                "tokens_written": self.tokens_written, "verified_swap_ins": self.verified,
                "compute_waits": self.barrier_waits}

    def close(self) -> None:
        self.synchronize()
        self.dataplane.close()
        self.host.close()
