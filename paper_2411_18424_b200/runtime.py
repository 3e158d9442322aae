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


def token_segments(spans, extents_of, block_tokens: int) -> np.ndarray:
    """Token spans [(request, lo, hi)] -> int64 [n, 4] (request, lo, hi,
    physical block of token lo): one row per physically contiguous stretch of
    the request's block table `extents_of(request)` = [(start, length)] in
    logical order (Engine._gpu_extents, engine.py:317-325)."""
    T = block_tokens
    rows = []
    for req, lo, hi in spans:
        if hi <= lo:
            continue
        first, last = lo // T, (hi - 1) // T
        logical = 0
        for start, n in extents_of(req):
            b0, b1 = max(first, logical), min(last, logical + n - 1)
            if b0 <= b1:
                rows.append((req, max(lo, b0 * T), min(hi, (b1 + 1) * T), start + b0 - logical))
            logical += n
            if logical > last:
                break
        if logical <= last:
            raise IndexError(f"request {req}: tokens up to {hi} exceed its block table")
    return np.asarray(rows, dtype=np.int64).reshape(-1, 4)


def swap_rate_summary(iv: dict) -> dict:
    """Per direction, from device intervals [(start_ms, end_ms, bytes)]: GB/s
    while busy; transfers that ran alone (< 10% overlapped by the other
    direction) vs those that overlapped it (> 90%: host-link duplex); plans
    of >= 32 MiB vs smaller ones (fixed cost per launch)."""
    def merged(xs):
        out = []
        for a, b, _ in sorted(xs):
            if out and a <= out[-1][1]:
                out[-1][1] = max(out[-1][1], b)
            else:
                out.append([a, b])
        return out

    def rate(xs):
        t = sum(b - a for a, b, _ in xs)
        return round(sum(n for *_, n in xs) / (t * 1e-3) / 1e9, 2) if t > 0 else None

    res = {}
    for d, o in (("out", "in"), ("in", "out")):
        xs, other = iv.get(d, []), merged(iv.get(o, []))
        alone, duplex = [], []
        for a, b, n in xs:
            ov = sum(max(0.0, min(b, y) - max(a, x)) for x, y in other)
            if b > a and ov / (b - a) < 0.1:
                alone.append((a, b, n))
            elif b > a and ov / (b - a) > 0.9:
                duplex.append((a, b, n))
        big = [x for x in xs if x[2] >= 32 << 20]
        small = [x for x in xs if x[2] < 32 << 20]
        res[d] = {"gib": round(sum(n for *_, n in xs) / 2**30, 2),
                  "transfers": len(xs), "gbs_while_busy": rate(xs),
                  "gbs_alone": rate(alone), "transfers_alone": len(alone),
                  "gbs_overlapping_other_direction": rate(duplex),
                  "transfers_overlapping": len(duplex),
                  "gbs_plans_ge_32mib": rate(big), "gbs_plans_lt_32mib": rate(small),
                  "mean_plan_mib": round(sum(n for *_, n in xs) / len(xs) / 2**20, 2)
                  if xs else None}
    return res


class Runtime:
    def __init__(self, geometry: KVGeometry, gpu_blocks: int, cpu_blocks: int,
                 device="cuda:0", copy_impl: str = "kernel", write_kv: bool = True,
                 verify: bool = False, timing: bool = False,
                 duplex_policy: str = "latency", sm_partition: int = 0,
                 layered_swap_in: bool = False, **executor_kw) -> None:
        if geometry.split_kv:
            raise ValueError("runtime token writes assume fused K/V planes")
        self.geometry = geometry
        self.cache = PagedKVCache(geometry, gpu_blocks, device=device)
        self.host = HostKVPool(cpu_blocks, geometry.block_bytes, numa_node=None, device=device)
        self.dataplane = SwapDataPlane(self.cache, self.host)
        self.executor = StreamExecutor(self.dataplane, copy_impl=copy_impl, timing=timing,
                                       duplex_policy=duplex_policy, sm_partition=sm_partition,
                                       layered_swap_in=layered_swap_in, **executor_kw)
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
        self._mismatch = torch.zeros(1, dtype=torch.int32, device=dev)
        self._kv_bad = torch.zeros(1, dtype=torch.int32, device=dev)
        self.kv_bytes_read = 0

    # -- token KV pattern -----------------------------------------------------

    def _pattern(self, reqs: torch.Tensor, tokens: torch.Tensor) -> torch.Tensor:
        """int32 [n, P, 2, words]: the deterministic KV of each (request, token)
        that kvs_kv_tokens writes (torch restatement, used by tests)."""
        base = (tokens * 0x01000193 + reqs * 0x5BD1E995).view(-1, 1, 1, 1)
        v = (base + self._plane_term + self._kv_term + self._word_term) & 0xFFFFFFFF
        return (v - ((v >> 31) << 32)).to(torch.int32)

    def segments(self, engine, spans) -> np.ndarray:
        return token_segments(spans, engine._gpu_extents, self.geometry.block_tokens)

    # -- engine hooks ------------------------------------------------------------

    def compute(self, engine, spans, skip=()) -> None:
        """One iteration's compute on the compute stream: wait for conflicting
        transfers (except `skip`, already waited for per layer), then write
        the KV of every produced token (one launch)."""
        self.barrier(engine, spans, skip)
        self.write(engine, spans)

    def barrier(self, engine, spans, skip=()) -> None:
        extents = []
        for req, _, _ in spans:
            extents.extend(engine._gpu_extents(req))
        self.barrier_waits += self.executor.compute_barrier(extents, skip=skip)

    def write(self, engine, spans) -> None:
        if not self.write_kv:
            return
        segs = self.segments(engine, spans)
        if len(segs):
            self.dataplane.kv_tokens(0, segs, stream=self.executor.compute)
            self.tokens_written += int((segs[:, 2] - segs[:, 1]).sum())

    @property
    def token_bytes(self) -> int:
        """KV bytes of one token across all planes (K and V)."""
        return self.geometry.block_bytes // self.geometry.block_tokens

    def read_segments(self, engine, spans) -> np.ndarray:
        """The resident-KV segments attend() reads for `spans` (reuse them
        across the per-layer calls of one iteration)."""
        return self.segments(engine, [(req, 0, lo) for req, lo, _ in spans])

    def attend(self, engine, spans, planes: Optional[tuple[int, int]] = None,
               segs: Optional[np.ndarray] = None, stream=None) -> int:
        """Attention stand-in: read (and check) the resident KV of every
        computing request, tokens [0, lo) of each span, in `planes`; returns
        the bytes read.  Mismatches accumulate on the device (kv_errors())."""
        if not self.write_kv:
            return 0
        if segs is None:
            segs = self.read_segments(engine, spans)
        if not len(segs):
            return 0
        self.dataplane.kv_tokens(1, segs, stream=stream or self.executor.compute,
                                 mismatch_ptr=self._kv_bad.data_ptr(), planes=planes)
        tokens = int((segs[:, 2] - segs[:, 1]).sum())
        n = self.geometry.num_planes if planes is None else planes[1] - planes[0]
        nbytes = tokens * self.token_bytes * n // self.geometry.num_planes
        self.kv_bytes_read += nbytes
        return nbytes

    def kv_check_ptr(self) -> int:
        """Device address of the KV-check mismatch counter (captured steps)."""
        return self._kv_bad.data_ptr()

    def account_reads(self, segs: np.ndarray) -> int:
        """Bytes a whole step's KV check of `segs` reads (every plane), counted
        like attend() counts them; returns the bytes."""
        if not self.write_kv or segs is None or not len(segs):
            return 0
        nbytes = int((segs[:, 2] - segs[:, 1]).sum()) * self.token_bytes
        self.kv_bytes_read += nbytes
        return nbytes

    def kv_errors(self) -> int:
        """Words that differed from their tokens' KV in every attend() so far."""
        self.executor.compute.synchronize()
        return int(self._kv_bad.item())

    def swap_in_landed(self, engine, req: int) -> None:
        if not self.verify:
            return
        st = engine.states[req]
        valid = st.context_tokens - st.recompute_tokens
        if valid <= 0:
            return
        self.executor.compute_barrier(engine._gpu_extents(req))
        segs = self.segments(engine, [(req, 0, valid)])
        with torch.cuda.stream(self.executor.compute):
            self._mismatch.zero_()
        self.dataplane.kv_tokens(1, segs, stream=self.executor.compute,
                                 mismatch_ptr=self._mismatch.data_ptr())
        self.executor.compute.synchronize()
        bad = int(self._mismatch.item())
        if bad:
            raise KVIntegrityError(
                f"request {req}: {bad} KV words of its {valid} tokens differ after swap-in "
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
                "kv_bytes_read": self.kv_bytes_read,
                "compute_waits": self.barrier_waits}

    def swap_rates(self) -> dict:
        """Swap GB/s while a transfer of each direction executes (needs
        timing=True), and why it is what it is (swap_rate_summary)."""
        recs = [r for r in self.executor.history if r.nbytes and r.start_event is not None]
        if not recs:
            return {}
        self.synchronize()
        ref = recs[0].start_event
        iv = {"out": [], "in": []}
        for r in recs:
            iv[r.direction].append((ref.elapsed_time(r.start_event), ref.elapsed_time(r.event),
                                    r.nbytes + r.refresh_bytes))
        return swap_rate_summary(iv)

    def close(self) -> None:
        self.synchronize()
        self.dataplane.close()
        self.host.close()
