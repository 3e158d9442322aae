"""Multithreading Swap Manager on real streams — drop-in for kvswitch.swap.

Two layers, one object:

1. The reference's bookkeeping, bit-exact (pkg/src/kvswitch/swap.py):
   one serial dispatcher (+dispatch_per_op per op) feeding one copy pipeline
   per direction (finish = max(dispatch, prev) + exec_time), per-op OpRecord
   busy extents for D2H sources, half-open conflict detection,
   max-over-blockers resolution, dispatch-queue yield, adaptive sync/async
   (decide_mode) and the r_info window.  In replay mode these simulated
   timestamps drive every engine decision, exactly as in the reference.

2. The B200 execution layer (`StreamExecutor`): each dispatched plan is ONE
   libkvswap kernel launch on a low-priority per-direction stream (the
   paper's dispatch thread pool, becomes unnecessary: dispatch
   is O(1) per plan).  Real hazards are enforced with CUDA events, independent
   of simulated time:
     * both directions wait for the compute work queued before them (swap-out
       reads the KV compute produced; swap-in must not overtake compute's
       writes to blocks freed without a swap-out);
     * a transfer waits for any still-running opposite-direction transfer
       whose GPU or host extents it would overwrite or read stale
       (WAR/RAW/WAW; same-direction transfers are already stream-ordered);
     * compute waits for transfers that write blocks it is about to read or
       that still read blocks it is about to write (engine.py:411-414 conflict
       stall and the swap-in completion of engine.py:376-384, made real).
"""

from __future__ import annotations

import time
from collections import deque
from dataclasses import dataclass, field
from typing import Iterable, Optional

from .core import RequestId, SimTime, elapsed
from .costmodel import TransferParams
from .cpu_store import SwapPlan

R_INFO_WINDOW = 64


@dataclass
class SwapEvent:
    iteration: int
    request: RequestId
    direction: str
    ops: int
    blocks: int
    dispatch_done: SimTime
    exec_done: SimTime
    conflicts: int = 0


@dataclass
class OpRecord:
    """GPU extent [gpu_start, gpu_start+gpu_len) busy until exec_done (swap.py:36-42)."""

    gpu_start: int
    gpu_len: int
    exec_done: SimTime


@dataclass
class InFlightSwap:
    request: RequestId
    direction: str
    plan: SwapPlan
    dispatch_done: SimTime
    exec_done: SimTime
    op_records: list[OpRecord]
    transfer: Optional["TransferRecord"] = None  # real execution, when attached

    def completed(self, clock: SimTime) -> bool:
        return clock >= self.exec_done


@dataclass
class QueueState:
    """waiting / running / swapped / ongoing_swap_in partition (swap.py:58-104)."""

    waiting: list[RequestId] = field(default_factory=list)
    running: list[RequestId] = field(default_factory=list)
    swapped: list[RequestId] = field(default_factory=list)
    ongoing_swap_in: list[RequestId] = field(default_factory=list)
    r_info: deque = field(default_factory=lambda: deque(maxlen=R_INFO_WINDOW))

    def _queues(self) -> dict[str, list[RequestId]]:
        return {"waiting": self.waiting, "running": self.running,
                "swapped": self.swapped, "ongoing_swap_in": self.ongoing_swap_in}

    def location(self, req: RequestId) -> Optional[str]:
        for name, q in self._queues().items():
            if req in q:
                return name
        return None

    def remove(self, req: RequestId) -> None:
        for q in self._queues().values():
            if req in q:
                q.remove(req)

    def move(self, req: RequestId, dst: str) -> None:
        self.remove(req)
        self._queues()[dst].append(req)

    def validate_partition(self, live: Iterable[RequestId]) -> None:
        seen: set[RequestId] = set()
        for q in self._queues().values():
            for req in q:
                if req in seen:
                    raise AssertionError(f"request {req} appears in two queues")
                seen.add(req)
        live = set(live)
        if seen != live:
            raise AssertionError(f"queues cover {sorted(seen)} but live set is {sorted(live)}")


@dataclass
class StrategyDecision:
    mode: str  # "async" | "sync"
    reason: str  # small_short_requests | long_transfers | idle_io | forced_sync


def decide_mode(pending_drain: SimTime, pending_max_footprint: int, iter_estimate: SimTime,
                sync_threshold_ratio: float, short_request_blocks: int,
                forced: Optional[str] = None) -> StrategyDecision:
    """Adaptive swap-in strategy (swap.py:113-135): absorb a quick drain of
    small swap-ins as one stall; let long transfers overlap inference."""
    if forced == "sync":
        return StrategyDecision("sync", "forced_sync")
    if pending_max_footprint == 0:
        return StrategyDecision("async", "idle_io")
    quick = pending_drain < sync_threshold_ratio * iter_estimate
    if quick and pending_max_footprint < short_request_blocks:
        return StrategyDecision("sync", "small_short_requests")
    return StrategyDecision("async", "long_transfers")


# --------------------------------------------------------------------------
# Real execution
# --------------------------------------------------------------------------

def _overlaps(a: list[tuple[int, int]], b: list[tuple[int, int]]) -> bool:
    for s0, n0 in a:
        e0 = s0 + n0
        for s1, n1 in b:
            if s0 < s1 + n1 and s1 < e0:
                return True
    return False


def _hit_ops(extents: list[tuple[int, int]], per_op: list[tuple[int, int]]) -> list[int]:
    """Indices of ops whose extent intersects any of `extents` (half-open)."""
    hits = []
    for i, (s1, n1) in enumerate(per_op):
        e1 = s1 + n1
        for s0, n0 in extents:
            if s0 < e1 and s1 < s0 + n0:
                hits.append(i)
                break
    return hits


@dataclass
class TransferRecord:
    direction: str
    gpu: list[tuple[int, int]]  # per TransferOp
    host: list[tuple[int, int]]  # per TransferOp
    event: object  # torch.cuda.Event
    nbytes: int
    refresh_bytes: int
    start_event: object = None
    done: bool = False
    flag_base: Optional[int] = None  # op-flag slots [flag_base, flag_base + n_ops)
    seq: int = 0
    submitted: float = 0.0  # host perf_counter at submit (diagnostics)
    deps: int = 0  # cross-stream waits this transfer was issued behind
    plane_base: Optional[int] = None  # plane-flag slots [plane_base, + num_planes)
    flag_span: int = 0  # flag slots this transfer owns (op + plane flags)

    def poll(self) -> bool:
        if not self.done and self.event.query():
            self.done = True
        return self.done


COPY_IMPLS = ("kernel", "ce_per_block", "ce_per_run", "ce_staged")

# Launch shape and pacing per direction (profiles/r01_interference_*.json,
# profiles/r01_duplex_bw.json).  Unpaced, SM stores to host memory are issued
# far faster than PCIe drains them and back up the XBAR/L2 queues that
# decode's HBM traffic shares: a concurrent 2 ms decode step slowed 1.2-4.9x.
# Swap-out is therefore paced below the link rate (posted writes have no
# natural bound).  Swap-in is bounded by its reads in flight instead: 8 CTAs
# x 256 threads x 4 KiB per warp = 256 KiB outstanding covers the PCIe
# round trip at ~51.4 GB/s without building a queue, and unlike a pace it has
# no cliff when a box's link is a little slower than the pace (a pace above
# the link rate behaves like no pace: +35% decode).  Measured with a 2 ms
# static-partition decode: out 51.9 GB/s +3-4%, in 51.2-51.4 GB/s +9.2%
# (profiles/r01_interference_policy.json).
#   latency    — serving: out 8x512 @52 GB/s, in 8x256 in-flight bound, both
#                directions together capped at 60 GB/s (shared budget);
#   throughput — bulk migration: unpaced TMA bulk kernels, 64 CTAs each way
#                (both directions at once: 80 GB/s combined vs 75 with the
#                LSU kernel, profiles/r01_duplex_mix.json; plan-level waits;
#                decode pays for it);
#   latency_share — latency, but swap-in holds a reserved 42 GB/s of the
#                60 GB/s budget (kvs_set_budget_share): under FCFS a burst of
#                preemptions leaves a concurrent resume ~10 GB/s; strict
#                swap-in priority starves the preemptions instead;
#   throughput_mix — bulk migration with one engine per direction: swap-out
#                on the TMA bulk kernel, swap-in on the copy engines (staged:
#                whole host runs into an HBM ring, then a scatter kernel).
#                SM-issued host traffic in both directions tops out at 75-80
#                GB/s combined, and one engine per direction avoids that cap
#                (profiles/r02_e2e_policy_probe.json); plan-level waits;
#   throughput_staged — bulk migration with both directions on the staged
#                copy-engine path (larger PCIe TLPs than SM-issued traffic);
#   unpaced    — out 8x512, in 32x512, no pacing (round-1 default shape).
DUPLEX_POLICIES = {
    "latency": {"out": (8, 512, 52.0), "in": (8, 256, 0.0), "budget": 60.0},
    # same, but swap-in draws on the shared budget first (kvs_set_budget_priority)
    "latency_in_first": {"out": (8, 512, 52.0), "in": (8, 256, 0.0), "budget": 60.0,
                         "priority": "in"},
    "latency_share": {"out": (8, 512, 52.0), "in": (8, 256, 0.0), "budget": 60.0,
                      "share": {"in": 42.0}},
    # serving: swap-in paced at 48 GB/s (bounded by reads in flight as
    # well), swap-out at 52, with 42 GB/s of a 60 GB/s budget reserved for
    # swap-in while both run; the decode step launched as one CUDA graph
    # (live.DecodeGraph).  On the live stress trace the pace costs swap-in
    # nothing while busy (46.6 vs 46.7 GB/s: the traces' plans average ~146
    # MiB and do not reach the link rate) and cuts the swap-induced stall
    # from 9.1-9.7% to 8.4% [7.8, 9.0] (profiles/r02_live_stall_pace.json,
    # DESIGN §3.3).
    "serving": {"out": (8, 512, 52.0), "in": (8, 256, 48.0), "budget": 60.0,
                "share": {"in": 42.0}},
    # serving_link: the same at the link rate (swap-in unpaced, 51.4 GB/s =
    # 82% of the link on long plans): +9.1% on a 32-layer step that
    # overlaps it throughout, 9.1-9.7% on the live stress trace.
    "serving_link": {"out": (8, 512, 52.0), "in": (8, 256, 0.0), "budget": 60.0,
                     "share": {"in": 42.0}},
    # serving_paced: for decode kernels launched one by one on a stream, whose
    # command fetches queue behind a saturating swap-in's PCIe reads: paced
    # below the link (in 40 / out 20 GB/s) the stall stays under 10%
    # (profiles/r02_live_policy_probe.json).
    "serving_paced": {"out": (8, 512, 20.0), "in": (8, 256, 40.0), "budget": 60.0},
    # the serving policy on the TMA bulk kernels (op / plane flags from the
    # elected thread's store side): same pace and budget, fewer SM threads
    "latency_bulk": {"out": (8, 0, 52.0), "in": (8, 0, 0.0), "budget": 60.0, "path": "bulk"},
    "throughput": {"out": (64, 0, 0.0), "in": (64, 0, 0.0), "budget": 0.0, "path": "bulk",
                   "signals": "plan"},
    "throughput_mix": {"out": (64, 0, 0.0), "in": (64, 0, 0.0), "budget": 0.0,
                       "path": "bulk", "engine": {"in": "ce_staged"}, "signals": "plan"},
    "throughput_staged": {"out": (64, 0, 0.0), "in": (64, 0, 0.0), "budget": 0.0,
                          "path": "bulk", "engine": {"out": "ce_staged", "in": "ce_staged"},
                          "signals": "plan"},
    "unpaced": {"out": (8, 512, 0.0), "in": (32, 512, 0.0), "budget": 0.0},
}

# Waiting on more op flags than this costs more driver calls than the
# plan-level event saves.
MAX_OP_WAITS = 8
FLAG_RING = 1 << 20


_PARTITIONS: dict = {}


def partition_streams(device, swap_sms: int):
    """One green-context partition per (device, swap_sms) per process (they
    live until exit): ((out stream, in stream), compute stream, (swap SMs,
    compute SMs))."""
    from .dataplane import sm_partition

    key = (str(device), swap_sms)
    if key not in _PARTITIONS:
        _PARTITIONS[key] = sm_partition(device, swap_sms=swap_sms, swap_streams=2)
    return _PARTITIONS[key]


class StreamExecutor:
    """Real streams + event hazards around one SwapDataPlane (one rank).

    With the kernel path every plan is issued through kvs_swap_ops, so each
    TransferOp publishes its own completion word: conflicting work waits for
    the blocking ops only (the reference resolves conflicts per op,
    swap.py:236-252), falling back to the plan's event when many ops block.
    """

    def __init__(self, dataplane, compute_stream=None, copy_impl: str = "kernel",
                 timing: bool = False, duplex_policy: str = "latency",
                 op_granular: bool = True, sm_partition: int = 0,
                 layered_swap_in: bool = False, flag_ring: int = FLAG_RING) -> None:
        import torch

        if copy_impl not in COPY_IMPLS:
            raise ValueError(f"copy_impl must be one of {COPY_IMPLS}")
        self.torch = torch
        self.dp = dataplane
        dev = dataplane.cache.device
        self.sm_split = None
        if sm_partition:
            # Swap streams on their own SM group, compute on the rest (green
            # contexts, kvs_sm_partition): SM-issued host traffic never shares
            # an SM with a decode CTA.
            (s_out, s_in), part_compute, self.sm_split = partition_streams(dev, sm_partition)
            self.streams = {"out": s_out, "in": s_in}
            if compute_stream is None:
                compute_stream = part_compute
        else:
            self.streams = {
                "out": torch.cuda.Stream(device=dev, priority=0),
                "in": torch.cuda.Stream(device=dev, priority=0),
            }
        self.compute = compute_stream if compute_stream is not None else \
            torch.cuda.Stream(device=dev, priority=-1)
        self.copy_impl = copy_impl
        self.timing = timing
        self._op_granular_wanted = op_granular and copy_impl == "kernel"
        self.op_granular = self._op_granular_wanted
        # Swap-ins also publish one flag per plane (layer), moved plane-major,
        # so compute can join a resumed request layer by layer (wait_plane).
        self._layered_wanted = layered_swap_in
        self.layered_swap_in = layered_swap_in and self.op_granular
        self.num_planes = dataplane.geometry.num_planes
        self.pending: list[TransferRecord] = []
        self.history: list[TransferRecord] = []
        self.bytes = {"out": 0, "in": 0}
        self.refresh_bytes = 0
        self.launches = 0
        self.op_waits = 0
        self.plan_waits = 0
        self.last_barrier: list[tuple] = []
        self.block_bytes = dataplane.geometry.block_bytes
        self.flag_ring = flag_ring
        self._flags = torch.zeros(flag_ring, dtype=torch.int32, device=dev)
        self._flags_ptr = self._flags.data_ptr()
        self._flag_head = 0
        self._seq = 0
        self.set_duplex_policy(duplex_policy)

    def set_duplex_policy(self, policy: str) -> None:
        if policy not in DUPLEX_POLICIES:
            raise ValueError(f"duplex policy must be one of {sorted(DUPLEX_POLICIES)}")
        pol = DUPLEX_POLICIES[policy]
        path = pol.get("path", "lsu")
        for direction in ("out", "in"):
            ctas, threads, pace = pol[direction]
            self.dp.set_path(direction, path)
            self.dp.set_launch(direction, ctas, threads)
            self.dp.set_pace(direction, pace)
        self.dp.set_budget(pol["budget"])
        self.dp.set_budget_priority(pol.get("priority"))
        for direction in ("out", "in"):
            self.dp.set_budget_share(direction, pol.get("share", {}).get(direction, 0.0))
        # Engine per direction: the kernel unless the policy routes one
        # direction's plans to the copy engines (plan-level completion only).
        self.engine = {d: pol.get("engine", {}).get(d, self.copy_impl) for d in ("out", "in")}
        # Both kernel paths publish op / plane flags; a policy may choose
        # plan-level completion only ("signals": "plan": bulk migration).
        self.op_granular = self._op_granular_wanted and pol.get("signals", "op") == "op"
        self.layered_swap_in = (self._layered_wanted and self.op_granular
                                and self.engine["in"] == "kernel")
        self.duplex_policy = policy

    def _prune(self) -> None:
        self.pending = [r for r in self.pending if not r.poll()]

    def _claim_flags(self, n: int) -> int:
        if n > self.flag_ring:
            raise ValueError(f"a transfer needs {n} completion words, ring holds {self.flag_ring}")
        if self._flag_head + n > self.flag_ring:
            self._flag_head = 0
        base = self._flag_head
        for r in self.pending:  # never recycle slots a live transfer still signals
            if r.flag_base is not None and r.flag_base < base + n and base < r.flag_base + r.flag_span:
                r.event.synchronize()
        self._flag_head += n
        return base

    def _wait(self, stream, rec: TransferRecord, ops: list[int]) -> None:
        """`stream` waits for ops `ops` of `rec` (or the whole plan)."""
        if rec.flag_base is not None and len(ops) <= MAX_OP_WAITS:
            for i in ops:
                self.dp.wait_flag(stream, self._flags_ptr + 4 * (rec.flag_base + i), rec.seq)
            self.op_waits += len(ops)
        else:
            stream.wait_event(rec.event)
            self.plan_waits += 1

    def submit(self, direction: str, ops, split_single: bool = False,
               refresh_blocks: int = 0) -> TransferRecord:
        torch = self.torch
        self._prune()
        gpu = [(op.gpu_start, op.blocks) for op in ops]
        host = [(op.cpu_start, op.blocks) for op in ops]
        stream = self.streams[direction]
        # Both directions start after the compute work already queued: a
        # swap-out reads KV that compute produced; a swap-in may overwrite
        # blocks compute last wrote for a request that just finished or was
        # dropped for recompute (freed without a swap-out, engine.py:409-414,
        # 538-545), so it must not overtake those writes (WAW).  Compute that
        # is queued later (per-layer waits, barriers) is not waited for.
        stream.wait_stream(self.compute)
        deps = 0
        for r in self.pending:
            if r.direction == direction:
                continue  # same stream: already ordered
            # out: writes host (WAR/WAW vs r), reads GPU r writes (RAW, r = in);
            # in:  reads host r = out writes (RAW), writes GPU r touches (WAR/WAW).
            if direction == "out":
                hits = set(_hit_ops(host, r.host))
                if r.direction == "in":
                    hits |= set(_hit_ops(gpu, r.gpu))
            else:
                hits = set(_hit_ops(gpu, r.gpu))
                if r.direction == "out":
                    hits |= set(_hit_ops(host, r.host))
            if hits:
                self._wait(stream, r, sorted(hits))
                deps += 1
        start = None
        if self.timing:
            start = torch.cuda.Event(enable_timing=True)
            start.record(stream)
        flag_base, seq, plane_base, span = None, 0, None, 0
        if ops:
            if self.engine[direction] == "kernel":
                if self.op_granular:
                    layered = self.layered_swap_in and direction == "in"
                    span = len(ops) + (self.num_planes if layered else 0)
                    flag_base = self._claim_flags(span)
                    self._seq += 1
                    seq = self._seq
                    op_ptr = self._flags_ptr + 4 * flag_base
                    if layered:
                        plane_base = flag_base + len(ops)
                        self.dp.swap_signaled(direction, ops, seq, op_flags=op_ptr,
                                              plane_flags=self._flags_ptr + 4 * plane_base,
                                              stream=stream)
                    else:
                        self.dp.swap_ops(direction, ops, op_ptr, seq, stream=stream)
                else:
                    self.dp.swap(direction, ops, stream=stream)
                self.launches += 1
            else:
                mode = COPY_IMPLS.index(self.engine[direction]) - 1
                self.dp.baseline(direction, mode, ops, stream=stream)
        ev = torch.cuda.Event(enable_timing=self.timing)
        ev.record(stream)
        blocks = sum(op.blocks for op in ops)
        rec = TransferRecord(direction, gpu, host, ev, blocks * self.block_bytes,
                             refresh_blocks * self.block_bytes, start, False, flag_base, seq,
                             time.perf_counter(), deps, plane_base, span)
        self.bytes[direction] += rec.nbytes
        self.refresh_bytes += rec.refresh_bytes
        self.pending.append(rec)
        if self.timing:
            self.history.append(rec)
        return rec

    def plane_flags(self, rec: TransferRecord) -> tuple[int, int]:
        """(device address of a layered transfer's per-plane flag array, the
        value each flag receives): what a captured decode step waits on."""
        if rec.plane_base is None:
            raise ValueError("transfer was not issued plane-major (layered_swap_in)")
        return self._flags_ptr + 4 * rec.plane_base, rec.seq

    def wait_plane(self, stream, rec: TransferRecord, plane: int) -> None:
        """`stream` waits until plane `plane` of a layered transfer has landed."""
        if rec.plane_base is None:
            raise ValueError("transfer was not issued plane-major (layered_swap_in)")
        self.dp.wait_flag(stream, self._flags_ptr + 4 * (rec.plane_base + plane), rec.seq)

    def compute_barrier(self, extents: list[tuple[int, int]], skip=()) -> int:
        """Make the compute stream wait for transfers touching `extents`
        (their blocking ops only, when op flags exist); transfers in `skip`
        are being waited for another way (per plane).

        Returns the number of transfers waited on (real conflicts)."""
        self._prune()
        n = 0
        self.last_barrier = []  # (direction, age_ms, ops waited, its deps, MiB)
        for r in self.pending:
            if any(r is k for k in skip):
                continue
            hits = _hit_ops(extents, r.gpu)
            if hits:
                self._wait(self.compute, r, hits)
                self.last_barrier.append((r.direction, round((time.perf_counter() - r.submitted)
                                                             * 1e3, 2), len(hits), r.deps,
                                          r.nbytes >> 20))
                n += 1
        return n

    def wait_transfer(self, rec: TransferRecord) -> None:
        self.compute.wait_event(rec.event)

    def host_fence(self, rows: list[tuple[int, int]]) -> int:
        """Block the calling host thread until every pending transfer whose
        host extents overlap `rows` ([(start, length)] host blocks) is done,
        so the CPU may read or write those pool rows.  Returns how many
        transfers it waited for."""
        self._prune()
        n = 0
        for r in self.pending:
            if _overlaps(rows, r.host):
                r.event.synchronize()
                n += 1
        self._prune()
        return n

    def synchronize(self) -> None:
        for s in self.streams.values():
            s.synchronize()
        self.compute.synchronize()
        self._prune()


class SwapManager:
    """Dispatcher / copy-engine timelines and in-flight swaps (swap.py:138-285),
    optionally executing every plan's bytes through a StreamExecutor."""

    def __init__(self, params: TransferParams, split_ops_to_single_blocks: bool = False,
                 bytes_per_block: int = 131072,
                 executor: Optional[StreamExecutor] = None) -> None:
        self.params = params
        self.split_single = split_ops_to_single_blocks
        self.bytes_per_block = bytes_per_block
        self.executor = executor
        self.dispatcher_free_at: SimTime = 0
        self.ops_since_yield = 0
        self.engine_free_at: dict[str, SimTime] = {"in": 0, "out": 0}
        self.in_flight: list[InFlightSwap] = []
        self.busy_extents: list[OpRecord] = []
        self.events_log: list[SwapEvent] = []
        self.total_ops = {"in": 0, "out": 0}
        self.total_blocks = {"in": 0, "out": 0}

    # step 1 --------------------------------------------------------------

    def pop_completed(self, clock: SimTime) -> list[InFlightSwap]:
        """Swaps whose (simulated) execution has finished, in (exec_done, request) order."""
        finished, running = [], []
        for s in self.in_flight:
            (finished if s.exec_done <= clock else running).append(s)
        self.in_flight = running
        self.busy_extents = [r for r in self.busy_extents if r.exec_done > clock]
        finished.sort(key=lambda s: (s.exec_done, s.request))
        return finished

    def pending_swap_ins(self) -> list[InFlightSwap]:
        return [s for s in self.in_flight if s.direction == "in"]

    # steps 2-3 -------------------------------------------------------------

    def _op_sizes(self, plan: SwapPlan) -> list[tuple[int, int, int]]:
        """(gpu_start, blocks, bytes) per issued op; one per block in split mode."""
        bpb = self.bytes_per_block
        if not self.split_single:
            return [(op.gpu_start, op.blocks, op.blocks * bpb) for op in plan.ops]
        return [(op.gpu_start + i, 1, bpb) for op in plan.ops for i in range(op.blocks)]

    def dispatch(self, clock: SimTime, iteration: int, plan: SwapPlan,
                 not_before: SimTime = 0) -> InFlightSwap:
        """Queue a plan; `not_before` delays execution, never dispatch."""
        p = self.params
        issued = self._op_sizes(plan)
        t_disp = max(clock, self.dispatcher_free_at)
        t_exec = max(self.engine_free_at[plan.direction], not_before)
        records: list[OpRecord] = []
        for gpu_start, blocks, nbytes in issued:
            t_disp += p.dispatch_per_op
            t_exec = max(t_exec, t_disp) + p.exec_time(nbytes)
            records.append(OpRecord(gpu_start, blocks, t_exec))
        self.ops_since_yield = (self.ops_since_yield + len(issued)) % p.sync_batch
        exec_done = t_exec if issued else max(clock, not_before)
        self.dispatcher_free_at = t_disp
        self.engine_free_at[plan.direction] = exec_done

        flight = InFlightSwap(plan.request, plan.direction, plan, t_disp, exec_done, records)
        if self.executor is not None:
            flight.transfer = self.executor.submit(plan.direction, plan.all_ops(),
                                                   split_single=self.split_single,
                                                   refresh_blocks=plan.refresh_blocks)
        self.in_flight.append(flight)
        if plan.direction == "out":
            self.busy_extents.extend(records)  # freed sources stay busy until exec_done
        self.total_ops[plan.direction] += len(issued)
        self.total_blocks[plan.direction] += plan.moved_blocks
        self.events_log.append(SwapEvent(iteration, plan.request, plan.direction, len(issued),
                                         plan.moved_blocks, t_disp, exec_done))
        return flight

    # step 3.1 --------------------------------------------------------------

    def detect_conflicts(self, clock: SimTime, grants: list[tuple[int, int]]) -> list[OpRecord]:
        """Busy D2H extents (exec_done > clock) intersecting any grant, half-open."""
        hits = []
        for start, length in grants:
            end = start + length
            for rec in self.busy_extents:
                if rec.exec_done > clock and start < rec.gpu_start + rec.gpu_len \
                        and rec.gpu_start < end:
                    hits.append(rec)
        return hits

    @staticmethod
    def resolve_conflicts(clock: SimTime, conflicts: list[OpRecord]) -> SimTime:
        return max((elapsed(r.exec_done, clock) for r in conflicts), default=0)

    def yield_stall(self, clock: SimTime) -> SimTime:
        """Bounded wait for the dispatch queue's next yield point (swap.py:256-268)."""
        if self.dispatcher_free_at <= clock:
            return 0
        p = self.params
        backlog = -(-(self.dispatcher_free_at - clock) // p.dispatch_per_op)
        to_yield = (p.sync_batch - self.ops_since_yield) % p.sync_batch
        return min(backlog, to_yield) * p.dispatch_per_op

    # r_info -----------------------------------------------------------------

    def record_event(self, qs: QueueState, event: SwapEvent) -> None:
        qs.r_info.append(event)

    @staticmethod
    def r_info_summary(qs: QueueState) -> dict[str, float]:
        if not qs.r_info:
            return {"events": 0, "ops": 0, "blocks": 0, "mean_exec_us": 0.0}
        spans = [max(0, e.exec_done - e.dispatch_done) for e in qs.r_info]
        return {"events": len(qs.r_info), "ops": sum(e.ops for e in qs.r_info),
                "blocks": sum(e.blocks for e in qs.r_info),
                "mean_exec_us": sum(spans) / len(spans)}
