"""Live mode: the engine loop driven by real GPU time.

Replay mode (engine.py) reproduces the reference's decisions on its
simulated clock.  Live mode keeps every decision *rule* of the reference
(same scheduler, allocator, reuse store, adaptive sync/async) but lets the
B200 decide *when* things happen:

* the clock is wall time of this process (idle gaps between arrivals are
  skipped, as the reference's loop does at engine.py:366-371);
* a swap-in completes when its kernel's CUDA event completes
  (engine.py:376-384 step 1 made real), not at a modeled exec_done;
* an iteration's compute is a real HBM-streaming kernel on a high-priority
  stream, sized to the reference's iteration_time (costmodel.py:74-82), so
  swap kernels and "decode" contend for SMs / L2 / HBM like in serving;
* conflicts (grants over blocks a D2H is still reading, engine.py:411-414)
  and sync swap-ins (engine.py:436-446) become real stream waits whose cost
  lands in the measured iteration time.

Reported: P50/P95/P99 TTFT, P99/P99.9 TBT (real microseconds), swap GB/s
while serving, and swap-induced decode stall = decode-kernel time with
concurrent swaps / the same kernel alone - 1.  Decisions legitimately
diverge from replay (SURVEY §0 finding 6); correctness is the byte check.
"""

from __future__ import annotations

import ctypes
import gc
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .costmodel import TransferParams, iteration_time
from .core import elapsed
from .engine import (EFFICIENCY_INTERVAL_ITERS, RUNNING, SWAPPING_IN, Engine, EngineConfig,
                     IterationRecord, MetricsReport, percentile)
from .swap import decide_mode

LIVE_DEADLOCK_ITERATIONS = 200_000


def b200_transfer_params(gbs: float = 51.0) -> TransferParams:
    """Cost-model stand-in for *predictions* in live mode: one launch per plan
    (dispatch ~ 1 us/op amortised), measured PCIe rate."""
    return TransferParams(dispatch_per_op=1, bandwidth=int(gbs * 1000), per_op_latency_floor=2,
                          sync_batch=8)


class DecodeEmulator:
    """Weight-streaming decode stand-in (include/kvswap_workload.h)."""

    def __init__(self, device, weight_bytes: int = 16 << 30, ctas: int = 0,
                 stream=None) -> None:
        """`stream`: where decode will run (calibrated there, e.g. the compute
        side of an SM partition); `ctas` 0 = 2 x the device's SMs."""
        self.lib = _lib.load()
        self.device = torch.device(device)
        self.index = self.device.index if self.device.index is not None else 0
        self.weights = torch.empty(weight_bytes, dtype=torch.uint8, device=self.device)
        self.weights.view(torch.int32).random_()
        self.sink = torch.zeros(4, dtype=torch.int32, device=self.device)
        torch.cuda.synchronize(self.device)  # calibrate on an idle GPU
        self.ctas = ctas
        self.stream = stream
        self.bytes_per_us = self.calibrate()

    def launch(self, stream, nbytes: int) -> None:
        rc = self.lib.kvs_stream_read(self.index, int(stream.cuda_stream),
                                      ctypes.c_void_p(self.weights.data_ptr()),
                                      self.weights.numel(), int(nbytes), self.ctas,
                                      ctypes.c_void_p(self.sink.data_ptr()))
        _lib.check(rc, "kvs_stream_read")

    def bytes_for_us(self, us: float) -> int:
        return max(16, int(us * self.bytes_per_us) // 16 * 16)

    def launch_us(self, stream, us: float) -> int:
        nbytes = self.bytes_for_us(us)
        self.launch(stream, nbytes)
        return nbytes

    def calibrate(self, nbytes: int = 8 << 30) -> float:
        s = self.stream if self.stream is not None else torch.cuda.Stream(device=self.device)
        self.launch(s, nbytes)
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(3):
            self.launch(s, nbytes)
        e1.record(s)
        s.synchronize()
        return 3 * nbytes / (e0.elapsed_time(e1) * 1e3)


class DecodeGraph:
    """A decode step launched as one CUDA graph (kvs_graph_*, include/
    kvswap_workload.h), as serving engines launch a model's per-layer decode.

    Each iteration the step is re-captured on the graph's private stream and
    the executable graph is updated in place (cudaGraphExecUpdate) — the
    structure is fixed (attention + weight kernel per layer, plane-flag waits
    in layered steps) while the batch and modeled time change.  Why it
    matters for the swap path: stream-launched kernels fetch
    their commands from host memory over the PCIe link a swap-in saturates."""

    def __init__(self, device, marks: int = 160) -> None:
        self.lib = _lib.load()
        dev = torch.device(device)
        idx = dev.index if dev.index is not None else torch.cuda.current_device()
        h = ctypes.c_void_p()
        _lib.check(self.lib.kvs_graph_create(idx, marks, ctypes.byref(h)), "kvs_graph_create")
        self.h = h
        self.marks = marks
        st = ctypes.c_uint64()
        _lib.check(self.lib.kvs_graph_stream(h, ctypes.byref(st)), "kvs_graph_stream")
        self.stream = torch.cuda.ExternalStream(st.value, device=torch.device("cuda", idx))

    def begin(self) -> torch.cuda.Stream:
        _lib.check(self.lib.kvs_graph_begin(self.h), "kvs_graph_begin")
        return self.stream

    def mark(self, slot: int) -> None:
        _lib.check(self.lib.kvs_graph_mark(self.h, slot), "kvs_graph_mark")

    def end(self) -> int:
        how = ctypes.c_int()
        _lib.check(self.lib.kvs_graph_end(self.h, ctypes.byref(how)), "kvs_graph_end")
        return how.value

    def launch(self, stream) -> None:
        _lib.check(self.lib.kvs_graph_launch(self.h, int(stream.cuda_stream)), "kvs_graph_launch")

    def capture_step(self, dataplane, decode: "DecodeEmulator", segs, mismatch_ptr: int,
                     w_bytes_per_layer: int, deps=(), marks: bool = False) -> int:
        """Capture a whole decode step in one native call
        (kvs_graph_decode_step): per layer, the plane-flag waits of `deps`
        ((flag array address, seq) pairs), the KV check of `segs` in that
        plane, and `w_bytes_per_layer` of weight streaming; marks 2l / 2l+1
        around layer l.  Returns how the executable graph was refreshed."""
        arr = None
        if segs is not None and len(segs):
            arr = np.ascontiguousarray(segs, dtype=np.int64).reshape(-1, 4)
        n_deps = len(deps)
        flags = (ctypes.c_uint64 * max(1, n_deps))(*[int(p) for p, _ in deps])
        seqs = (ctypes.c_uint32 * max(1, n_deps))(*[int(q) & 0xFFFFFFFF for _, q in deps])
        st = _lib.KvsDecodeStep(
            arr.ctypes.data if arr is not None else None, 0 if arr is None else arr.shape[0],
            dataplane.geometry.block_tokens, mismatch_ptr or None,
            decode.weights.data_ptr(), decode.weights.numel(), int(w_bytes_per_layer),
            decode.sink.data_ptr(), decode.ctas, n_deps,
            ctypes.addressof(flags) if n_deps else None,
            ctypes.addressof(seqs) if n_deps else None, 1 if marks else 0, 0)
        how = ctypes.c_int()
        _lib.check(self.lib.kvs_graph_decode_step(self.h, dataplane.handle, ctypes.byref(st),
                                                  ctypes.byref(how)), "kvs_graph_decode_step")
        return how.value

    def elapsed(self, a: int, b: int) -> float:
        ms = ctypes.c_float()
        _lib.check(self.lib.kvs_graph_elapsed(self.h, a, b, ctypes.byref(ms)),
                   "kvs_graph_elapsed")
        return ms.value

    def stats(self) -> dict:
        out = (ctypes.c_int64 * 3)()
        _lib.check(self.lib.kvs_graph_stats(self.h, out), "kvs_graph_stats")
        return {"instantiations": out[0], "updates": out[1], "launches": out[2]}

    def close(self) -> None:
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.kvs_graph_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self) -> None:  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


@dataclass
class LiveStats:
    decode_ms: float = 0.0  # measured decode-kernel time (with concurrent swaps)
    decode_nominal_ms: float = 0.0  # the same bytes at the calibrated solo rate
    # split by whether swap transfers were in flight when the decode launched
    busy_ms: float = 0.0
    busy_nominal_ms: float = 0.0
    quiet_ms: float = 0.0
    quiet_nominal_ms: float = 0.0
    iterations: int = 0
    idle_waits: int = 0
    wall_s: float = 0.0
    # per computing iteration: (decode kernel ms, KV bytes read, weight bytes
    # streamed, swaps in flight, layered).  Layered iterations count their
    # decode kernels only (per-layer events), not their plane-flag waits.
    samples: list = None
    solo_ms: tuple = (None, None)  # solo decode step before / after the run
    bytes_per_us: float = 0.0  # calibrated solo decode rate (nominal times)
    classified: str = "transfer pending at launch (host)"

    def __post_init__(self) -> None:
        if self.samples is None:
            self.samples = []

    @property
    def decode_stall(self) -> float:
        if self.decode_nominal_ms <= 0:
            return 0.0
        return self.decode_ms / self.decode_nominal_ms - 1.0

    @property
    def swap_induced_stall(self) -> Optional[float]:
        """Decode slowdown while swaps run, relative to decode with none in
        flight in the same run (same clocks, same power state)."""
        if self.busy_nominal_ms <= 0 or self.quiet_ms <= 0 or self.quiet_nominal_ms <= 0:
            return None
        return (self.busy_ms / self.busy_nominal_ms) / (self.quiet_ms / self.quiet_nominal_ms) - 1

    def classify_by_overlap(self, transfers: list) -> None:
        """Re-label every decode sample by what actually ran beside it on the
        device: busy if transfers overlapped >= half of its kernel interval,
        quiet if none did; partial overlaps are dropped.  (The host-side flag
        — "a transfer was pending at launch" — also marks decode that waited
        for a transfer on the device and then ran alone.)  Recomputes the
        busy / quiet sums behind swap_induced_stall."""
        merged: list = []
        for a, b in sorted(transfers):
            if merged and a <= merged[-1][1]:
                merged[-1][1] = max(merged[-1][1], b)
            else:
                merged.append([a, b])
        starts = np.asarray([m[0] for m in merged])
        out = []
        self.busy_ms = self.busy_nominal_ms = self.quiet_ms = self.quiet_nominal_ms = 0.0
        for smp in self.samples:
            ms, kv, w, _, layered, t0, t1 = smp
            i = int(np.searchsorted(starts, t1)) if merged else 0
            ov = 0.0
            for a, b in merged[max(0, i - 64):i]:
                ov += max(0.0, min(b, t1) - max(a, t0))
            frac = ov / (t1 - t0) if t1 > t0 else 0.0
            if 0.0 < frac < 0.5:
                continue
            busy = frac >= 0.5
            out.append((ms, kv, w, busy, layered, t0, t1))
            nominal = (kv + w) / self.bytes_per_us / 1e3 if self.bytes_per_us else 0.0
            if busy:
                self.busy_ms += ms
                self.busy_nominal_ms += nominal
            else:
                self.quiet_ms += ms
                self.quiet_nominal_ms += nominal
        self.samples = out
        self.classified = "device overlap"

    def stall_model(self, boot: int = 1000, seed: int = 0) -> Optional[dict]:
        """Swap-induced decode stall controlled for the batch mix, with a 95%
        bootstrap interval.

        A quiet iteration's decode time is fitted as a + b*KV bytes + c*weight
        bytes (least squares over every quiet iteration of the run: same
        clocks, same power state, same kernels).  The stall is the busy
        iterations' measured time over the fit's prediction for their own
        mix, minus one.  The interval resamples quiet and busy iterations
        (refitting each time), so a policy that costs nothing has an
        interval around 0 — the noise floor the point estimate alone hides."""
        if not self.samples:
            return None
        a = np.asarray([x[:4] for x in self.samples], dtype=np.float64)
        busy = a[:, 3] > 0
        q, b = a[~busy], a[busy]
        if len(q) < 20 or len(b) < 5:
            return None

        def design(x):
            return np.column_stack([np.ones(len(x)), x[:, 1] / 1e9, x[:, 2] / 1e9])

        def stall(qx, bx):
            coef, *_ = np.linalg.lstsq(design(qx), qx[:, 0], rcond=None)
            pred = design(bx) @ coef
            return float(bx[:, 0].sum() / max(1e-9, pred.sum()) - 1.0)

        point = stall(q, b)
        coef, *_ = np.linalg.lstsq(design(q), q[:, 0], rcond=None)
        resid = q[:, 0] - design(q) @ coef
        r2 = 1.0 - float(resid.var()) / max(1e-12, float(q[:, 0].var()))
        rng = np.random.default_rng(seed)
        draws = [stall(q[rng.integers(0, len(q), len(q))], b[rng.integers(0, len(b), len(b))])
                 for _ in range(boot)]
        lo, hi = np.percentile(draws, [2.5, 97.5])
        return {"stall": round(point, 4), "ci95": [round(float(lo), 4), round(float(hi), 4)],
                "busy_iterations": int(len(b)), "quiet_iterations": int(len(q)),
                "layered_iterations": int(sum(1 for x in self.samples if x[4])),
                "busy_means": self.classified,
                "quiet_fit_r2": round(r2, 4),
                "quiet_fit_resid_pct": round(float(np.abs(resid).mean() / q[:, 0].mean()) * 100, 2)}


class RankAgreement:
    """Control-plane agreement of a tensor-parallel group in live mode.

    Every TP rank runs the same engine over its own KV-head shard.  Replay
    decisions are deterministic, but live ones read the wall clock and poll
    CUDA events, which differ per rank.  So once per iteration the ranks agree
    on (a) the clock (max over ranks) and (b) which in-flight swaps have
    landed (a swap counts only once it landed on every rank): one all_reduce(MIN)
    over [-clock, landed_0, landed_1, ...].  A second, scalar one agrees on the
    iteration's end time.  Identical inputs -> identical decisions on every
    rank; the KV bytes never leave their rank (no collective on the data path).
    """

    def __init__(self, group=None, device=None) -> None:
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.device = (torch.device(device) if dist.get_backend(group) == "nccl"
                       else torch.device("cpu"))
        self.calls = 0
        self.seconds = 0.0

    def _min(self, values: list[int]) -> list[int]:
        t0 = time.perf_counter()
        t = torch.tensor(values, dtype=torch.int64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        out = t.tolist()
        self.calls += 1
        self.seconds += time.perf_counter() - t0
        return out

    def clock(self, local_us: int) -> int:
        return -self._min([-int(local_us)])[0]

    def landed(self, local_us: int, flags: list[bool]) -> tuple[int, list[bool]]:
        out = self._min([-int(local_us)] + [1 if f else 0 for f in flags])
        return -out[0], [bool(x) for x in out[1:]]


class LiveEngine(Engine):
    """Engine whose clock, swap completions and compute are real (one GPU;
    with `agreement`, one TP rank of a group that decides in lockstep)."""

    def __init__(self, config: EngineConfig, conversations, runtime, decode: DecodeEmulator,
                 time_scale: float = 1.0, agreement: Optional[RankAgreement] = None,
                 layered: bool = False, attend: bool = True,
                 per_layer_decode: bool = True, control_plane: Optional[str] = None,
                 graph_decode: bool = True) -> None:
        """layered: resumed requests join decode layer by layer (SURVEY §8f
        rank 2).  A swap-in at the head of the swap-in stream whose modeled
        completion falls inside this iteration joins the batch now, and so do
        sync-mode swap-ins (swap.py:113-135); decode layer l waits only for
        layer l of their KV (plane flags), instead of the reference's
        iteration-wise completion (engine.py:376-384).

        attend: each iteration also reads (and checks) the resident KV of
        every computing request, as attention would, inside the iteration's
        modeled time; any byte that differs from what its token wrote fails
        the run (runtime.KVIntegrityError).

        per_layer_decode: a decode step is one attention + one weight-stream
        kernel per layer (plane), as a model's layers are — in every
        iteration, so a layered join's per-layer kernels and an ordinary
        step's have the same launch structure and the swap-induced stall
        compares like with like.

        graph_decode: the step's kernels (and a layered step's plane-flag
        waits) are launched as one CUDA graph (DecodeGraph), as serving
        engines launch decode; False launches them one by one on the stream."""
        if runtime is None:
            raise ValueError("live mode needs a Runtime (real data plane)")
        super().__init__(config, conversations, runtime=runtime, control_plane=control_plane)
        self.decode = decode
        self.time_scale = time_scale
        self.agreement = agreement
        self.layered = layered and runtime.executor.layered_swap_in
        if layered and not self.layered:
            raise ValueError("layered admission needs Runtime(layered_swap_in=True) "
                             "with the kernel copy path")
        self._deferred: Optional[list] = None
        self.layered_joins = 0
        self.attend = attend and runtime.write_kv
        self.per_layer_decode = per_layer_decode
        planes = runtime.geometry.num_planes
        self.graph = (DecodeGraph(runtime.executor.compute.device, marks=2 * planes + 2)
                      if graph_decode and per_layer_decode and planes > 1 else None)
        self.live = LiveStats(bytes_per_us=decode.bytes_per_us)
        # per computing iteration: (duration_us, cpu_us, wait_ms, kernel_ms,
        #                           synced, conflict_waits, n_prefill, n_decode)
        self._trace: list[tuple] = []

    # -- clock ----------------------------------------------------------------

    def _now(self) -> int:
        return int((time.perf_counter() - self._t0) * 1e6) + self._skip

    # -- step 1 made real ------------------------------------------------------

    def _sync_clock(self) -> int:
        """This iteration's clock (agreed across the TP group, if any) and,
        with a group, the agreed landed-set of in-flight swaps."""
        now = self._now()
        if self.agreement is None:
            self._landed = None
            return now
        flags = [f.transfer is None or f.transfer.poll() for f in self.manager.in_flight]
        now, self._landed = self.agreement.landed(now, flags)
        return now

    def _end_clock(self) -> int:
        now = self._now()
        return now if self.agreement is None else self.agreement.clock(now)

    def _collect_live(self) -> bool:
        moved = False
        keep = []
        landed = self._landed
        for i, f in enumerate(self.manager.in_flight):
            done = (f.transfer is None or f.transfer.poll()) if landed is None else landed[i]
            if not done:
                keep.append(f)
                continue
            if f.direction == "out":
                done = {id(r) for r in f.op_records}
                self.manager.busy_extents = [r for r in self.manager.busy_extents
                                             if id(r) not in done]
            elif self._mark_running(f.request):
                moved = True
        self.manager.in_flight = keep
        return moved

    def _mark_running(self, req) -> bool:
        if self._deferred is None:
            return super()._mark_running(req)
        # Joining layer by layer: running now, bytes checked once decode has
        # waited for every layer (verification needs the whole KV).
        st = self.states.get(req)
        if st is None or st.phase != SWAPPING_IN:
            return False
        st.phase = RUNNING
        self.qs.move(req, "running")
        self._mark_turn(req, 2)
        self._deferred.append(req)
        return True

    def _join_layered(self, flights) -> list:
        """Move `flights` (pending swap-ins) into the running set now; returns
        their transfers, whose plane flags decode will wait on per layer."""
        deps = []
        self._deferred = self._deferred or []
        for f in flights:
            self.manager.in_flight.remove(f)
            if self._mark_running(f.request):
                deps.append(f.transfer)
        return deps

    def _wait_any(self, budget_us: int) -> None:
        """Nothing to compute: block on the earliest pending transfer (or a tick)."""
        pending = [f for f in self.manager.in_flight if f.transfer is not None]
        self.live.idle_waits += 1
        if pending:
            pending[0].transfer.event.synchronize()
        else:
            time.sleep(budget_us * 1e-6)

    # -- loop --------------------------------------------------------------------

    def warmup(self) -> None:
        """Touch every kernel / driver path the loop uses once before the clock
        starts (CUDA lazy loading would otherwise charge a first-use stall to
        whichever turn hits it): swap kernels of every op-table size class in
        both directions, op-flag waits, the KV-token kernel, the decode kernel."""
        ex = self.runtime.executor
        dp = self.runtime.dataplane
        n = min(dp.cache.num_blocks, dp.host.num_blocks)
        flags = torch.zeros(4096, dtype=torch.int32, device=dp.cache.device)
        for n_ops in (1, 33, 257):
            if n_ops > n:
                break
            ops = [(1, i, i) for i in range(n_ops)]
            for direction in ("out", "in"):
                s = ex.streams[direction]
                if ex.copy_impl == "kernel":
                    dp.swap_ops(direction, ops, flags.data_ptr(), 1, stream=s)
                    dp.wait_flag(ex.compute, flags.data_ptr(), 1)
                else:
                    from .swap import COPY_IMPLS
                    dp.baseline(direction, COPY_IMPLS.index(ex.copy_impl) - 1, ops, stream=s)
                s.synchronize()
        segs = np.asarray([[0, 0, 2 * self.spec.block_size_tokens, 0]], dtype=np.int64)
        dp.kv_tokens(0, segs, stream=ex.compute)
        self.decode.launch_us(ex.compute, 10.0)
        ex.compute.synchronize()
        torch.cuda.synchronize(dp.cache.device)

    def solo_decode_ms(self, steps: int = 20, us: float = 2000.0) -> float:
        """Median of `steps` solo decode steps of `us` modeled microseconds."""
        comp = self.runtime.executor.compute
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        evs[0].record(comp)
        for i in range(steps):
            self.decode.launch_us(comp, us)
            evs[i + 1].record(comp)
        comp.synchronize()
        return float(np.median([evs[i].elapsed_time(evs[i + 1]) for i in range(steps)]))

    def run(self) -> MetricsReport:
        self.warmup()
        before = self.solo_decode_ms()
        gc.collect()
        gc.freeze()  # long-lived engine state leaves the collector's young generations
        try:
            rep = self._run()
        finally:
            gc.unfreeze()
        self.runtime.synchronize()
        self.live.solo_ms = (before, self.solo_decode_ms())
        return rep

    def _run(self) -> MetricsReport:
        for conv in self.conversations:
            from .engine import RequestState
            self.states[conv.id] = RequestState(conv=conv)
            self._push_future(conv.arrival, conv.id)
        stalls = {"sync": 0, "conflict": 0, "yield": 0, "recompute": 0}
        windows: list[tuple[int, float]] = []
        win_tokens = win_time = win_batch = 0
        idle = 0
        first_arrival = self.conversations[0].arrival if self.conversations else 0
        ex = self.runtime.executor
        compute = ex.compute
        if self.agreement is not None:
            self.agreement.clock(0)  # the TP group starts its clocks together
        self._landed = None
        self._t0 = time.perf_counter()
        # Time origin on the device for this run's decode and transfer intervals.
        self._ref_ev = torch.cuda.Event(enable_timing=True)
        self._ref_ev.record(compute)
        self._skip = first_arrival
        wall0 = time.perf_counter()

        while True:
            self.clock = self._sync_clock()
            self._inject_arrivals()
            if not self._live_ids():
                if not self._future:
                    break
                nxt = self._future[0][0]
                if nxt > self.clock:
                    self._skip += nxt - self.clock
                continue
            self.iteration += 1
            start = self.clock
            t_iter = time.perf_counter()
            progress = self._collect_live()
            self._maybe_new_epoch()
            actions = self._schedule()
            grants: list[tuple[int, int]] = []
            self._outs_ready_at = self.clock
            for req in actions.swap_out:
                self._preempt(req)
                progress = True
            self._grow_decoders(grants)
            for req in actions.swap_in:
                progress = self._start_swap_in(req, grants) or progress
            for req in actions.admit:
                progress = self._admit(req, grants) or progress

            # Real conflicts: grants over blocks a D2H still reads.
            e_pre = torch.cuda.Event(enable_timing=True)
            e_pre.record(compute)  # GPU-side waits of this iteration start here
            conf_now = ex.compute_barrier(grants) if grants else 0
            grant_waits = list(ex.last_barrier) if grants else []
            self.conflict_count += conf_now

            pending = [f for f in self.manager.in_flight if f.direction == "in"]
            drain = max((elapsed(f.exec_done, self.clock) for f in pending), default=0)
            biggest = max((self._footprint_blocks(self.states[f.request]) for f in pending),
                          default=0)
            est = iteration_time(sum(self.states[r].pending_input for r in self.qs.running),
                                 len(self.qs.running), self.infer)
            decision = decide_mode(drain, biggest, est, self.cfg.sync_threshold_ratio,
                                   self.cfg.short_request_blocks,
                                   forced=None if self.mode.adaptive else "sync")
            layer_deps: list = []
            self._deferred = None
            if decision.mode == "sync" and pending:
                self.sync_stall_count += 1
                if self.layered:
                    layer_deps = self._join_layered(pending)
                else:
                    for f in pending:
                        ex.wait_transfer(f.transfer)
                        self.manager.in_flight.remove(f)
                        self._mark_running(f.request)
                progress = True
            elif self.layered and pending:
                # The head of the (FIFO) swap-in stream, and the ones right
                # behind it, join now if modeled to land within this iteration.
                ready = []
                for f in pending:
                    if elapsed(f.exec_done, self.clock) > est:
                        break
                    ready.append(f)
                if ready:
                    layer_deps = self._join_layered(ready)
                    progress = True
            self.layered_joins += len(layer_deps)
            if not self.mode.adaptive:
                for f in list(self.manager.in_flight):
                    ex.wait_transfer(f.transfer)

            prefillers, decoders, prefill_tokens, recompute, spans = self._assemble_batch()
            if not (prefillers or decoders):
                self._wait_any(self.infer.decode_base)
                end = self._end_clock()
                idle = idle + (0 if progress else 1)
                if idle >= LIVE_DEADLOCK_ITERATIONS:
                    from .engine import DeadlockError
                    raise DeadlockError(self._diagnostic_dump())
                self.clock = end
                continue
            nominal_us = iteration_time(prefill_tokens, len(decoders), self.infer) * self.time_scale
            t_cpu = time.perf_counter()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            # The step's modeled time is spent reading the batch's KV
            # (attention) and streaming weights for the rest.
            reads = spans if self.attend else []
            kv_bytes = sum(lo for _, lo, _ in reads) * self.runtime.token_bytes
            w_us = max(0.0, nominal_us - kv_bytes / self.decode.bytes_per_us)
            if layer_deps:
                # Decode layer by layer; layer l waits for layer l of every
                # joining request's KV.  This iteration's KV writes follow the
                # last layer, when every joining request's KV has landed.
                self.runtime.barrier(self, spans, skip=layer_deps)
                waits_seen = grant_waits + list(ex.last_barrier)
                swapping = True
                planes = self.runtime.geometry.num_planes
                kv_b = w_b = 0
                layer_evs = []
                segs = self.runtime.read_segments(self, reads) if reads else None
                g = self.graph
                if g is not None:
                    # one native call captures the step: per layer the plane-flag
                    # waits, the KV check and the weight stream, with marks
                    w_layer = self.decode.bytes_for_us(w_us / planes) if w_us > 0 else 0
                    g.capture_step(self.runtime.dataplane, self.decode, segs,
                                   self.runtime.kv_check_ptr(), w_layer,
                                   deps=[ex.plane_flags(dep) for dep in layer_deps], marks=True)
                    kv_b = self.runtime.account_reads(segs) if segs is not None else 0
                    w_b = w_layer * planes
                    layer_evs = [(2 * layer, 2 * layer + 1) for layer in range(planes)]
                else:  # kernel by kernel on the compute stream
                    e0.record(compute)
                    for layer in range(planes):
                        for dep in layer_deps:
                            ex.wait_plane(compute, dep, layer)
                        ea = torch.cuda.Event(enable_timing=True)
                        ea.record(compute)  # this layer's KV has landed: decode starts
                        if reads:
                            kv_b += self.runtime.attend(self, reads, planes=(layer, layer + 1),
                                                       segs=segs, stream=compute)
                        if w_us > 0:
                            w_b += self.decode.launch_us(compute, w_us / planes)
                        eb = torch.cuda.Event(enable_timing=True)
                        eb.record(compute)
                        layer_evs.append((ea, eb))
                if g is not None:
                    e0.record(compute)
                    g.launch(compute)
                t_rt = time.perf_counter()  # host: barrier + decode capture / launches
                e1.record(compute)
                self.runtime.write(self, spans)
            else:
                self.runtime.compute(self, spans)
                waits_seen = grant_waits + list(ex.last_barrier)
                swapping = any(not r.poll() for r in ex.pending)
                layer_evs = None
                planes = self.runtime.geometry.num_planes
                if self.per_layer_decode and planes > 1:
                    kv_b = w_b = 0
                    segs = self.runtime.read_segments(self, reads) if reads else None
                    g = self.graph
                    if g is None:
                        e0.record(compute)
                        for layer in range(planes):
                            if reads:
                                kv_b += self.runtime.attend(self, reads,
                                                           planes=(layer, layer + 1),
                                                           segs=segs, stream=compute)
                            if w_us > 0:
                                w_b += self.decode.launch_us(compute, w_us / planes)
                    else:
                        w_layer = self.decode.bytes_for_us(w_us / planes) if w_us > 0 else 0
                        g.capture_step(self.runtime.dataplane, self.decode, segs,
                                       self.runtime.kv_check_ptr(), w_layer)
                        kv_b = self.runtime.account_reads(segs) if segs is not None else 0
                        w_b = w_layer * planes
                        # the step starts at the graph launch: the host's
                        # capture time is not decode time
                        e0.record(compute)
                        g.launch(compute)
                else:
                    e0.record(compute)
                    kv_b = self.runtime.attend(self, reads) if reads else 0
                    w_b = self.decode.launch_us(compute, w_us) if w_us > 0 else 0
                t_rt = time.perf_counter()  # host: barrier + KV append + decode capture / launches
                e1.record(compute)
            compute.synchronize()
            if self._deferred:
                for req in self._deferred:  # now every layer has landed
                    self.runtime.swap_in_landed(self, req)
            self._deferred = None
            end = self._end_clock()
            kernel_ms = e0.elapsed_time(e1)
            self._trace.append((end - start, int((t_cpu - t_iter) * 1e6), e_pre.elapsed_time(e0),
                                kernel_ms, decision.mode == "sync" and bool(pending),
                                conf_now, len(prefillers),
                                len(decoders), waits_seen[:6], int((t_rt - t_cpu) * 1e6)))
            nominal_ms = (kv_b + w_b) / self.decode.bytes_per_us / 1e3
            # Layered steps include plane-flag waits: their decode sample is
            # the per-layer kernel time, waits excluded.
            if layer_evs is None:
                dec_ms = kernel_ms
            elif self.graph is not None:
                dec_ms = sum(self.graph.elapsed(a, b) for a, b in layer_evs)
            else:
                dec_ms = sum(a.elapsed_time(b) for a, b in layer_evs)
            self.live.samples.append((dec_ms, kv_b, w_b, swapping, layer_evs is not None,
                                      self._ref_ev.elapsed_time(e0),
                                      self._ref_ev.elapsed_time(e1)))
            self.live.decode_ms += dec_ms
            self.live.decode_nominal_ms += nominal_ms
            if swapping:
                self.live.busy_ms += dec_ms
                self.live.busy_nominal_ms += nominal_ms
            else:
                self.live.quiet_ms += dec_ms
                self.live.quiet_nominal_ms += nominal_ms
            self.live.iterations += 1
            duration = end - start
            emitted = self._emit_tokens(prefillers, decoders, end)
            progress = progress or emitted > 0
            overhead = max(0, duration - int(kernel_ms * 1e3))
            stalls["sync"] += overhead  # everything that is not decode compute
            stalls["recompute"] += recompute * self.infer.prefill_per_token
            rec = IterationRecord(self.iteration, start, end, prefill_tokens, len(decoders),
                                  overhead, 0, 0, recompute * self.infer.prefill_per_token,
                                  emitted)
            self.records.append(rec)
            win_tokens += emitted
            win_time += duration
            win_batch = max(win_batch, len(prefillers) + len(decoders))
            if self.iteration % EFFICIENCY_INTERVAL_ITERS == 0 and win_time > 0:
                windows.append((win_batch, win_tokens * 1e6 / win_time))
                win_tokens = win_time = win_batch = 0
            self.clock = end
            for req in list(self.qs.running):
                st = self.states[req]
                if st.remaining_output == 0 and st.pending_input == 0:
                    self._finish_turn(req)
                    progress = True
            idle = 0 if progress else idle + 1
            if idle >= LIVE_DEADLOCK_ITERATIONS:
                from .engine import DeadlockError
                raise DeadlockError(self._diagnostic_dump())

        self.runtime.synchronize()
        self.live.wall_s = time.perf_counter() - wall0
        ex = self.runtime.executor
        if ex.timing:
            self.live.classify_by_overlap(
                [(self._ref_ev.elapsed_time(r.start_event), self._ref_ev.elapsed_time(r.event))
                 for r in ex.history if r.start_event is not None and r.nbytes])
        if self.attend:
            bad = self.runtime.kv_errors()
            if bad:
                from .runtime import KVIntegrityError
                raise KVIntegrityError(f"{bad} KV words read by decode differ from what their "
                                       f"tokens wrote")
        return self._report(stalls, self._efficiencies(windows), first_arrival)

    def spike_breakdown(self, q: float = 0.99) -> dict:
        """Where the slowest (>= q quantile) iterations spend their time."""
        if not self._trace:
            return {}
        durs = sorted(t[0] for t in self._trace)
        cut = durs[min(len(durs) - 1, int(q * len(durs)))]
        slow = [t for t in self._trace if t[0] >= cut]
        n = len(slow)
        return {
            "quantile": q, "threshold_ms": cut / 1e3, "iterations": n,
            "mean_ms": sum(t[0] for t in slow) / n / 1e3,
            "mean_cpu_ms": sum(t[1] for t in slow) / n / 1e3,
            "mean_gpu_wait_ms": sum(t[2] for t in slow) / n,
            "mean_runtime_host_ms": sum(t[9] for t in slow) / n / 1e3,
            "mean_decode_kernel_ms": sum(t[3] for t in slow) / n,
            "frac_with_sync_swap_in": sum(1 for t in slow if t[4]) / n,
            "frac_with_conflict_wait": sum(1 for t in slow if t[5]) / n,
            "mean_prefill_requests": sum(t[6] for t in slow) / n,
            "overall_mean_ms": sum(durs) / len(durs) / 1e3,
            "overall_mean_cpu_ms": sum(t[1] for t in self._trace) / len(self._trace) / 1e3,
        }

    def iteration_anatomy(self) -> dict:
        """Where a computing iteration's wall time goes, on average (ms): host
        scheduling; the runtime's host-side launches (decode step capture +
        graph update + KV append); on the device, the interval from the
        iteration's first GPU-side wait to the decode step's start (host
        launch latency or conflict / sync-swap-in waits, whichever is longer)
        and the decode step itself.  TBT is one iteration per token."""
        if not self._trace:
            return {}
        n = len(self._trace)
        mean = lambda i, scale: round(sum(t[i] for t in self._trace) / n * scale, 4)  # noqa: E731
        return {"iterations": n, "mean_ms": mean(0, 1e-3), "schedule_ms": mean(1, 1e-3),
                "launch_ms": mean(9, 1e-3), "pre_decode_device_ms": mean(2, 1.0),
                "decode_ms": mean(3, 1.0)}

    def latency_summary(self) -> dict:
        def pct(xs, q):
            return percentile(xs, q) / 1e3 if xs else None
        return {
            "ttft_p50_ms": pct(self.ttft_samples, 0.50),
            "ttft_p95_ms": pct(self.ttft_samples, 0.95),
            "ttft_p99_ms": pct(self.ttft_samples, 0.99),
            "tbt_p50_ms": pct(self.tbt_samples, 0.50),
            "tbt_p99_ms": pct(self.tbt_samples, 0.99),
            "tbt_p999_ms": pct(self.tbt_samples, 0.999),
            "decode_stall_frac": round(self.live.decode_stall, 4),
            "swap_induced_decode_stall": (None if self.live.swap_induced_stall is None
                                          else round(self.live.swap_induced_stall, 4)),
            "decode_time_with_swaps_frac": round(
                self.live.busy_ms / max(1e-9, self.live.decode_ms), 4),
            "stall_model": self.live.stall_model(),
            "solo_decode_ms": [None if x is None else round(x, 4) for x in self.live.solo_ms],
            "solo_decode_drift": (None if None in self.live.solo_ms else
                                  round(self.live.solo_ms[1] / self.live.solo_ms[0] - 1, 4)),
            "iterations": self.live.iterations,
            "idle_waits": self.live.idle_waits,
            "layered_joins": self.layered_joins,
            "kv_read_gib": round(self.runtime.kv_bytes_read / 2**30, 2),
            "wall_s": round(self.live.wall_s, 2),
            "slow_iterations": self.spike_breakdown(),
            "tp_agreement": None if self.agreement is None else {
                "ranks": self.agreement.world, "calls": self.agreement.calls,
                "mean_us": round(self.agreement.seconds / max(1, self.agreement.calls) * 1e6, 1)},
        }
