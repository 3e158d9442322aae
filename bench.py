"""KV-swap benchmark (BASELINE.json metric: KV swap GB/s vs PCIe peak per GPU;
P99 TTFT/TBT on the multi-turn preemption trace).

Workload (N=1, BASELINE config 2 "block-group vs fragmented allocation
sweep", LLaMA-3-8B KV shape, 1 B200): one step = the swap-out of a
4096-block plan (8 GiB: 4096 x 2 MiB all-layer blocks, runs of --group blocks
at random non-overlapping positions on both sides, logical order shuffled)
from HBM into mapped pinned host memory, then the swap-in of the same bytes
into a different random table — each plan ONE libkvswap kernel launch.
Inputs (8 GiB per direction) exceed the 126 MB L2: no flush needed.

  value  = all ranks' swapped bytes / max-over-ranks device time (GB/s),
           KV already resident in HBM / host pool when timing starts.
  e2e    = the same bytes through the public API: CpuStore.plan_swap_out /
           plan_swap_in (control plane) -> SwapManager.dispatch -> kvs_swap,
           64 requests of 64 blocks, wall clock incl. planning + sync; the
           round trip's bytes are verified after the timed steps.
  --impl reference: the CPU path on the host cores, same plans, same sizes:
           the oracle's C restatement moves the bytes (the reference kvswitch
           is a simulator that moves none), and the reference's
           own control plane (baseline/_ref) is timed per call; rank 0 only.

Multi-GPU: one process per GPU; each rank swaps its own KV shard over its own
PCIe link — no collective on the data path ("scaling": "weak").
`python bench.py --gpus N` without torchrun relaunches itself under
torch.distributed.run with N ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "KV swap GB/s vs PCIe peak per GPU; P99 TTFT/TBT on multi-turn preemption trace"
PCIE_GEN5_X16_GBS = 63.0  # 64 GT/s raw per direction after 128b/130b
PLAN_BLOCKS = 4096
POOL_BLOCKS = 8192
HOST_POOL_BLOCKS = 5120  # 10 GiB pinned per rank (x8 ranks on one host)
SWEEP_GROUPS = (1, 2, 4, 8, 16, 32, 64, 128, 256)


def pools(plan_blocks: int) -> tuple[int, int]:
    """(GPU pool, host pool) blocks for a plan size: 8192 / 5120 at config 2's
    4096-block plans (smaller plans, used only by tests, scale them down)."""
    return (POOL_BLOCKS * plan_blocks // PLAN_BLOCKS,
            HOST_POOL_BLOCKS * plan_blocks // PLAN_BLOCKS)

# Live traces (BASELINE config 3): LLaMA-3-8B KV, 512 x 2 MiB GPU blocks.
# "stress" is the saturated 64-conversation variant; "default" is the
# reference's default workload size (workload.py:44-53: 200 conversations,
# think 10 s) at 2 req/s.  Both replay-pinned (tests/golden/engine.json
# vtc_config3_bench / vtc_config3_default / llama8b-style markov cases).
TRACES = {
    "stress_vtc": {"convs": 64, "rate": 4.0, "think": 2.0, "cpu": 4096, "pattern": "vtc"},
    "stress_markov": {"convs": 64, "rate": 4.0, "think": 2.0, "cpu": 4096, "pattern": "markov"},
    "default_vtc": {"convs": 200, "rate": 2.0, "think": 10.0, "cpu": 8192, "pattern": "vtc"},
}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--group", type=int, default=16)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--plan-blocks", type=int, default=PLAN_BLOCKS,
                    help="blocks per plan (default = config 2's 4096; smaller only for tests)")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-trace", action="store_true")
    ap.add_argument("--traces", default=",".join(TRACES),
                    help=f"comma list of live traces to run, from {sorted(TRACES)}")
    ap.add_argument("--trace-convs", type=int, default=0,
                    help="override every trace's conversation count (tests)")
    ap.add_argument("--no-layered", action="store_true",
                    help="trace: resumed requests join only once all their KV landed")
    ap.add_argument("--sm-partition", type=int, default=8,
                    help="serving + trace: swap kernels on their own N-SM green context, "
                         "decode on the rest (0 = share all SMs)")
    ap.add_argument("--e2e-policy", default="throughput_staged",
                    help="StreamExecutor duplex policy of the headline e2e leg")
    ap.add_argument("--serving-policy", default="serving",
                    help="StreamExecutor duplex policy of the live traces' FastSwitch arm")
    ap.add_argument("--control-plane", default="native", choices=["native", "python"],
                    help="e2e legs and live traces: the C++ control plane (native_ctrl) or "
                         "the Python one (same decisions)")
    ap.add_argument("--stream-decode", action="store_true",
                    help="live traces / serving: launch decode kernels one by one instead "
                         "of as one CUDA graph per step")
    return ap.parse_args(argv)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_if_needed(args) -> None:
    """`--gpus N` without a launcher: become N ranks under torch.distributed.run
    (127.0.0.1 rendezvous).  Under a launcher, WORLD_SIZE must equal --gpus."""
    if "WORLD_SIZE" not in os.environ:
        if args.gpus > 1:
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                   f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                   "--master-port", str(_free_port()), str(Path(__file__).resolve()),
                   *sys.argv[1:]]
            raise SystemExit(subprocess.call(cmd))
        return
    _, world, _ = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started "
                         f"WORLD_SIZE={world} ranks")


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cpu_info(threads: int) -> dict:
    """Where the CPU baseline ran: cores, model, NUMA nodes and the node of
    the calling thread (its buffers are first-touched there)."""
    node = None
    try:
        cpu = os.sched_getcpu()
        for d in Path(f"/sys/devices/system/cpu/cpu{cpu}").glob("node*"):
            node = int(d.name[4:])
    except (OSError, AttributeError, ValueError):
        pass
    try:
        nodes = len(list(Path("/sys/devices/system/node").glob("node[0-9]*"))) or 1
    except OSError:
        nodes = 1
    if node is None and nodes == 1:
        node = 0
    return {"cores": threads, "cpu_count": os.cpu_count(), "cpu_model": cpu_model(),
            "numa_node": node, "numa_nodes": nodes}


# --------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int) -> None:
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._drain, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _drain(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[2:]):
                if flag.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------- plans

def make_plans(group: int, seed: int, plan_blocks: int = PLAN_BLOCKS, runs=None, pair=None):
    """(out_ops, in_ops): the swap-out of `plan_blocks` in runs of `group`, and
    the swap-in of exactly those host blocks into another random table.
    `runs` / `pair` default to paper_2411_18424_b200.synthetic; the reference
    arm passes the oracle's (identical, tests/test_oracle.py) generators."""
    if runs is None:
        from paper_2411_18424_b200.synthetic import pair_tables, random_runs
        runs, pair = random_runs, pair_tables
    rng = np.random.default_rng(seed)
    gpu_pool, host_pool = pools(plan_blocks)
    out_ops = runs(rng, plan_blocks, group, gpu_pool, host_pool)
    in_ops = runs(rng, plan_blocks, group, gpu_pool, host_pool)
    host_blocks = np.concatenate([np.arange(c, c + b) for b, g, c in out_ops])
    gpu_blocks = np.concatenate([np.arange(g, g + b) for b, g, c in in_ops])
    in_ops = pair(gpu_blocks, host_blocks)
    return out_ops.astype(np.int32), in_ops.astype(np.int32)


# ------------------------------------------------------------- CPU baselines

class _Timed:
    """Wrap a bound method; accumulate per-call wall time."""

    def __init__(self, fn):
        self.fn, self.calls, self.seconds = fn, 0, 0.0

    def __call__(self, *a, **kw):
        t = time.perf_counter()
        try:
            return self.fn(*a, **kw)
        finally:
            self.seconds += time.perf_counter() - t
            self.calls += 1

    def us(self):
        return round(self.seconds / self.calls * 1e6, 2) if self.calls else None


def control_plane_cost(which: str) -> dict:
    """Per-call cost of the control plane on the bench's stress trace
    (replay, Markov priorities — the pattern the reference itself accepts):
    plan_swap_out (cpu_store.py:209), plan_swap_in (cpu_store.py:289),
    BlockGroupPool.allocate (alloc.py:218), SwapManager.dispatch
    (swap.py:181) and engine µs per iteration (engine.py:351).

    which="reference": the unmodified reference, installed offline into
    baseline/_ref; if absent there, says so.  which="ours": this package's
    Python control plane; which="native": its C++ control plane
    (native_ctrl.py, libkvctrl)."""
    t = TRACES["stress_markov"]
    doc = {"ablation": "full", "block": {"bytes_per_block": 2097152},
           "gpu_pool": {"total_blocks": 512}, "cpu_pool": {"total_blocks": t["cpu"]},
           "workload": {"num_conversations": t["convs"], "arrival_rate_per_s": t["rate"],
                        "think_time_mean_s": t["think"]},
           "trace": {"pattern": "markov", "frequency": 0.04}}
    if which == "reference":
        ref = ROOT / "baseline" / "_ref"
        if not (ref / "kvswitch").is_dir():
            return {"impl": "reference", "unavailable": "baseline/_ref not installed"}
        if str(ref) not in sys.path:
            sys.path.insert(0, str(ref))
        import kvswitch
        from kvswitch import config as C
        from kvswitch.engine import Engine as E
        s = C.build(doc)
        eng = E(s.engine, kvswitch.generate(s.workload))
        label = f"reference kvswitch {getattr(kvswitch, '__version__', '0.1.0')} (baseline/_ref)"
    else:
        from paper_2411_18424_b200 import config as mconfig
        from paper_2411_18424_b200.engine import Engine as E
        from paper_2411_18424_b200.workload import generate
        cfg, wl, _ = mconfig.build(doc)
        cp = "native" if which == "native" else "python"
        eng = E(cfg, generate(wl), control_plane=cp)
        label = ("paper_2411_18424_b200 (this package, replay mode, "
                 + ("native C++ control plane)" if cp == "native" else "Python control plane)"))
    hooks = {"plan_swap_out": (eng.store, "plan_swap_out"),
             "plan_swap_in": (eng.store, "plan_swap_in"),
             "allocate": (eng.pool, "allocate"), "dispatch": (eng.manager, "dispatch")}
    timers = {}
    for name, (obj, attr) in hooks.items():
        timers[name] = _Timed(getattr(obj, attr))
        setattr(obj, attr, timers[name])
    t0 = time.perf_counter()
    rep = eng.run()
    el = time.perf_counter() - t0
    return {"impl": label, "workload": "bench stress trace (64 conversations, 4 req/s, "
                                       "think 2 s, 512 x 2 MiB blocks, markov f=0.04), replay",
            **{f"{k}_us": v.us() for k, v in timers.items()},
            **{f"{k}_calls": v.calls for k, v in timers.items()},
            "iter_us": round(el / max(1, rep.iterations) * 1e6, 2),
            "iterations": rep.iterations, "run_s": round(el, 2)}


def cpu_oracle_rate(geo, group: int, seconds: float, threads: int, plan_blocks: int):
    """The oracle's C restatement moving the bench's own plans (same seed,
    sizes and pools) between host buffers, on all host threads."""
    from oracle import c_oracle
    from oracle.bytes_oracle import random_runs, table_to_ops
    out_ops, in_ops = make_plans(group, 0, plan_blocks, random_runs, table_to_ops)
    gpu_pool, host_pool = pools(plan_blocks)
    planes = np.full((geo.num_planes, gpu_pool, geo.plane_chunk_bytes), 7, dtype=np.uint8)
    host = np.zeros((host_pool, geo.block_bytes), dtype=np.uint8)
    nbytes = plan_blocks * geo.block_bytes

    def step():
        c_oracle.apply_plan_arrays("out", planes, host, out_ops, nthreads=threads)
        c_oracle.apply_plan_arrays("in", planes, host, in_ops, nthreads=threads)

    step()  # first touch
    moved, reps = 0, 0
    t0 = time.perf_counter()
    while True:
        step()
        moved += 2 * nbytes
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return moved / el / 1e9, (f"{reps} x (swap-out + swap-in) of the bench's {plan_blocks}-block "
                              f"({nbytes >> 20} MiB) plans in runs of {group}, "
                              f"{gpu_pool}-block 'GPU' and {host_pool}-block host "
                              f"buffers, {el:.1f} s")


def run_reference(args, geo):
    rank, world, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU reference arm
    threads = os.cpu_count() or 1
    from oracle import c_oracle
    from oracle.bytes_oracle import random_runs, table_to_ops
    out_ops, in_ops = make_plans(args.group, 0, args.plan_blocks, random_runs, table_to_ops)
    gpu_pool, host_pool = pools(args.plan_blocks)
    planes = np.full((geo.num_planes, gpu_pool, geo.plane_chunk_bytes), 7, dtype=np.uint8)
    host = np.zeros((host_pool, geo.block_bytes), dtype=np.uint8)

    def step():
        c_oracle.apply_plan_arrays("out", planes, host, out_ops, nthreads=threads)
        c_oracle.apply_plan_arrays("in", planes, host, in_ops, nthreads=threads)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    nbytes = 2 * args.plan_blocks * geo.block_bytes * args.steps
    val = nbytes / el / 1e9
    sample = (f"per step: swap-out + swap-in of the bench's {args.plan_blocks}-block "
              f"({args.plan_blocks * geo.block_bytes >> 20} MiB) plans in runs of {args.group} "
              f"(same seed and pools as the GPU arm), host buffers, oracle C restatement, "
              f"{threads} pthreads")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(el / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload_config(args, geo),
        "cpu_baseline": {"value": round(val, 3), "unit": "GB/s", "kind": "port",
                         "sample": sample, **host_cpu_info(threads),
                         "control_plane": control_plane_cost("reference")},
        "e2e": {"value": round(val, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def workload_config(args, geo) -> dict:
    nb = args.plan_blocks * geo.block_bytes
    return {"workload": f"config2 block-group swap: {args.plan_blocks}-block plans "
                        f"({nb / 2**30:g} GiB) out then in, runs of {args.group}, "
                        f"{geo.name} KV shape",
            "model_kv": geo.name, "block_bytes": geo.block_bytes,
            "plan_blocks": args.plan_blocks, "group_blocks": args.group,
            "gpu_pool_blocks": pools(args.plan_blocks)[0],
            "host_pool_blocks": pools(args.plan_blocks)[1],
            "l2": f"inputs {nb / 2**30:g} GiB/direction > 126 MB L2, no flush",
            "parallelism": f"replicas{args.gpus} (per-rank KV shard, own PCIe link)"}


# ------------------------------------------------------------------ our arm

def run_ours(args, geo):
    import torch
    import torch.distributed as dist

    from paper_2411_18424_b200.dataplane import (HostKVPool, PagedKVCache, SwapDataPlane,
                                                 host_link_info, numa_nodes, pcie_switch_groups)

    rank, world, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device")
    # KVS_BENCH_BACKEND=gloo lets N ranks share fewer GPUs (a code-path check
    # of the N>1 bench on a 1-GPU box; its numbers are not a scaling result).
    backend = os.environ.get("KVS_BENCH_BACKEND", "nccl")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            try:
                dist.init_process_group("nccl", device_id=dev)
            except Exception as exc:  # control-plane agreement works over gloo too
                print(f"bench: NCCL init failed ({exc}); using gloo", file=sys.stderr)
                backend = "gloo"
                dist.init_process_group("gloo")
        else:
            dist.init_process_group(backend)

    gpu_pool, host_pool = pools(args.plan_blocks)
    cache = PagedKVCache(geo, gpu_pool, device=dev)
    host = HostKVPool(host_pool, geo.block_bytes, numa_node=None, device=dev)
    host_numa = host.numa_node
    numa_per_rank, links = [host_numa], [host_link_info(dev)]
    if world > 1:  # where each rank's swap space lives, and which host link it uses
        numa_per_rank = [None] * world
        dist.all_gather_object(numa_per_rank, host_numa)
        links = [None] * world
        dist.all_gather_object(links, host_link_info(dev))
    dp = SwapDataPlane(cache, host, ctas={"out": args.ctas, "in": args.ctas})
    cache.planes.view(torch.int32).random_()
    out_ops, in_ops = make_plans(args.group, seed=rank, plan_blocks=args.plan_blocks)
    nbytes_dir = args.plan_blocks * geo.block_bytes
    s = torch.cuda.Stream(device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-timed steps (KV resident in HBM / host pool) ----
    def step(evs=None):
        if evs is not None:
            evs[0].record(s)
        dp.swap("out", out_ops, stream=s)
        if evs is not None:
            evs[1].record(s)
        dp.swap("in", in_ops, stream=s)
        if evs is not None:
            evs[2].record(s)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = dp.launches
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(s)
        for k in range(args.steps):
            step(evs[k])
        t_end.record(s)
        torch.cuda.synchronize()
    barrier()
    gpu_launches = dp.launches - launches0
    sec = t_start.elapsed_time(t_end) * 1e-3
    out_ms = [e[0].elapsed_time(e[1]) for e in evs]
    in_ms = [e[1].elapsed_time(e[2]) for e in evs]
    sec_max = max_over_ranks(sec)
    value = world * 2 * nbytes_dir * args.steps / sec_max / 1e9
    out_gbs = nbytes_dir / (statistics.mean(out_ms) * 1e-3) / 1e9
    in_gbs = nbytes_dir / (statistics.mean(in_ms) * 1e-3) / 1e9

    # ---- the same steps on the staged copy-engine path (whole host runs on
    #      the copy engines through an HBM ring + gather / scatter kernels) ----
    def step_staged(evs):
        evs[0].record(s)
        dp.baseline("out", 2, out_ops, stream=s)
        evs[1].record(s)
        dp.baseline("in", 2, in_ops, stream=s)
        evs[2].record(s)

    sev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)]
           for _ in range(args.warmup + args.steps)]
    for k in range(args.warmup + args.steps):
        step_staged(sev[k])
    torch.cuda.synchronize()
    sev = sev[args.warmup:]
    st_out = [e[0].elapsed_time(e[1]) for e in sev]
    st_in = [e[1].elapsed_time(e[2]) for e in sev]
    staged = {
        "engine": "copy engines, one copy per host run (<= 128 MiB slot) + kvs_stage_kernel "
                  "gather / scatter (HBM ring, 4 slots)",
        "per_direction_gbs": {"out": round(nbytes_dir / (statistics.mean(st_out) * 1e-3) / 1e9, 3),
                              "in": round(nbytes_dir / (statistics.mean(st_in) * 1e-3) / 1e9, 3)},
        "gbs": round(2 * nbytes_dir * len(sev) / ((sum(st_out) + sum(st_in)) * 1e-3) / 1e9, 3),
        "frac": None,
    }
    staged["frac"] = {d: round(v / PCIE_GEN5_X16_GBS, 4)
                      for d, v in staged["per_direction_gbs"].items()}

    # ---- e2e: public API (control plane + dispatch) with host round trip ----
    e2e = run_e2e(args, geo, dp, dev, barrier, max_over_ranks, world, args.e2e_policy)
    # the same leg with the kernel carrying both directions (TMA bulk), and
    # under the serving policy (LSU, op flags, pace + budget)
    e2e_kernel = run_e2e(args, geo, dp, dev, barrier, max_over_ranks, world, "throughput")
    e2e_serving = run_e2e(args, geo, dp, dev, barrier, max_over_ranks, world,
                          args.serving_policy)
    dp.set_launch("out", args.ctas, 0)
    dp.set_launch("in", args.ctas, 0)

    # ---- copy-engine peak, all ranks at once (host-link / root-port probe) ----
    barrier()
    ce = ce_peak(dev, host, cache)
    ce_all = [ce]
    if world > 1:
        ce_all = [None] * world
        dist.all_gather_object(ce_all, ce)

    # ---- group-size sweep (config 2): kernel paths vs copy-engine comparators ----
    sweep = None
    if rank == 0 and not args.no_sweep:
        sweep = group_sweep(dp, s, torch.cuda.Stream(device=dev))

    # ---- the SM partition is an optimisation: fall back to shared SMs if the
    #      driver cannot create green contexts on this box ----
    if args.sm_partition:
        from paper_2411_18424_b200.swap import partition_streams
        try:
            partition_streams(dev, args.sm_partition)
        except (RuntimeError, ValueError) as exc:
            print(f"bench: SM partition unavailable ({exc}); sharing all SMs", file=sys.stderr)
            args.sm_partition = 0

    # ---- serving configuration: swaps under a concurrent decode load ----
    serving = None
    if rank == 0:
        g = not args.stream_decode
        serving = {"full_rate_shared_sms": serving_interference(dp, dev, s, 0, "latency",
                                                                  graph=g)}
        if args.sm_partition:
            part = f"swap_on_{args.sm_partition}_sms"
            serving[args.serving_policy + "_" + part] = serving_interference(
                dp, dev, s, args.sm_partition, args.serving_policy, graph=g)
            # the same at the link rate (swap-in unpaced)
            serving["serving_link_" + part] = serving_interference(
                dp, dev, s, args.sm_partition, "serving_link", graph=g)
            # the same policy with the decode kernels launched one by one: their
            # command fetches share the PCIe link with the swap-in
            serving[args.serving_policy + "_stream_decode_" + part] = serving_interference(
                dp, dev, s, args.sm_partition, args.serving_policy, graph=False)
            serving["serving_paced_stream_decode_" + part] = serving_interference(
                dp, dev, s, args.sm_partition, "serving_paced", graph=False)

    # ---- live multi-turn preemption traces: P99 TTFT / TBT (metric part 2) ----
    trace = None
    if not args.no_trace:
        host.close()  # free the 10 GiB pinned pool before the trace's own pools
        trace = {}
        for name in [t for t in args.traces.split(",") if t]:
            trace[name] = run_trace(args, geo, dev, name)

    root_ports = {lk["root_port"] for lk in links if lk.get("root_port")}
    # GPUs behind one PCIe switch share its uplink (nvidia-smi topo -mp, PCIe only)
    switches = pcie_switch_groups(world) if world > 1 and rank == 0 else {}
    # Ranks behind one root port (or switch) share its link: the aggregate
    # roofline is the smaller of one link per rank and one per shared port.
    if root_ports:
        link_cap = PCIE_GEN5_X16_GBS * min(world, len(root_ports))
    elif switches.get("groups"):
        link_cap = PCIE_GEN5_X16_GBS * len(switches["groups"])
    else:
        link_cap = PCIE_GEN5_X16_GBS * world

    barrier()
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        # after every rank's GPU work (the other ranks wait at the barrier below)
        threads = os.cpu_count() or 1
        rate, sample = cpu_oracle_rate(geo, args.group, 10.0, threads, args.plan_blocks)
        cpu = {"value": round(rate, 3), "unit": "GB/s", "kind": "port", "sample": sample,
               **host_cpu_info(threads),
               "control_plane": control_plane_cost("reference"),
               "control_plane_ours": control_plane_cost("ours"),
               "control_plane_native": control_plane_cost("native")}
    if rank == 0:
        dominant, dom_ms = ("in", in_ms) if sum(in_ms) >= sum(out_ms) else ("out", out_ms)
        achieved = nbytes_dir / (statistics.mean(dom_ms) * 1e-3) / 1e9
        traffic = ncu_traffic(dominant)
        config = workload_config(args, geo)  # identical to the reference arm's
        ce_sum = {d: round(sum(c[d] for c in ce_all), 3) for d in ("out", "in")}
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(sec_max / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (random KV bytes, seeded random block tables)",
            "backend": backend if world > 1 else None,
            "config": config,
            "host_pool": {"blocks": host_pool, "numa_node": host_numa,
                          "numa_node_per_rank": numa_per_rank, "numa_nodes": numa_nodes()},
            "per_direction_gbs": {"out": round(out_gbs, 3), "in": round(in_gbs, 3)},
            # every timed step's per-direction time: a dip here is the box, not a mean
            "step_ms": {"out": [round(x, 2) for x in out_ms], "in": [round(x, 2) for x in in_ms]},
            "staged": staged,
            "roofline": {"bound": "pcie", "achieved": round(achieved, 3),
                         "peak": PCIE_GEN5_X16_GBS, "unit": "GB/s",
                         "frac": round(achieved / PCIE_GEN5_X16_GBS, 4), "traffic": traffic,
                         "aggregate": {"gbs": round(value, 3), "links": world,
                                       "frac": round(value / (world * PCIE_GEN5_X16_GBS), 4),
                                       "root_ports": len(root_ports) or None,
                                       "topology_cap_gbs": link_cap,
                                       "pcie_switch_groups": switches.get("groups"),
                                       "pcie_matrix": switches.get("matrix"),
                                       "frac_of_topology": round(value / link_cap, 4),
                                       "ce_all_ranks_concurrent_gbs": ce_sum,
                                       "ce_per_rank_gbs": ce_all},
                         "host_links": links,
                         "kernel": f"kvs_swap_kernel<{dominant}>",
                         "peak_source": "PCIe Gen5 x16 per direction after 128b/130b "
                                        "(BASELINE.md §4; MEASURED_PEAKS.json has no PCIe entry)",
                         "ce_measured_gbs": ce,
                         "frac_of_ce": {d: round((out_gbs if d == "out" else in_gbs) / ce[d], 4)
                                        for d in ("out", "in")} if ce else None,
                         "hbm": {"achieved": round(achieved, 3),
                                 "peak": measured_hbm_peak(), "unit": "GB/s"},
                         "ncu": ncu_link_rates()},
            "e2e": e2e,
            "e2e_kernel_both_ways": e2e_kernel,
            "e2e_serving": e2e_serving,
            "gpu_launches": gpu_launches,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "sweep": sweep,
            "serving": serving,
            "trace": trace,
        }
        print(json.dumps(line), flush=True)
    barrier()
    host.close()
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, geo, dp, dev, barrier, max_over_ranks, world, policy):
    """The same bytes through CpuStore + SwapManager.dispatch (the drop-in
    API), then — untimed — the same round trip with the GPU blocks poisoned
    between swap-out and swap-in, compared with a snapshot: the leg's bytes
    are verified, not assumed."""
    import torch

    from paper_2411_18424_b200.costmodel import TransferParams
    from paper_2411_18424_b200.cpu_store import CpuStore
    from paper_2411_18424_b200.swap import DUPLEX_POLICIES, StreamExecutor, SwapManager
    from paper_2411_18424_b200.synthetic import random_runs

    ex = StreamExecutor(dp, duplex_policy=policy)
    path = DUPLEX_POLICIES[policy].get("path", "lsu")
    engines = {d: (f"kernel ({'TMA bulk' if path == 'bulk' else 'LSU'})"
                   if ex.engine[d] == "kernel" else f"copy engines ({ex.engine[d]})")
               for d in ("out", "in")}
    mgr = SwapManager(TransferParams(), bytes_per_block=geo.block_bytes, executor=ex)
    gpu_pool, host_pool = pools(args.plan_blocks)
    if args.control_plane == "native":  # the same API on the C++ control plane
        from paper_2411_18424_b200.native_ctrl import NativeCpuStore as CpuStore  # noqa: F811
    store = CpuStore(host_pool, reuse_enabled=True)
    n_req = 64
    per = max(1, args.plan_blocks // n_req)
    rng = np.random.default_rng(7)
    runs = random_runs(rng, args.plan_blocks, args.group, gpu_pool, host_pool)
    tables, cursor = [], 0
    per_runs = max(1, per // args.group)
    for _ in range(n_req):
        tables.append([(int(g), int(b)) for b, g, _ in runs[cursor:cursor + per_runs]])
        cursor += per_runs
    foot = [sum(b for _, b in t) for t in tables]

    def step(poison=None):
        for r in range(n_req):
            mgr.dispatch(0, 0, store.plan_swap_out(r, foot[r], tables[r]))
        if poison is not None:
            ex.synchronize()
            poison()
        for r in range(n_req):
            mgr.dispatch(0, 0, store.plan_swap_in(r, tables[r]))
        ex.synchronize()
        for r in range(n_req):
            store.release(r)
        mgr.in_flight.clear()
        mgr.busy_extents.clear()

    for _ in range(max(1, args.warmup)):
        step()
    barrier()
    torch.cuda.synchronize()
    l0 = dp.launches  # every libkvswap kernel: swap kernels and staged gather / scatter
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = max_over_ranks(time.perf_counter() - t0)
    launches = dp.launches - l0

    blocks = torch.as_tensor(np.concatenate([np.arange(g, g + b) for t in tables for g, b in t]),
                             device=dev)
    planes = dp.cache.planes
    snap = planes.index_select(1, blocks)

    def poison():
        planes.index_fill_(1, blocks, 0xFF)
        torch.cuda.synchronize()  # the executor's streams do not order after torch's

    step(poison)
    verified = bool(torch.equal(planes.index_select(1, blocks), snap))
    del snap
    torch.cuda.empty_cache()
    if not verified:
        raise AssertionError(f"e2e ({policy}) round trip bytes differ after swap-in")
    moved = sum(foot) * geo.block_bytes
    for d in ("out", "in"):
        dp.set_path(d, "lsu")
        dp.set_pace(d, 0.0)
        dp.set_budget_share(d, 0.0)
    dp.set_budget(0.0)
    dp.set_budget_priority(None)
    return {"value": round(world * 2 * moved * args.steps / el / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": moved, "d2h_bytes_per_step": moved,
            "policy": policy, "engines": engines,
            "api": f"CpuStore.plan_swap_out/plan_swap_in -> SwapManager.dispatch -> "
                   f"StreamExecutor ({policy} policy) -> kvs_swap / kvs_memcpy_baseline "
                   f"(C ABI); wall clock incl. planning and sync",
            "control_plane": args.control_plane,
            "requests_per_step": n_req, "gpu_launches": launches,
            "bytes_verified": verified}


def run_trace(args, geo, dev, name):
    """Live-mode multi-turn preemption trace on this GPU (paper_2411_18424_b200.live):
    FastSwitch (block groups + reuse + adaptive async + layered admission, one
    kernel per plan) vs the vLLM-style baseline (per-block copies on the copy
    engines), on the same conversations and priorities."""
    import dataclasses

    from paper_2411_18424_b200 import config as mconfig
    from paper_2411_18424_b200.live import DecodeEmulator, LiveEngine, b200_transfer_params
    from paper_2411_18424_b200.runtime import Runtime
    from paper_2411_18424_b200.workload import generate

    t = dict(TRACES[name])
    if args.trace_convs:
        t["convs"] = args.trace_convs
    _, world, _ = dist_env()
    agreement = None
    if world > 1:
        # one TP group: every rank swaps its own KV-head shard, decisions in lockstep
        from paper_2411_18424_b200.live import RankAgreement
        geo = geo.with_tp(world)
        agreement = RankAgreement(device=dev)
    stream, ctas, sms = None, 0, None
    if args.sm_partition:
        from paper_2411_18424_b200.swap import partition_streams
        _, stream, sms = partition_streams(dev, args.sm_partition)
        ctas = 2 * sms[1]
    decode = DecodeEmulator(dev, weight_bytes=16 << 30, ctas=ctas, stream=stream)
    doc = {"block": {"bytes_per_block": geo.block_bytes}, "gpu_pool": {"total_blocks": 512},
           "cpu_pool": {"total_blocks": t["cpu"]},
           "workload": {"num_conversations": t["convs"], "arrival_rate_per_s": t["rate"],
                        "think_time_mean_s": t["think"]},
           "trace": {"pattern": t["pattern"], "frequency": 0.04}}
    out = {"workload": f"{t['convs']} conversations, {t['rate']:g} req/s, think "
                       f"{t['think']:g} s, 512 x {geo.block_bytes / 2**20:g} MiB GPU blocks "
                       f"per rank (TP{world}), {t['cpu']}-block host pool, {t['pattern']} "
                       f"priorities f=0.04, decode = {geo.num_planes} per-layer steps of "
                       f"KV reads of every resident token + {decode.bytes_per_us / 1e3:.0f} GB/s "
                       f"weight streaming per rank; FastSwitch swaps under the "
                       f"'{args.serving_policy}' policy",
           "pattern": t["pattern"], "tp": world, "sm_partition": sms,
           "control_plane": args.control_plane,
           "decode_launch": "stream" if args.stream_decode else "cuda_graph", "runs": {}}
    for run, mode, impl in (("fastswitch", "full", "kernel"),
                            ("vllm_like", "baseline", "ce_per_block")):
        cfg, wl, _ = mconfig.build({**doc, "ablation": mode})
        cfg = dataclasses.replace(cfg, transfer=b200_transfer_params())
        layered = impl == "kernel" and not args.no_layered
        rt = Runtime(geo, cfg.gpu_pool.total_blocks, cfg.cpu_pool_blocks, device=dev,
                     copy_impl=impl, timing=True, sm_partition=args.sm_partition,
                     layered_swap_in=layered,
                     duplex_policy=args.serving_policy if impl == "kernel" else "latency")
        eng = LiveEngine(cfg, generate(wl), rt, decode, agreement=agreement, layered=layered,
                         control_plane=args.control_plane, graph_decode=not args.stream_decode)
        eng.turn_trace = []
        rep = eng.run()
        lat = eng.latency_summary()
        anat = eng.ttft_anatomy()
        st = rt.stats()
        out["runs"][run] = {"ablation": mode, "copy_impl": impl,
                            **{k: lat[k] for k in ("ttft_p50_ms", "ttft_p95_ms", "ttft_p99_ms",
                                                   "tbt_p50_ms", "tbt_p99_ms", "tbt_p999_ms",
                                                   "decode_stall_frac",
                                                   "swap_induced_decode_stall", "stall_model",
                                                   "solo_decode_ms", "solo_decode_drift",
                                                   "wall_s")},
                            "ttft_tail_ms": {"turns": anat.get("turns"),
                                             **anat.get("tail_mean_ms", {})},
                            "layered_joins": lat["layered_joins"],
                            "kv_read_gib_verified": lat["kv_read_gib"],
                            "tokens": rep.total_tokens,
                            "swap_gib": {"out": round(st["bytes_out"] / 2**30, 2),
                                         "in": round(st["bytes_in"] / 2**30, 2)},
                            "swap_rates": rt.swap_rates(),
                            "iteration_anatomy": eng.iteration_anatomy(),
                            "kernel_launches": st["kernel_launches"]}
        rt.close()
    del decode
    torch_empty_cache()
    return out


def serving_interference(dp, dev, s, sm_partition: int = 0, policy: str = "latency",
                         layers: int = 32, graph: bool = True):
    """Swap-induced decode stall, measured: 2 ms HBM-streaming decode steps
    (each `layers` per-layer kernels, as the live engine runs them) on a
    high-priority stream while a 2 GiB swap runs, per direction and both at
    once, under a serving policy (swap.DUPLEX_POLICIES: paced kernels, shared
    budget, optional reserved share)."""
    import torch

    from paper_2411_18424_b200.live import DecodeEmulator
    from paper_2411_18424_b200.swap import DUPLEX_POLICIES
    from paper_2411_18424_b200.synthetic import random_runs

    if sm_partition:
        from paper_2411_18424_b200.swap import partition_streams
        (s, s2), comp, sms = partition_streams(dev, sm_partition)
        dec = DecodeEmulator(dev, weight_bytes=16 << 30, ctas=2 * sms[1], stream=comp)
    else:
        sms = None
        dec = DecodeEmulator(dev, weight_bytes=16 << 30)
        comp = torch.cuda.Stream(device=dev, priority=-1)
        s2 = torch.cuda.Stream(device=dev)
    rng = np.random.default_rng(5)
    gp, hp = dp.cache.num_blocks // 2, dp.host.num_blocks // 2
    n = min(1024, hp // 2)
    ops = random_runs(rng, n, 16, gp, hp).astype(np.int32)
    ops_in = ops.copy()
    ops_in[:, 1] += gp
    ops_in[:, 2] += hp
    nbytes = n * dp.geometry.block_bytes

    # the decode step as one CUDA graph, as the live engine and serving
    # engines launch it (DecodeGraph); graph=False: kernel by kernel
    g = None
    if graph:
        from paper_2411_18424_b200.live import DecodeGraph
        g = DecodeGraph(dev, marks=0)
        gs = g.begin()
        for _ in range(layers):
            dec.launch_us(gs, 2000.0 / layers)
        g.end()

    def steps(k):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(k + 1)]
        evs[0].record(comp)
        for i in range(k):
            if g is not None:
                g.launch(comp)
            else:
                for _ in range(layers):
                    dec.launch_us(comp, 2000.0 / layers)
            evs[i + 1].record(comp)
        return evs

    steps(3)
    torch.cuda.synchronize()
    ev = steps(20)
    torch.cuda.synchronize()
    solo = statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(20))
    pol = DUPLEX_POLICIES[policy]
    for d in ("out", "in"):
        c, t, pace = pol[d]
        dp.set_path(d, pol.get("path", "lsu"))
        dp.set_launch(d, c, t)
        dp.set_pace(d, pace)
        dp.set_budget_share(d, pol.get("share", {}).get(d, 0.0))
    dp.set_budget(pol["budget"])
    dp.set_budget_priority(pol.get("priority"))
    out = {"policy": policy, "sm_partition": sms, "decode_step_solo_ms": round(solo, 3),
           "decode_kernels_per_step": layers,
           "decode_launch": "cuda_graph" if g is not None else "stream", "runs": {}}
    for name, dirs in (("out", ("out",)), ("in", ("in",)), ("duplex", ("out", "in"))):
        torch.cuda.synchronize()
        t = {}
        for d in dirs:
            st = s if d == "out" else s2
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            dp.swap(d, ops if d == "out" else ops_in, stream=st)
            e1.record(st)
            t[d] = (e0, e1)
        ev = steps(40)
        torch.cuda.synchronize()
        end = max(t[d][0].elapsed_time(t[d][1]) for d in dirs)
        st_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(40)
                 if t[dirs[0]][0].elapsed_time(ev[i]) <= end]
        out["runs"][name] = {
            "swap_gbs": {d: round(nbytes / (t[d][0].elapsed_time(t[d][1]) * 1e-3) / 1e9, 2)
                         for d in dirs},
            "decode_steps": len(st_ms),
            "decode_slowdown": round(statistics.median(st_ms) / solo - 1, 4) if st_ms else None}
    for d in ("out", "in"):
        dp.set_path(d, "lsu")
        dp.set_launch(d, 0, 0)
        dp.set_pace(d, 0.0)
        dp.set_budget_share(d, 0.0)
    dp.set_budget(0.0)
    dp.set_budget_priority(None)
    if g is not None:
        g.close()
    del dec
    return out


def torch_empty_cache():
    import torch
    torch.cuda.empty_cache()


def ce_peak(dev, host, cache):
    """Large pinned cudaMemcpyAsync per direction (copy-engine reference point)."""
    import torch
    n = 1 << 30
    h = host.tensor.view(-1)[:n]
    d = cache.planes.view(-1)[:n]
    s = torch.cuda.Stream(device=dev)
    res = {}
    for name, fn in (("in", lambda: d.copy_(h, non_blocking=True)),
                     ("out", lambda: h.copy_(d, non_blocking=True))):
        with torch.cuda.stream(s):
            fn()
            s.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(3):
                fn()
            e1.record(s)
            s.synchronize()
        res[name] = round(3 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9, 3)
    return res


SWEEP_ENGINES = ("kernel_lsu", "kernel_bulk", "ce_per_block", "ce_per_run", "ce_staged")


def group_sweep(dp, s, s2):
    """Config 2: swap GB/s vs group size for every engine —
    K1/K2 LSU (v1) and TMA bulk (v2), K3 per-block (vLLM swap_blocks, the
    reference's split_single path, swap.py:170-179), K3 per-run (one 2D copy
    per run), staged (whole host runs on the copy engines through an HBM ring
    + a gather / scatter kernel) — per direction (a 4096-block plan) and
    both directions at once (2048-block plans each way on disjoint halves of
    the pools; combined GB/s over the union of both streams' lifetimes)."""
    import torch

    from paper_2411_18424_b200.synthetic import random_runs
    geo = dp.geometry
    gp, hp = dp.cache.num_blocks, dp.host.num_blocks
    plan = min(PLAN_BLOCKS, hp // 2)
    nbytes = plan * geo.block_bytes
    rng = np.random.default_rng(11)

    def launch(engine, d, ops, stream):
        if engine.startswith("kernel"):
            dp.set_path(d, "bulk" if engine == "kernel_bulk" else "lsu")
            dp.swap(d, ops, stream=stream)
        else:
            dp.baseline(d, ("ce_per_block", "ce_per_run", "ce_staged").index(engine), ops,
                        stream=stream)

    def timed(fn_by_stream):
        torch.cuda.synchronize()
        marks = []
        for st, fn in fn_by_stream:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            marks.append((e0, e1))
        torch.cuda.synchronize()
        ref = marks[0][0]
        lo = min(ref.elapsed_time(a) for a, _ in marks)
        hi = max(ref.elapsed_time(b) for _, b in marks)
        return (hi - lo) * 1e-3

    warm = random_runs(rng, min(256, plan), 16, gp, hp).astype(np.int32)
    for e in SWEEP_ENGINES:  # first use of every path outside the timed calls
        for d in ("out", "in"):
            launch(e, d, warm, s)
    torch.cuda.synchronize()
    rows = []
    for g in SWEEP_GROUPS:
        ops = random_runs(rng, plan, g, gp, hp).astype(np.int32)
        half = plan // 2
        h_out = random_runs(rng, half, g, gp // 2, hp // 2).astype(np.int32)
        h_in = random_runs(rng, half, g, gp // 2, hp // 2).astype(np.int32)
        h_in[:, 1] += gp // 2
        h_in[:, 2] += hp // 2
        row = {"group": g, "ops": int(len(ops))}
        for e in SWEEP_ENGINES:
            for d in ("out", "in"):
                sec = timed([(s, lambda: launch(e, d, ops, s))])
                row[f"{d}_{e}"] = round(nbytes / sec / 1e9, 2)
            sec = timed([(s, lambda: launch(e, "out", h_out, s)),
                         (s2, lambda: launch(e, "in", h_in, s2))])
            row[f"duplex_{e}"] = round(2 * half * geo.block_bytes / sec / 1e9, 2)
        rows.append(row)
    for d in ("out", "in"):
        dp.set_path(d, "lsu")
    return {"plan_blocks": plan, "block_bytes": geo.block_bytes, "engines": SWEEP_ENGINES,
            "unit": "GB/s", "rows": rows}


def measured_hbm_peak():
    try:
        return json.load(open(ROOT / "MEASURED_PEAKS.json"))["hbm_gbs"]
    except (OSError, KeyError, ValueError):
        return 6650.0  # B200_PROFILING.md fallback


def ncu_traffic(direction: str):
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    try:
        d = json.load(open(ROOT / "profiles" / "ncu_kernel_summary.json"))
        return d["kernels"][direction]["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def ncu_link_rates():
    """Host-link and HBM rates of both swap kernels from the committed ncu
    capture (profiles/ncu_kernel_summary.json): payload vs wire bytes."""
    try:
        d = json.load(open(ROOT / "profiles" / "ncu_kernel_summary.json"))
    except (OSError, ValueError):
        return None
    out = {"source": d.get("source")}
    for k, v in d.get("kernels", {}).items():
        out[k] = {"pcie_write_gbs": v.get("pcie_write_gbs"), "pcie_read_gbs": v.get("pcie_read_gbs"),
                  "dram_gbs": v.get("dram_gbs"), "duration_s": v.get("duration_s")}
    return out


def main():
    args = parse()
    relaunch_if_needed(args)
    from paper_2411_18424_b200.geometry import PRESETS
    geo = PRESETS[args.model]
    if args.impl == "reference":
        run_reference(args, geo)
    else:
        run_ours(args, geo)


if __name__ == "__main__":
    main()
