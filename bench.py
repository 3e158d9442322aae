"""KV-swap benchmark (BASELINE.json metric: KV swap GB/s vs PCIe peak per GPU).

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
           64 requests of 64 blocks, wall clock incl. planning + sync.
  --impl reference: the oracle's C restatement of the same plans on the
           host cores (the reference kvswitch is a simulator that moves no
           bytes), rank 0 only.

Multi-GPU: one process per GPU (torchrun); each rank swaps its own KV shard
over its own PCIe link — no collective on the data path ("scaling": "weak").
"""

from __future__ import annotations

import argparse
import json
import os
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--group", type=int, default=16)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--trace-convs", type=int, default=64)
    ap.add_argument("--no-trace", action="store_true")
    ap.add_argument("--trace-pattern", default="vtc", choices=["vtc", "markov", "random"],
                    help="trace priority pattern (config 3 names VTC; markov is the "
                         "reference's parity-pinned pattern)")
    ap.add_argument("--no-layered", action="store_true",
                    help="trace: resumed requests join only once all their KV landed")
    ap.add_argument("--sm-partition", type=int, default=8,
                    help="serving + trace: swap kernels on their own N-SM green context, "
                         "decode on the rest (0 = share all SMs)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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

def make_plans(group: int, seed: int):
    from paper_2411_18424_b200.synthetic import pair_tables, random_runs
    rng = np.random.default_rng(seed)
    out_ops = random_runs(rng, PLAN_BLOCKS, group, POOL_BLOCKS, HOST_POOL_BLOCKS)
    in_ops = random_runs(rng, PLAN_BLOCKS, group, POOL_BLOCKS, HOST_POOL_BLOCKS)
    # swap-in reads back exactly the host blocks swap-out wrote
    host_blocks = np.concatenate([np.arange(c, c + b) for b, g, c in out_ops])
    gpu_blocks = np.concatenate([np.arange(g, g + b) for b, g, c in in_ops])
    in_ops = pair_tables(gpu_blocks, host_blocks)
    return out_ops.astype(np.int32), in_ops.astype(np.int32)


# ------------------------------------------------------------- reference arm

def cpu_oracle_rate(geo, group: int, seconds: float, threads: int):
    """Oracle C restatement of the same plan shape on host memory (bounded sample)."""
    from oracle import c_oracle
    from oracle.bytes_oracle import random_runs
    sample_blocks = 512  # 1 GiB per direction at 2 MiB blocks
    pool = 1024
    rng = np.random.default_rng(1)
    planes = np.zeros((geo.num_planes, pool, geo.plane_chunk_bytes), dtype=np.uint8)
    host = np.zeros((pool, geo.block_bytes), dtype=np.uint8)
    planes[:] = 7
    ops = random_runs(rng, sample_blocks, min(group, sample_blocks), pool, pool)
    moved = 0
    t0 = time.perf_counter()
    reps = 0
    while True:
        c_oracle.apply_plan_arrays("out", planes, host, ops, nthreads=threads)
        c_oracle.apply_plan_arrays("in", planes, host, ops, nthreads=threads)
        moved += 2 * sample_blocks * geo.block_bytes
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return moved / el / 1e9, f"{reps} x (swap-out + swap-in) of a {sample_blocks}-block " \
        f"({sample_blocks * geo.block_bytes >> 20} MiB) plan in runs of {group}, host->host, " \
        f"{el:.1f} s"


def run_reference(args, geo):
    rank, world, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU reference arm
    threads = os.cpu_count() or 1
    from oracle import c_oracle
    from oracle.bytes_oracle import random_runs
    sample_blocks, pool = 512, 1024
    rng = np.random.default_rng(1)
    planes = np.full((geo.num_planes, pool, geo.plane_chunk_bytes), 7, dtype=np.uint8)
    host = np.zeros((pool, geo.block_bytes), dtype=np.uint8)
    ops = random_runs(rng, sample_blocks, min(args.group, sample_blocks), pool, pool)

    def step():
        c_oracle.apply_plan_arrays("out", planes, host, ops, nthreads=threads)
        c_oracle.apply_plan_arrays("in", planes, host, ops, nthreads=threads)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    nbytes = 2 * sample_blocks * geo.block_bytes * args.steps
    val = nbytes / el / 1e9
    sample = (f"per step: swap-out + swap-in of a {sample_blocks}-block "
              f"({sample_blocks * geo.block_bytes >> 20} MiB) plan in runs of {args.group}, "
              f"host buffers, oracle C restatement, {threads} pthreads")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(el / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": f"config2 block-group swap, {geo.name} KV shape, group={args.group}",
                   "plan_blocks": sample_blocks, "block_bytes": geo.block_bytes},
        "cpu_baseline": {"value": round(val, 3), "unit": "GB/s", "cores": threads,
                         "kind": "port", "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": round(val, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm

def run_ours(args, geo):
    import torch
    import torch.distributed as dist

    from paper_2411_18424_b200.dataplane import (HostKVPool, PagedKVCache, SwapDataPlane,
                                                 host_link_info, numa_nodes)

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
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    cache = PagedKVCache(geo, POOL_BLOCKS, device=dev)
    host = HostKVPool(HOST_POOL_BLOCKS, geo.block_bytes, numa_node=None, device=dev)
    host_numa = host.numa_node
    dp = SwapDataPlane(cache, host, ctas={"out": args.ctas, "in": args.ctas})
    cache.planes.view(torch.int32).random_()
    out_ops, in_ops = make_plans(args.group, seed=rank)
    nbytes_dir = PLAN_BLOCKS * geo.block_bytes
    s = torch.cuda.Stream(device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

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
    sec_max = sec
    if world > 1:
        t = torch.tensor([sec], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec_max = float(t.item())
    value = world * 2 * nbytes_dir * args.steps / sec_max / 1e9
    out_gbs = nbytes_dir / (statistics.mean(out_ms) * 1e-3) / 1e9
    in_gbs = nbytes_dir / (statistics.mean(in_ms) * 1e-3) / 1e9

    # ---- e2e: public API (control plane + dispatch) with host round trip ----
    e2e = run_e2e(args, geo, dp, dev, barrier, world)
    dp.set_launch("out", args.ctas, 0)
    dp.set_launch("in", args.ctas, 0)

    # ---- copy-engine peak on this box (roofline context) ----
    ce = ce_peak(dev, host, cache) if rank == 0 else None

    # ---- group-size sweep (config 2), kernel vs copy-engine comparators ----
    sweep = None
    if rank == 0 and not args.no_sweep:
        sweep = group_sweep(dp, s)

    # ---- the SM partition is an optimisation: fall back to shared SMs if the
    #      driver cannot create green contexts on this box ----
    if args.sm_partition:
        from paper_2411_18424_b200.swap import partition_streams
        try:
            partition_streams(dev, args.sm_partition)
        except (RuntimeError, ValueError) as exc:
            print(f"bench: SM partition unavailable ({exc}); sharing all SMs", file=sys.stderr)
            args.sm_partition = 0

    # ---- serving configuration: paced swaps under a concurrent decode load ----
    serving = serving_interference(dp, dev, s) if rank == 0 else None
    if rank == 0 and args.sm_partition:
        serving = {"shared_sms": serving,
                   f"swap_on_{args.sm_partition}_sms": serving_interference(
                       dp, dev, s, args.sm_partition)}

    # ---- live multi-turn preemption trace: P99 TTFT / TBT (metric part 2) ----
    trace = None
    if not args.no_trace:
        host.close()  # free the 10 GiB pinned pool before the trace's own pools
        trace = run_trace(args, geo, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rate, sample = cpu_oracle_rate(geo, args.group, 10.0, threads)
        cpu = {"value": round(rate, 3), "unit": "GB/s", "cores": threads, "kind": "port",
               "sample": sample, "cpu_model": cpu_model()}

    numa_per_rank = [host_numa]
    links = [host_link_info(dev)]
    if world > 1:  # where each rank's swap space lives, and which host link it uses
        numa_per_rank = [None] * world
        dist.all_gather_object(numa_per_rank, host_numa)
        links = [None] * world
        dist.all_gather_object(links, host_link_info(dev))
    root_ports = {l["root_port"] for l in links if l.get("root_port")}
    # Ranks behind one root port share its link: the aggregate roofline is the
    # smaller of one link per rank and one per distinct root port.
    link_cap = PCIE_GEN5_X16_GBS * (min(world, len(root_ports)) if root_ports else world)
    if rank == 0:
        dominant, dom_ms = ("in", in_ms) if sum(in_ms) >= sum(out_ms) else ("out", out_ms)
        achieved = nbytes_dir / (statistics.mean(dom_ms) * 1e-3) / 1e9
        traffic = ncu_traffic(dominant)
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(sec_max / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (random KV bytes, seeded random block tables)",
            "config": {"workload": f"config2 block-group swap: {PLAN_BLOCKS}-block plans "
                                   f"({nbytes_dir >> 30} GiB) out then in, runs of {args.group}, "
                                   f"{geo.name} KV shape",
                       "model_kv": geo.name, "block_bytes": geo.block_bytes,
                       "plan_blocks": PLAN_BLOCKS, "group_blocks": args.group,
                       "parallelism": f"replicas{world} (per-rank KV shard, own PCIe link)",
                       "l2": "inputs 8 GiB/direction > 126 MB L2, no flush",
                       "host_pool": {"blocks": HOST_POOL_BLOCKS, "numa_node": host_numa,
                                     "numa_node_per_rank": numa_per_rank,
                                     "numa_nodes": numa_nodes()}},
            "per_direction_gbs": {"out": round(out_gbs, 3), "in": round(in_gbs, 3)},
            "roofline": {"bound": "pcie", "achieved": round(achieved, 3),
                         "peak": PCIE_GEN5_X16_GBS, "unit": "GB/s",
                         "frac": round(achieved / PCIE_GEN5_X16_GBS, 4), "traffic": traffic,
                         "aggregate": {"gbs": round(value, 3), "links": world,
                                       "frac": round(value / (world * PCIE_GEN5_X16_GBS), 4),
                                       "root_ports": len(root_ports) or None,
                                       "topology_cap_gbs": link_cap,
                                       "frac_of_topology": round(value / link_cap, 4)},
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
            "gpu_launches": gpu_launches,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "sweep": sweep,
            "serving": serving,
            "trace": trace,
        }
        print(json.dumps(line), flush=True)
    host.close()
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, geo, dp, dev, barrier, world):
    """Same bytes through CpuStore + SwapManager.dispatch (the drop-in API)."""
    import torch

    from paper_2411_18424_b200.synthetic import random_runs
    from paper_2411_18424_b200.costmodel import TransferParams
    from paper_2411_18424_b200.cpu_store import CpuStore
    from paper_2411_18424_b200.swap import StreamExecutor, SwapManager

    # bulk round trip: the throughput policy (TMA bulk kernels both ways, plan-level waits)
    ex = StreamExecutor(dp, duplex_policy="throughput")
    mgr = SwapManager(TransferParams(), bytes_per_block=geo.block_bytes, executor=ex)
    store = CpuStore(HOST_POOL_BLOCKS, reuse_enabled=True)
    n_req, per = 64, PLAN_BLOCKS // 64
    rng = np.random.default_rng(7)
    runs = random_runs(rng, PLAN_BLOCKS, args.group, POOL_BLOCKS, HOST_POOL_BLOCKS)
    tables, cursor = [], 0
    per_runs = per // args.group if per >= args.group else 1
    for r in range(n_req):
        ext = [(int(g), int(b)) for b, g, _ in runs[cursor:cursor + per_runs]]
        cursor += per_runs
        tables.append(ext)
    foot = [sum(b for _, b in t) for t in tables]

    def step():
        for r in range(n_req):
            plan = store.plan_swap_out(r, foot[r], tables[r])
            mgr.dispatch(0, 0, plan)
        for r in range(n_req):
            plan = store.plan_swap_in(r, tables[r])
            mgr.dispatch(0, 0, plan)
        ex.synchronize()
        for r in range(n_req):
            store.release(r)
        mgr.in_flight.clear()
        mgr.busy_extents.clear()

    for _ in range(max(1, args.warmup)):
        step()
    barrier()
    torch.cuda.synchronize()
    l0 = ex.launches
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    launches = ex.launches - l0
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([el], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    moved = sum(foot) * geo.block_bytes
    for d in ("out", "in"):
        dp.set_path(d, "lsu")
    return {"value": round(world * 2 * moved * args.steps / el / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": moved, "d2h_bytes_per_step": moved,
            "api": "CpuStore.plan_swap_out/plan_swap_in -> SwapManager.dispatch -> "
                   "StreamExecutor (throughput policy: TMA bulk kernels) -> kvs_swap (C ABI); "
                   "wall clock incl. planning and sync",
            "requests_per_step": n_req, "gpu_launches": launches}


def run_trace(args, geo, dev):
    """Live-mode multi-turn preemption trace on this GPU (paper_2411_18424_b200.live):
    FastSwitch (block groups + reuse + adaptive async, one kernel per plan) vs the
    vLLM-style baseline (per-block copies on the copy engines)."""
    import dataclasses

    from paper_2411_18424_b200 import config as mconfig
    from paper_2411_18424_b200.live import DecodeEmulator, LiveEngine, b200_transfer_params
    from paper_2411_18424_b200.runtime import Runtime
    from paper_2411_18424_b200.workload import generate

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
           "cpu_pool": {"total_blocks": 4096},
           "workload": {"num_conversations": args.trace_convs, "arrival_rate_per_s": 4.0,
                        "think_time_mean_s": 2.0},
           "trace": {"pattern": args.trace_pattern, "frequency": 0.04}}
    out = {"workload": f"{args.trace_convs} conversations, 4 req/s, think 2 s, 512 x "
                       f"{geo.block_bytes / 2**20:g} MiB GPU blocks per rank (TP{world}), "
                       f"{args.trace_pattern} priorities f=0.04 (BASELINE config 3: VTC), "
                       f"decode = {decode.bytes_per_us / 1e3:.0f} GB/s weight "
                       f"streaming per rank",
           "tp": world, "sm_partition": sms, "runs": {}}
    for name, mode, impl in (("fastswitch", "full", "kernel"),
                             ("vllm_like", "baseline", "ce_per_block")):
        cfg, wl, _ = mconfig.build({**doc, "ablation": mode})
        cfg = dataclasses.replace(cfg, transfer=b200_transfer_params())
        layered = impl == "kernel" and not args.no_layered
        rt = Runtime(geo, cfg.gpu_pool.total_blocks, cfg.cpu_pool_blocks, device=dev,
                     copy_impl=impl, timing=True, sm_partition=args.sm_partition,
                     layered_swap_in=layered)
        eng = LiveEngine(cfg, generate(wl), rt, decode, agreement=agreement, layered=layered)
        eng.turn_trace = []
        rep = eng.run()
        lat = eng.latency_summary()
        anat = eng.ttft_anatomy()
        st = rt.stats()
        out["runs"][name] = {"ablation": mode, "copy_impl": impl,
                             **{k: lat[k] for k in ("ttft_p50_ms", "ttft_p99_ms", "tbt_p99_ms",
                                                    "tbt_p999_ms", "decode_stall_frac",
                                                    "swap_induced_decode_stall", "wall_s")},
                             "ttft_tail_ms": {"turns": anat.get("turns"),
                                              **anat.get("tail_mean_ms", {})},
                             "layered_joins": lat["layered_joins"],
                             "kv_read_gib_verified": lat["kv_read_gib"],
                             "tokens": rep.total_tokens,
                             "swap_gib": {"out": round(st["bytes_out"] / 2**30, 2),
                                          "in": round(st["bytes_in"] / 2**30, 2)},
                             "kernel_launches": st["kernel_launches"]}
        rt.close()
    del decode
    torch_empty_cache()
    return out


def serving_interference(dp, dev, s, sm_partition: int = 0):
    """Swap-induced decode stall, measured: 2 ms HBM-streaming decode steps on a
    high-priority stream while a 2 GiB swap runs, per direction, with the
    serving ("latency") policy: paced kernels + shared budget (swap.py)."""
    import statistics

    import torch

    from paper_2411_18424_b200.synthetic import random_runs
    from paper_2411_18424_b200.live import DecodeEmulator
    from paper_2411_18424_b200.swap import DUPLEX_POLICIES

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
    n = 1024
    ops = random_runs(rng, n, 16, POOL_BLOCKS // 2, HOST_POOL_BLOCKS // 2).astype(np.int32)
    ops_in = ops.copy()
    ops_in[:, 1] += POOL_BLOCKS // 2
    ops_in[:, 2] += HOST_POOL_BLOCKS // 2
    nbytes = n * dp.geometry.block_bytes

    def steps(k):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(k + 1)]
        evs[0].record(comp)
        for i in range(k):
            dec.launch_us(comp, 2000.0)
            evs[i + 1].record(comp)
        return evs

    steps(3)
    torch.cuda.synchronize()
    ev = steps(20)
    torch.cuda.synchronize()
    solo = statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(20))
    policy = os.environ.get("KVS_SERVING_POLICY", "latency")
    pol = DUPLEX_POLICIES[policy]
    for d in ("out", "in"):
        c, t, pace = pol[d]
        dp.set_launch(d, c, t)
        dp.set_pace(d, pace)
    dp.set_budget(pol["budget"])
    dp.set_budget_priority(pol.get("priority"))
    out = {"policy": policy, "sm_partition": sms, "decode_step_solo_ms": round(solo, 3),
           "runs": {}}
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
        dp.set_launch(d, 0, 0)
        dp.set_pace(d, 0.0)
    dp.set_budget(0.0)
    dp.set_budget_priority(None)
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


def group_sweep(dp, s):
    import torch
    from paper_2411_18424_b200.synthetic import random_runs
    geo = dp.geometry
    out = []
    rng = np.random.default_rng(11)
    nbytes = PLAN_BLOCKS * geo.block_bytes
    for g in (1, 4, 16, 64, 256):
        ops = random_runs(rng, PLAN_BLOCKS, g, POOL_BLOCKS, HOST_POOL_BLOCKS).astype(np.int32)
        row = {"group": g}
        for d in ("out", "in"):
            for impl, fn in (("kernel", lambda: dp.swap(d, ops, stream=s)),
                             ("ce_per_run", lambda: dp.baseline(d, 1, ops, stream=s)),
                             ("ce_batch", lambda: dp.baseline(d, 2, ops, stream=s))):
                fn()
                s.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                fn()
                e1.record(s)
                s.synchronize()
                row[f"{d}_{impl}"] = round(nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)
        out.append(row)
    return out


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
    from paper_2411_18424_b200.geometry import PRESETS
    geo = PRESETS[args.model]
    if args.impl == "reference":
        run_reference(args, geo)
    else:
        run_ours(args, geo)


if __name__ == "__main__":
    main()
