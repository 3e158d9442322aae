"""Live-mode multi-turn preemption trace on one B200: P99 TTFT/TBT, swap GB/s
while serving, swap-induced decode stall.  Compares ablations / copy paths.

python tools/live_trace.py --convs 60 --rate 2 --modes full:kernel,baseline:ce_per_block
Writes gpurun_out/live_trace.json.
"""

import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2411_18424_b200 import config as mconfig  # noqa: E402
from paper_2411_18424_b200.geometry import PRESETS  # noqa: E402
from paper_2411_18424_b200.live import DecodeEmulator, LiveEngine, b200_transfer_params  # noqa: E402
from paper_2411_18424_b200.runtime import Runtime  # noqa: E402
from paper_2411_18424_b200.workload import generate  # noqa: E402


def run_one(args, mode, impl, decode, geo):
    doc = {
        "ablation": mode,
        "block": {"bytes_per_block": geo.block_bytes},
        "gpu_pool": {"total_blocks": args.gpu_blocks},
        "cpu_pool": {"total_blocks": args.cpu_blocks},
        "workload": {"num_conversations": args.convs, "arrival_rate_per_s": args.rate,
                     "think_time_mean_s": args.think},
        "trace": {"pattern": args.pattern, "frequency": args.freq},
    }
    cfg, wl, _ = mconfig.build(doc)
    cfg = type(cfg)(**{**cfg.__dict__, "transfer": b200_transfer_params(args.pcie_gbs)})
    rt = Runtime(geo, cfg.gpu_pool.total_blocks, cfg.cpu_pool_blocks, copy_impl=impl,
                 verify=args.verify, timing=True, duplex_policy=args.policy,
                 sm_partition=args.sm_partition, layered_swap_in=args.layered)
    eng = LiveEngine(cfg, generate(wl), rt, decode, layered=args.layered and impl == "kernel",
                     attend=not args.no_attend,
                     per_layer_decode=not args.single_kernel_decode,
                     graph_decode=not args.stream_decode,
                     control_plane=args.control_plane)
    eng.turn_trace = []
    t0 = time.perf_counter()
    rep = eng.run()
    wall = time.perf_counter() - t0
    lat = eng.latency_summary()
    st = rt.stats()
    # swap throughput while serving: bytes / summed per-transfer device time
    ex = rt.executor
    secs = {"out": 0.0, "in": 0.0}
    nbytes = {"out": 0, "in": 0}
    for r in ex.history:
        if r.start_event is not None and r.nbytes:
            secs[r.direction] += r.start_event.elapsed_time(r.event) * 1e-3
            nbytes[r.direction] += r.nbytes + r.refresh_bytes
    out = {
        "mode": mode, "copy_impl": impl, "wall_s": round(wall, 2),
        "policy": args.policy, "layered": args.layered, "sm_partition": args.sm_partition,
        "policy_def": {k: list(v) if isinstance(v, tuple) else v
                       for k, v in __import__("paper_2411_18424_b200.swap", fromlist=["x"])
                       .DUPLEX_POLICIES[args.policy].items()},
        "attend": not args.no_attend,
        "decode_launch": "cuda_graph" if eng.graph is not None else "stream",
        "control_plane": args.control_plane,
        "graph_stats": eng.graph.stats() if eng.graph is not None else None,
        "latency": lat,
        "iteration_anatomy": eng.iteration_anatomy(),
        "swap_rates": rt.swap_rates(),
        "report": {k: v for k, v in rep.to_dict().items() if k != "granularity_histogram"},
        "swap": {d: {"bytes": nbytes[d], "gbs_while_busy": round(nbytes[d] / secs[d] / 1e9, 2)
                     if secs[d] else None, "transfers": sum(1 for r in ex.history
                                                             if r.direction == d)}
                 for d in ("out", "in")},
        "runtime": st,
        "slowest_transfers_ms": sorted(
            ((round(r.start_event.elapsed_time(r.event), 2), r.direction, len(r.gpu),
              r.nbytes >> 20) for r in ex.history if r.start_event is not None),
            reverse=True)[:8],
        "slowest_iterations": sorted(eng._trace, reverse=True)[:8],
        "ttft_top": sorted(eng.ttft_samples, reverse=True)[:8],
        "ttft_anatomy": eng.ttft_anatomy(),
    }
    rt.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--convs", type=int, default=60)
    ap.add_argument("--rate", type=float, default=2.0)
    ap.add_argument("--think", type=float, default=10.0)
    ap.add_argument("--gpu-blocks", type=int, default=512)
    ap.add_argument("--cpu-blocks", type=int, default=8192)
    ap.add_argument("--pattern", default="markov")
    ap.add_argument("--freq", type=float, default=0.04)
    ap.add_argument("--pcie-gbs", type=float, default=51.0)
    ap.add_argument("--modes", default="full:kernel,baseline:ce_per_block")
    ap.add_argument("--weights-gib", type=int, default=16)
    ap.add_argument("--verify", action="store_true")
    ap.add_argument("--policy", default="serving")
    ap.add_argument("--sm-partition", type=int, default=0,
                    help="swap kernels on their own N-SM green context, decode on the rest")
    ap.add_argument("--layered", action="store_true",
                    help="resumed requests join decode layer by layer (plane flags)")
    ap.add_argument("--decode-ctas", type=int, default=0,
                    help="decode weight-stream kernel: 0 = 2 persistent CTAs per compute SM, "
                         "<0 = one CTA per -N KiB tile (block-scheduler balanced)")
    ap.add_argument("--single-kernel-decode", action="store_true",
                    help="one weight-stream kernel per step instead of one per layer")
    ap.add_argument("--stream-decode", action="store_true",
                    help="launch the per-layer decode kernels one by one on the stream "
                         "instead of as one CUDA graph")
    ap.add_argument("--control-plane", default="python", choices=["python", "native"])
    ap.add_argument("--policy-json", default="",
                    help='register a custom duplex policy under --policy, e.g. '
                         '\'{"out": [8, 512, 52], "in": [8, 256, 45], "budget": 60}\'')
    ap.add_argument("--no-attend", action="store_true",
                    help="decode streams weights only (no per-layer KV reads)")
    ap.add_argument("--out", default="gpurun_out/live_trace.json")
    args = ap.parse_args()
    if args.policy_json:
        from paper_2411_18424_b200.swap import DUPLEX_POLICIES
        pol = json.loads(args.policy_json)
        DUPLEX_POLICIES[args.policy] = {k: tuple(v) if k in ("out", "in") else v
                                        for k, v in pol.items()}
    geo = PRESETS[args.model]
    stream, ctas = None, 0
    if args.sm_partition:
        from paper_2411_18424_b200.swap import partition_streams
        _, stream, sms = partition_streams(torch.device("cuda:0"), args.sm_partition)
        ctas = 2 * sms[1]
    if args.decode_ctas:
        ctas = args.decode_ctas
    decode = DecodeEmulator("cuda:0", weight_bytes=args.weights_gib << 30, ctas=ctas,
                            stream=stream)
    results = {"decode_calibrated_gbs": round(decode.bytes_per_us / 1e3, 1), "runs": []}
    for item in args.modes.split(","):
        mode, impl = item.split(":")
        res = run_one(args, mode, impl, decode, geo)
        results["runs"].append(res)
        res["decode"] = {"ctas": ctas, "per_layer": not args.single_kernel_decode,
                         "calibrated_gbs": results["decode_calibrated_gbs"]}
        print(json.dumps({k: res[k] for k in ("mode", "copy_impl", "policy", "layered", "decode",
                                              "sm_partition", "wall_s", "latency", "swap",
                                              "swap_rates", "slowest_transfers_ms",
                                              "ttft_anatomy")}),
              flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(results, f, indent=1)


if __name__ == "__main__":
    main()
