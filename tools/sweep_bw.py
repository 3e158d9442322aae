"""Bandwidth sweep of the swap kernels vs copy-engine baselines (config 2).

python tools/sweep_bw.py [--blocks 4096] [--groups 1,4,16,64,256] [--ctas 8,16,32,64,148]
Writes gpurun_out/sweep_bw.json.
"""

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_18424_b200 import synthetic as orc  # noqa: E402  (plan generator)
from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane  # noqa: E402
from paper_2411_18424_b200.geometry import PRESETS  # noqa: E402


def timed(fn, stream, reps):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    fn()
    stream.synchronize()
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    stream.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--blocks", type=int, default=4096)
    ap.add_argument("--pool", type=int, default=8192)
    ap.add_argument("--groups", default="1,4,16,64,256")
    ap.add_argument("--ctas", default="4,8,16,32,64,148")
    ap.add_argument("--threads", default="512")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--baselines", default="1,2,0")
    ap.add_argument("--paths", default="lsu")
    ap.add_argument("--pieces", default="16384")
    ap.add_argument("--stages", default="4")
    ap.add_argument("--no-duplex", action="store_true")
    args = ap.parse_args()
    geo = PRESETS[args.model]
    cache = PagedKVCache(geo, args.pool, device="cuda:0")
    host = HostKVPool(args.pool, geo.block_bytes)
    dp = SwapDataPlane(cache, host)
    cache.planes.view(torch.int32).random_()
    s = torch.cuda.Stream()
    rng = np.random.default_rng(0)
    res = []
    nbytes = args.blocks * geo.block_bytes
    for g in [int(x) for x in args.groups.split(",")]:
        ops = orc.random_runs(rng, args.blocks, g, args.pool, args.pool)
        for d in ("out", "in"):
            combos = []
            for path in args.paths.split(","):
                if path == "lsu":
                    combos += [(path, 0, 0, t) for t in [int(x) for x in args.threads.split(",")]]
                else:
                    combos += [(path, pb, st, 32) for pb in [int(x) for x in args.pieces.split(",")]
                               for st in [int(x) for x in args.stages.split(",")]
                               if pb * st <= 227 * 1024]
            for path, pb, st, t in combos:
                dp.set_path(d, path, pb, st)
                for c in [int(x) for x in args.ctas.split(",")]:
                    dp.set_launch(d, c, t if path == "lsu" else 0)
                    sec = timed(lambda: dp.swap(d, ops, stream=s), s, args.reps)
                    res.append(dict(group=g, dir=d, impl="kernel", path=path, piece=pb, stages=st,
                                    ctas=c, threads=t, gbs=nbytes / sec / 1e9))
                    print(json.dumps(res[-1]), flush=True)
            dp.set_path(d, "lsu")
            for mode in [int(x) for x in args.baselines.split(",") if x]:
                if mode == 0 and g > 16:
                    continue
                sec = timed(lambda: dp.baseline(d, mode, ops, stream=s), s, 1)
                res.append(dict(group=g, dir=d, impl=["ce_per_block", "ce_per_run", "ce_staged"][mode],
                                gbs=nbytes / sec / 1e9))
                print(json.dumps(res[-1]), flush=True)
    if args.no_duplex:
        os.makedirs("gpurun_out", exist_ok=True)
        with open("gpurun_out/sweep_bw.json", "w") as f:
            json.dump(res, f, indent=1)
        return
    # duplex: out and in concurrently on two streams
    s2 = torch.cuda.Stream()
    ops = orc.random_runs(rng, args.blocks // 2, 16, args.pool // 2, args.pool // 2)
    ops_in = ops.copy()
    ops_in[:, 1] += args.pool // 2
    ops_in[:, 2] += args.pool // 2
    for c in (16, 32, 64):
        dp.set_launch("out", c, 512)
        dp.set_launch("in", c, 512)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        s2.wait_event(e0)
        for _ in range(args.reps):
            dp.swap("out", ops, stream=s)
            dp.swap("in", ops_in, stream=s2)
        ev = torch.cuda.Event()
        ev.record(s2)
        s.wait_event(ev)
        e1.record(s)
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) * 1e-3
        res.append(dict(group=16, dir="duplex", impl="kernel", ctas=c,
                        gbs=2 * args.reps * (args.blocks // 2) * geo.block_bytes / sec / 1e9))
        print(json.dumps(res[-1]), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/sweep_bw.json", "w") as f:
        json.dump(res, f, indent=1)
    host.close()


if __name__ == "__main__":
    main()
