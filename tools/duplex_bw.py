"""Full-duplex swap bandwidth: swap-out and swap-in plans running concurrently
on their two streams (preempt one request while resuming another).

python tools/duplex_bw.py [--ctas-out 4,8,16] [--ctas-in 16,32,64,148]
Writes gpurun_out/duplex_bw.json.
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


def run_pair(launch_out, launch_in, s_out, s_in, reps):
    """Both directions back to back `reps` times; per-direction event timing."""
    torch.cuda.synchronize()
    ev = {k: torch.cuda.Event(enable_timing=True) for k in ("o0", "o1", "i0", "i1")}
    ev["o0"].record(s_out)
    s_in.wait_event(ev["o0"])
    ev["i0"].record(s_in)
    for _ in range(reps):
        launch_out()
        launch_in()
    ev["o1"].record(s_out)
    ev["i1"].record(s_in)
    torch.cuda.synchronize()
    t_out = ev["o0"].elapsed_time(ev["o1"]) * 1e-3
    t_in = ev["i0"].elapsed_time(ev["i1"]) * 1e-3
    return t_out, t_in


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--blocks", type=int, default=2048)
    ap.add_argument("--group", type=int, default=16)
    ap.add_argument("--ctas-out", default="4,8,16,32")
    ap.add_argument("--ctas-in", default="8,16,32,64,148")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    geo = PRESETS[args.model]
    pool = 2 * args.blocks + 64
    cache = PagedKVCache(geo, pool, device="cuda:0")
    host = HostKVPool(pool, geo.block_bytes)
    dp = SwapDataPlane(cache, host)
    cache.planes.view(torch.int32).random_()
    rng = np.random.default_rng(0)
    half = pool // 2
    ops_out = orc.random_runs(rng, args.blocks, args.group, half, half).astype(np.int32)
    ops_in = orc.random_runs(rng, args.blocks, args.group, half, half).astype(np.int32)
    ops_in[:, 1:] += half  # disjoint halves: no hazards between the two directions
    nbytes = args.blocks * geo.block_bytes
    s_out, s_in = torch.cuda.Stream(), torch.cuda.Stream()
    res = []
    for co in [int(x) for x in args.ctas_out.split(",")]:
        for ci in [int(x) for x in args.ctas_in.split(",")]:
            dp.set_launch("out", co, 512)
            dp.set_launch("in", ci, 512)
            run_pair(lambda: dp.swap("out", ops_out, stream=s_out),
                     lambda: dp.swap("in", ops_in, stream=s_in), s_out, s_in, 1)
            t_out, t_in = run_pair(lambda: dp.swap("out", ops_out, stream=s_out),
                                   lambda: dp.swap("in", ops_in, stream=s_in), s_out, s_in,
                                   args.reps)
            row = dict(impl="kernel", ctas_out=co, ctas_in=ci,
                       out_gbs=round(args.reps * nbytes / t_out / 1e9, 2),
                       in_gbs=round(args.reps * nbytes / t_in / 1e9, 2))
            row["total_gbs"] = round(2 * args.reps * nbytes / max(t_out, t_in) / 1e9, 2)
            res.append(row)
            print(json.dumps(row), flush=True)
    for mode, name in ((1, "ce_per_run"), (2, "ce_staged")):
        t_out, t_in = run_pair(lambda: dp.baseline("out", mode, ops_out, stream=s_out),
                               lambda: dp.baseline("in", mode, ops_in, stream=s_in),
                               s_out, s_in, args.reps)
        row = dict(impl=name, out_gbs=round(args.reps * nbytes / t_out / 1e9, 2),
                   in_gbs=round(args.reps * nbytes / t_in / 1e9, 2),
                   total_gbs=round(2 * args.reps * nbytes / max(t_out, t_in) / 1e9, 2))
        res.append(row)
        print(json.dumps(row), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/duplex_bw.json", "w") as f:
        json.dump(res, f, indent=1)
    host.close()


if __name__ == "__main__":
    main()
