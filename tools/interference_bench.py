"""Swap-induced decode stall, measured directly (north star: <= 10%).

A decode step is the HBM-streaming stand-in (kvs_stream_read over a 16 GiB
"weights" buffer, 2 ms nominal, all SMs).  Each configuration runs a long
swap (8 GiB) on the swap stream and decode steps back to back on a
high-priority compute stream while the swap is in flight; decode-step time
is compared with the same steps alone, and the swap's GB/s under decode load
is reported.

python tools/interference_bench.py   -> gpurun_out/interference.json
"""

import json
import os
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import bytes_oracle as orc  # noqa: E402  (plan generator only)
from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane  # noqa: E402
from paper_2411_18424_b200.geometry import LLAMA3_8B  # noqa: E402
from paper_2411_18424_b200.live import DecodeEmulator  # noqa: E402

STEP_US = 2000.0
POOL = 4096


def decode_steps(dec, stream, n):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    evs[0].record(stream)
    for i in range(n):
        dec.launch_us(stream, STEP_US)
        evs[i + 1].record(stream)
    return evs


def main():
    geo = LLAMA3_8B
    cache = PagedKVCache(geo, POOL, device="cuda:0")
    host = HostKVPool(POOL, geo.block_bytes)
    dp = SwapDataPlane(cache, host)
    cache.planes.view(torch.int32).random_()
    dec = DecodeEmulator("cuda:0", weight_bytes=16 << 30)
    comp = torch.cuda.Stream(priority=-1)
    s_out, s_in = torch.cuda.Stream(), torch.cuda.Stream()
    rng = np.random.default_rng(0)
    half = POOL // 2
    ops_out = orc.random_runs(rng, half, 16, half, half).astype(np.int32)
    ops_in = orc.random_runs(rng, half, 16, half, half).astype(np.int32)
    ops_in[:, 1:] += half
    nbytes = half * geo.block_bytes

    # solo decode
    decode_steps(dec, comp, 5)
    torch.cuda.synchronize()
    evs = decode_steps(dec, comp, 40)
    torch.cuda.synchronize()
    solo = statistics.median(evs[i].elapsed_time(evs[i + 1]) for i in range(40))
    results = {"decode_step_solo_ms": round(solo, 4), "runs": []}
    print(json.dumps(results), flush=True)

    configs = []
    for path, ctas, extra in (("lsu", 4, {}), ("lsu", 8, {}), ("lsu", 32, {}),
                              ("bulk", 8, {"piece": 16384, "stages": 4}),
                              ("bulk", 16, {"piece": 16384, "stages": 4}),
                              ("bulk", 64, {"piece": 16384, "stages": 4})):
        for dirs in (("in",), ("out",), ("out", "in")):
            configs.append((path, ctas, extra, dirs))
    for path, ctas, extra, dirs in configs:
        for d in ("out", "in"):
            dp.set_path(d, path, extra.get("piece", 0), extra.get("stages", 0))
            dp.set_launch(d, ctas if path == "bulk" else (ctas if d == "in" or len(dirs) == 1
                                                          else 8), 0)
        torch.cuda.synchronize()
        t = {}
        for d in dirs:
            st = s_out if d == "out" else s_in
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            dp.swap(d, ops_out if d == "out" else ops_in, stream=st)
            e1.record(st)
            t[d] = (e0, e1)
        # decode steps while the swaps run (only steps that start before the swaps end count)
        evs = decode_steps(dec, comp, 60)
        torch.cuda.synchronize()
        swap_end = max(t[d][0].elapsed_time(t[d][1]) for d in dirs)
        steps, acc = [], 0.0
        base = evs[0]
        for i in range(60):
            start = t[dirs[0]][0].elapsed_time(evs[i])  # step start relative to swap start
            if start > swap_end:
                break
            steps.append(evs[i].elapsed_time(evs[i + 1]))
        row = {"path": path, "ctas": ctas, "dirs": "+".join(dirs),
               "decode_steps_overlapped": len(steps),
               "decode_slowdown": round(statistics.median(steps) / solo - 1, 4) if steps else None,
               "swap_gbs": {d: round(nbytes / (t[d][0].elapsed_time(t[d][1]) * 1e-3) / 1e9, 2)
                            for d in dirs}}
        results["runs"].append(row)
        print(json.dumps(row), flush=True)
    for d in ("out", "in"):
        dp.set_path(d, "lsu")
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/interference.json", "w") as f:
        json.dump(results, f, indent=1)
    host.close()


if __name__ == "__main__":
    main()
