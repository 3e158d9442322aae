"""Why short swap-ins run below the link rate: per-plan fixed cost or a
cold start after idle?  Swap-in of B-block plans (LLaMA-3-8B, random runs of
18 blocks, serving launch shape 8 x 256) timed per plan with CUDA events,
(a) each plan alone after an idle gap of `gap` ms (host sleep after a sync),
(b) six plans back to back on the stream.

python tools/warmup_probe.py   -> gpurun_out/warmup_probe.json
"""

import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_18424_b200 import synthetic as orc  # noqa: E402
from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane  # noqa: E402
from paper_2411_18424_b200.geometry import LLAMA3_8B  # noqa: E402

POOL = 2048


def main():
    geo = LLAMA3_8B
    cache = PagedKVCache(geo, POOL, device="cuda:0")
    host = HostKVPool(POOL, geo.block_bytes)
    dp = SwapDataPlane(cache, host)
    dp.set_launch("in", 8, 256)
    st = torch.cuda.Stream()
    rng = np.random.default_rng(9)
    res = {"runs": []}
    for blocks in (8, 32, 73, 256):
        plans = [orc.random_runs(rng, blocks, 18, POOL, POOL).astype(np.int32) for _ in range(6)]
        nbytes = blocks * geo.block_bytes
        row = {"blocks": blocks, "mib": blocks * 2}
        for gap in (0.0, 1.0, 20.0):
            times = []
            for rep in range(3):
                for ops in plans:
                    st.synchronize()
                    if gap:
                        time.sleep(gap * 1e-3)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    dp.swap("in", ops, stream=st)
                    e1.record(st)
                    st.synchronize()
                    if rep:
                        times.append(e0.elapsed_time(e1))
            row[f"alone_gap{gap:g}ms_gbs"] = round(nbytes / (statistics.median(times) * 1e-3) / 1e9, 2)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(13)]
        st.synchronize()
        evs[0].record(st)
        for i, ops in enumerate(plans + plans):
            dp.swap("in", ops, stream=st)
            evs[i + 1].record(st)
        st.synchronize()
        per = [evs[i].elapsed_time(evs[i + 1]) for i in range(12)]
        row["back_to_back_first_gbs"] = round(nbytes / (per[0] * 1e-3) / 1e9, 2)
        row["back_to_back_rest_gbs"] = round(nbytes / (statistics.median(per[1:]) * 1e-3) / 1e9, 2)
        res["runs"].append(row)
        print(json.dumps(row), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/warmup_probe.json", "w") as f:
        json.dump(res, f, indent=1)
    host.close()


if __name__ == "__main__":
    main()
