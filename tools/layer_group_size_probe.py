"""Swap-in GB/s of layer-pipelined (plane-major, plane-flagged) plans per
plan size and planes-per-group, at the serving launch shape (8 x 256): do
short plans lose their rate to the per-group fences or to the order?

python tools/layer_group_size_probe.py   -> gpurun_out/layer_group_size_probe.json
"""

import json
import os
import statistics
import sys
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
    flags = torch.zeros(1 << 16, dtype=torch.int32, device="cuda:0")
    fp = flags.data_ptr()
    st = torch.cuda.Stream()
    rng = np.random.default_rng(4)
    res = {"runs": []}
    seq = 0
    for blocks in (8, 16, 32, 73, 256):
        plans = [orc.random_runs(rng, blocks, 18, POOL, POOL).astype(np.int32) for _ in range(6)]
        row = {"blocks": blocks, "mib": 2 * blocks}
        for group in (-1, 0, 8, 16, 32):
            times = []
            for rep in range(3):
                for ops in plans:
                    seq += 1
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    if group < 0:
                        dp.swap("in", ops, stream=st)
                    else:
                        dp.set_layer_group(group)
                        dp.swap_layered("in", ops, fp, seq, stream=st)
                    e1.record(st)
                    st.synchronize()
                    if rep:
                        times.append(e0.elapsed_time(e1))
            name = "plain" if group < 0 else f"group{group or 'auto'}"
            row[name] = round(blocks * geo.block_bytes / (statistics.median(times) * 1e-3) / 1e9, 2)
        res["runs"].append(row)
        print(json.dumps(row), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/layer_group_size_probe.json", "w") as f:
        json.dump(res, f, indent=1)
    host.close()


if __name__ == "__main__":
    main()
