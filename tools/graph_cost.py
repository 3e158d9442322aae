"""Host cost of launching one decode step (32 layers x attention + weight
kernel) kernel by kernel vs as a re-captured, in-place-updated CUDA graph
(live.DecodeGraph): CPU µs per step, the GPU idle.

python tools/graph_cost.py   -> gpurun_out/graph_cost.json
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
from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane  # noqa: E402
from paper_2411_18424_b200.geometry import LLAMA3_8B  # noqa: E402
from paper_2411_18424_b200.live import DecodeEmulator, DecodeGraph  # noqa: E402


def main():
    geo = LLAMA3_8B
    cache = PagedKVCache(geo, 512, device="cuda:0")
    host = HostKVPool(16, geo.block_bytes)
    dp = SwapDataPlane(cache, host)
    dec = DecodeEmulator("cuda:0", weight_bytes=1 << 30)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    comp = torch.cuda.Stream()
    g = DecodeGraph("cuda:0", marks=2 * geo.num_planes + 2)
    rng = np.random.default_rng(0)
    res = {}
    for kind in ("stream", "graph", "graph_marks"):
        times = []
        for it in range(300):
            n = int(rng.integers(4, 40))
            segs = np.stack([np.arange(n), np.zeros(n, dtype=np.int64),
                             rng.integers(1, 64, n), rng.integers(0, 400, n)], 1).astype(np.int64)
            t0 = time.perf_counter()
            st = comp if kind == "stream" else g.begin()
            for layer in range(geo.num_planes):
                if kind == "graph_marks":
                    g.mark(2 * layer)
                dp.kv_tokens(1, segs, stream=st, mismatch_ptr=bad.data_ptr(),
                             planes=(layer, layer + 1))
                dec.launch(st, 1 << 20)
                if kind == "graph_marks":
                    g.mark(2 * layer + 1)
            if kind != "stream":
                g.end()
                g.launch(comp)
            times.append((time.perf_counter() - t0) * 1e6)
            comp.synchronize()
        res[kind] = {"cpu_us_per_step_median": round(statistics.median(times[20:]), 1),
                     "cpu_us_per_step_p90": round(float(np.percentile(times[20:], 90)), 1)}
        print(kind, res[kind], flush=True)
    res["graph_stats"] = g.stats()
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/graph_cost.json", "w") as f:
        json.dump(res, f, indent=1)
    g.close()
    host.close()


if __name__ == "__main__":
    main()
