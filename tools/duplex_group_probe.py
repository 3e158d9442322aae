"""Both directions at once on the TMA bulk kernel, per group size and seed:
the bench sweep's duplex_kernel_bulk is ~80 GB/s at every group size except
g=8 (~52, in two rounds).  Is it the group size, the plan, or the launch?

For each (group, seed): 1280-block plans each way on disjoint halves of the
pools (as bench.group_sweep), combined GB/s over both streams' lifetimes,
and each kernel's own start/end (does one wait for the other?).

python tools/duplex_group_probe.py   -> gpurun_out/duplex_group_probe.json
"""

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane  # noqa: E402
from paper_2411_18424_b200.geometry import LLAMA3_8B  # noqa: E402
from paper_2411_18424_b200.synthetic import random_runs  # noqa: E402


def main():
    geo = LLAMA3_8B
    gp, hp = 8192, 5120
    cache = PagedKVCache(geo, gp, device="cuda:0")
    host = HostKVPool(hp, geo.block_bytes)
    dp = SwapDataPlane(cache, host)
    for d in ("out", "in"):
        dp.set_path(d, "bulk")
    s, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    half = 1280
    res = {"runs": []}
    for g in (4, 6, 7, 8, 9, 10, 12, 16):
        for seed in (11, 12, 13):
            rng = np.random.default_rng([seed, g])
            h_out = random_runs(rng, half, g, gp // 2, hp // 2).astype(np.int32)
            h_in = random_runs(rng, half, g, gp // 2, hp // 2).astype(np.int32)
            h_in[:, 1] += gp // 2
            h_in[:, 2] += hp // 2
            for order in ("out_first", "in_first"):
                torch.cuda.synchronize()
                ev = {k: torch.cuda.Event(enable_timing=True) for k in ("o0", "o1", "i0", "i1")}
                pairs = [("o", s, "out", h_out), ("i", s2, "in", h_in)]
                if order == "in_first":
                    pairs.reverse()
                for tag, st, d, ops in pairs:
                    ev[tag + "0"].record(st)
                    dp.swap(d, ops, stream=st)
                    ev[tag + "1"].record(st)
                torch.cuda.synchronize()
                ref = ev["o0"]
                t = {k: ref.elapsed_time(e) for k, e in ev.items()}
                span = max(t["o1"], t["i1"]) - min(t["o0"], t["i0"])
                row = {"group": g, "seed": seed, "order": order, "ops": int(len(h_out)),
                       "gbs": round(2 * half * geo.block_bytes / (span * 1e-3) / 1e9, 2),
                       "out_ms": [round(t["o0"], 2), round(t["o1"], 2)],
                       "in_ms": [round(t["i0"], 2), round(t["i1"], 2)]}
                res["runs"].append(row)
                print(json.dumps(row), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/duplex_group_probe.json", "w") as f:
        json.dump(res, f, indent=1)
    host.close()


if __name__ == "__main__":
    main()
