"""Swap-in GB/s per completion-signal variant, alone, at the live traces'
plan shapes: why the live trace's swap-in runs ~47 GB/s while busy when the
plain kernel moves 51.4 GB/s.

Plans: B blocks of 2 MiB (LLaMA-3-8B) in random runs of mean 18 blocks
(the traces' granularity), swapped in at the serving launch shape (8 CTAs x
256 threads) through: kvs_swap (no flags), kvs_swap_ops (op flags),
kvs_swap_layered (plane flags, plane-major), kvs_swap_signaled (op + plane +
done), each with and without the 60 GB/s shared budget.

python tools/swapin_path_probe.py   -> gpurun_out/swapin_path_probe.json
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
    flags = torch.zeros(1 << 16, dtype=torch.int32, device="cuda:0")
    fp = flags.data_ptr()
    st = torch.cuda.Stream()
    rng = np.random.default_rng(3)
    res = {"runs": []}
    seq = 0
    for budget in (0.0, 60.0):
        dp.set_budget(budget)
        for blocks in (8, 32, 73, 256, 1024):
            plans = [orc.random_runs(rng, blocks, 18, POOL, POOL).astype(np.int32)
                     for _ in range(6)]
            row = {"budget": budget, "blocks": blocks, "mib": blocks * 2}
            for kind in ("plain", "ops", "layered", "signaled"):
                dp.set_launch("in", 8, 256)
                times = []
                for rep in range(2):
                    for ops in plans:
                        seq += 1
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record(st)
                        if kind == "plain":
                            dp.swap("in", ops, stream=st)
                        elif kind == "ops":
                            dp.swap_ops("in", ops, fp, seq, stream=st)
                        elif kind == "layered":
                            dp.swap_layered("in", ops, fp + 4 * 4096, seq, stream=st)
                        else:
                            dp.swap_signaled("in", ops, seq, op_flags=fp,
                                             plane_flags=fp + 4 * 4096, stream=st)
                        e1.record(st)
                        st.synchronize()
                        if rep:
                            times.append(e0.elapsed_time(e1))
                row[kind + "_gbs"] = round(blocks * geo.block_bytes / (statistics.median(times)
                                                                        * 1e-3) / 1e9, 2)
            res["runs"].append(row)
            print(json.dumps(row), flush=True)
    dp.set_budget(0.0)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/swapin_path_probe.json", "w") as f:
        json.dump(res, f, indent=1)
    host.close()


if __name__ == "__main__":
    main()
