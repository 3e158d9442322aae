"""Short swap-in plans timed on the device only: each plan is queued behind
a stream wait on a host-set flag, so the CUDA events around it exclude the
host's launch preparation (which the plain probes include when the stream
is idle).  Also reports the host time of each launch call.

python tools/gated_swapin_probe.py   -> gpurun_out/gated_swapin_probe.json
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
    flags = torch.zeros(1 << 16, dtype=torch.int32, device="cuda:0")
    fp = flags.data_ptr()
    gate = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    st = torch.cuda.Stream()
    rng = np.random.default_rng(3)
    res = {"runs": []}
    seq = 0
    for blocks in (8, 32, 73):
        plans = [orc.random_runs(rng, blocks, 18, POOL, POOL).astype(np.int32) for _ in range(6)]
        row = {"blocks": blocks, "mib": 2 * blocks}
        for kind in ("plain", "ops", "signaled"):
            for gated in (False, True):
                times, host_us = [], []
                for rep in range(3):
                    for ops in plans:
                        seq += 1
                        st.synchronize()
                        if gated:
                            gate.zero_()
                            torch.cuda.synchronize()
                            dp.wait_flag(st, gate.data_ptr(), seq & 0x7FFFFFFF or 1)
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(st)
                        t0 = time.perf_counter()
                        if kind == "plain":
                            dp.swap("in", ops, stream=st)
                        elif kind == "ops":
                            dp.swap_ops("in", ops, fp, seq, stream=st)
                        else:
                            dp.swap_signaled("in", ops, seq, op_flags=fp,
                                             plane_flags=fp + 4 * 4096, stream=st)
                        host_us.append((time.perf_counter() - t0) * 1e6)
                        e1.record(st)
                        if gated:
                            gate.fill_(seq & 0x7FFFFFFF or 1)  # default stream: releases st
                        st.synchronize()
                        if rep:
                            times.append(e0.elapsed_time(e1))
                key = f"{kind}{'_gated' if gated else ''}"
                row[key + "_gbs"] = round(blocks * geo.block_bytes /
                                          (statistics.median(times) * 1e-3) / 1e9, 2)
                if not gated:
                    row[kind + "_host_us"] = round(statistics.median(host_us), 1)
        res["runs"].append(row)
        print(json.dumps(row), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/gated_swapin_probe.json", "w") as f:
        json.dump(res, f, indent=1)
    host.close()


if __name__ == "__main__":
    main()
