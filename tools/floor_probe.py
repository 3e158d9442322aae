"""Where does the swap-in decode floor come from?  Run the same swap kernel
with its "host" pool placed in HBM (a device buffer: the same warps, the same
HBM writes, but no PCIe reads) at the same rate, against the 2 ms decode
step, on the 8-SM partition.  If the floor stays, it is the HBM write
pattern; if it vanishes, it is the host reads."""

import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_18424_b200 import synthetic as orc  # noqa: E402  (plan generator)
from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane  # noqa: E402
from paper_2411_18424_b200.geometry import LLAMA3_8B  # noqa: E402
from paper_2411_18424_b200.live import DecodeEmulator  # noqa: E402
from paper_2411_18424_b200.swap import partition_streams  # noqa: E402


class DevicePool:
    """Stand-in for HostKVPool backed by HBM."""

    def __init__(self, num_blocks, block_bytes):
        self.t = torch.empty(num_blocks * block_bytes, dtype=torch.uint8, device="cuda:0")
        self.dev_ptr = self.t.data_ptr()
        self.num_blocks = num_blocks
        self.block_bytes = block_bytes


def main():
    geo = LLAMA3_8B
    n = 2048
    cache = PagedKVCache(geo, 2 * n, device="cuda:0")
    (s_out, s_in), comp, sms = partition_streams(torch.device("cuda:0"), 8)
    dec = DecodeEmulator("cuda:0", weight_bytes=16 << 30, ctas=2 * sms[1], stream=comp)
    rng = np.random.default_rng(2)
    ops = orc.random_runs(rng, n, 16, 2 * n, 2 * n).astype(np.int32)
    nbytes = n * geo.block_bytes

    def steps(k):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(k + 1)]
        evs[0].record(comp)
        for i in range(k):
            dec.launch_us(comp, 2000.0)
            evs[i + 1].record(comp)
        return evs

    steps(3)
    torch.cuda.synchronize()
    ev = steps(30)
    torch.cuda.synchronize()
    solo = statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(30))
    out = {"decode_solo_ms": round(solo, 3), "runs": []}
    for pool_kind in ("host", "hbm"):
        pool = HostKVPool(2 * n, geo.block_bytes) if pool_kind == "host" else \
            DevicePool(2 * n, geo.block_bytes)
        dp = SwapDataPlane(cache, pool)
        for d, (c, t), pace in (("in", (8, 256), 0.0), ("in", (148, 32), 50.0),
                                ("out", (8, 512), 52.0)):
            dp.set_launch(d, c, t)
            dp.set_pace(d, pace)
            st = s_in if d == "in" else s_out
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            dp.swap(d, ops, stream=st)
            e1.record(st)
            ev = steps(60)
            torch.cuda.synchronize()
            span = e0.elapsed_time(e1)
            st_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(60)
                     if e0.elapsed_time(ev[i]) <= span]
            row = {"pool": pool_kind, "dir": d, "shape": f"{c}x{t}", "pace": pace,
                   "swap_gbs": round(nbytes / (span * 1e-3) / 1e9, 2),
                   "decode_slowdown": round(statistics.median(st_ms) / solo - 1, 4) if st_ms else None,
                   "steps": len(st_ms)}
            print(json.dumps(row), flush=True)
            out["runs"].append(row)
            dp.set_pace(d, 0.0)
        dp.close()
        if pool_kind == "host":
            pool.close()
    with open("gpurun_out/floor_probe.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
