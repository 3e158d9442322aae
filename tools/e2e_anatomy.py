"""Where the e2e leg's time goes (bench.run_e2e, throughput_staged policy):
host time planning and dispatching the 64 swap-outs and 64 swap-ins, the
wait for the device, and on the device the span from the first transfer's
start to the last one's end, per direction.

python tools/e2e_anatomy.py   -> gpurun_out/e2e_anatomy.json
"""

import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2411_18424_b200.costmodel import TransferParams  # noqa: E402
from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane  # noqa: E402
from paper_2411_18424_b200.geometry import LLAMA3_8B  # noqa: E402
from paper_2411_18424_b200.native_ctrl import NativeCpuStore  # noqa: E402
from paper_2411_18424_b200.swap import StreamExecutor, SwapManager  # noqa: E402
from paper_2411_18424_b200.synthetic import random_runs  # noqa: E402


def main():
    geo = LLAMA3_8B
    gp, hp = bench.pools(bench.PLAN_BLOCKS)
    cache = PagedKVCache(geo, gp, device="cuda:0")
    host = HostKVPool(hp, geo.block_bytes)
    dp = SwapDataPlane(cache, host)
    out = {"runs": {}}
    for policy in os.environ.get("POLICIES", "throughput_staged,throughput").split(","):
        for slot_mib in (64, 128):
            dp.set_staging(slot_mib << 20, 4)
            ex = StreamExecutor(dp, duplex_policy=policy, timing=True)
            mgr = SwapManager(TransferParams(), bytes_per_block=geo.block_bytes, executor=ex)
            store = NativeCpuStore(hp, reuse_enabled=True)
            rng = np.random.default_rng(7)
            runs = random_runs(rng, bench.PLAN_BLOCKS, 16, gp, hp)
            tables = [[(int(g), int(b)) for b, g, _ in runs[4 * r:4 * r + 4]] for r in range(64)]
            foot = [sum(b for _, b in t) for t in tables]
            rows = []
            for step in range(6):
                ex.history.clear()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for r in range(64):
                    mgr.dispatch(0, 0, store.plan_swap_out(r, foot[r], tables[r]))
                t1 = time.perf_counter()
                for r in range(64):
                    mgr.dispatch(0, 0, store.plan_swap_in(r, tables[r]))
                t2 = time.perf_counter()
                ex.synchronize()
                t3 = time.perf_counter()
                for r in range(64):
                    store.release(r)
                mgr.in_flight.clear()
                mgr.busy_extents.clear()
                ref = ex.history[0].start_event
                span = {}
                for d in ("out", "in"):
                    rs = [r for r in ex.history if r.direction == d]
                    span[d] = (min(ref.elapsed_time(r.start_event) for r in rs),
                               max(ref.elapsed_time(r.event) for r in rs))
                moved = 2 * sum(foot) * geo.block_bytes
                rows.append({"wall_ms": round((t3 - t0) * 1e3, 2),
                             "host_out_ms": round((t1 - t0) * 1e3, 2),
                             "host_in_ms": round((t2 - t1) * 1e3, 2),
                             "wait_ms": round((t3 - t2) * 1e3, 2),
                             "device_out_ms": [round(x, 2) for x in span["out"]],
                             "device_in_ms": [round(x, 2) for x in span["in"]],
                             "gbs_wall": round(moved / (t3 - t0) / 1e9, 2),
                             "gbs_device": round(moved / (max(span["out"][1], span["in"][1])
                                                          * 1e-3) / 1e9, 2)})
            out["runs"][f"{policy}:slot{slot_mib}"] = rows[2:]
            print(policy, slot_mib, json.dumps(rows[-1]), flush=True)
    os.makedirs(ROOT / "gpurun_out", exist_ok=True)
    (ROOT / "gpurun_out" / "e2e_anatomy.json").write_text(json.dumps(out, indent=1))
    host.close()


if __name__ == "__main__":
    main()
