"""e2e leg of bench.py (64 requests x 64 blocks through CpuStore ->
SwapManager.dispatch -> StreamExecutor, both directions overlapped, bytes
verified) under several duplex policies: which engine per direction carries
the most host-link GB/s when swap-outs and swap-ins run together.

python tools/e2e_policy_probe.py   -> gpurun_out/e2e_policy_probe.json
"""

import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane  # noqa: E402
from paper_2411_18424_b200.geometry import LLAMA3_8B  # noqa: E402
from paper_2411_18424_b200.swap import DUPLEX_POLICIES  # noqa: E402

EXTRA = {
    "mix_lsu16_cestaged": {"out": (16, 512, 0.0), "in": (8, 512, 0.0), "budget": 0.0,
                           "engine": {"in": "ce_staged"}, "signals": "plan"},
    "mix_cestaged_bulk": {"out": (64, 0, 0.0), "in": (64, 0, 0.0), "budget": 0.0,
                          "path": "bulk", "engine": {"out": "ce_staged"}, "signals": "plan"},
    "mix_cestaged_lsu": {"out": (8, 512, 0.0), "in": (32, 512, 0.0), "budget": 0.0,
                         "engine": {"out": "ce_staged"}, "signals": "plan"},
    "mix_bulk_cerun": {"out": (64, 0, 0.0), "in": (64, 0, 0.0), "budget": 0.0,
                       "path": "bulk", "engine": {"in": "ce_per_run"}, "signals": "plan"},
    "ce_run_both": {"out": (8, 512, 0.0), "in": (8, 512, 0.0), "budget": 0.0,
                    "engine": {"out": "ce_per_run", "in": "ce_per_run"}, "signals": "plan"},
}


def main():
    DUPLEX_POLICIES.update(EXTRA)
    args = bench.parse(["--steps", os.environ.get("STEPS", "5"), "--warmup", "2"])
    geo = LLAMA3_8B
    dev = torch.device("cuda", 0)
    gp, hp = bench.pools(args.plan_blocks)
    cache = PagedKVCache(geo, gp, device=dev)
    host = HostKVPool(hp, geo.block_bytes)
    dp = SwapDataPlane(cache, host)
    cache.planes.view(torch.int32).random_()
    out = {"group": args.group, "plan_blocks": args.plan_blocks, "runs": {}}
    names = os.environ.get("POLICIES", ",".join(["throughput", "throughput_mix",
                                                  "throughput_staged", *EXTRA]))
    for group in [int(g) for g in os.environ.get("GROUPS", "16").split(",")]:
        args.group = group
        for name in names.split(","):
            r = bench.run_e2e(args, geo, dp, dev, lambda: None, lambda x: x, 1, name)
            out["runs"][f"g{group}:{name}"] = {k: r[k] for k in ("value", "gpu_launches",
                                                                   "bytes_verified")}
            print(group, name, json.dumps(out["runs"][f"g{group}:{name}"]), flush=True)
            dp.set_launch("out", 0, 0)
            dp.set_launch("in", 0, 0)
    os.makedirs(ROOT / "gpurun_out", exist_ok=True)
    (ROOT / "gpurun_out" / "e2e_policy_probe.json").write_text(json.dumps(out, indent=1))
    host.close()


if __name__ == "__main__":
    main()
