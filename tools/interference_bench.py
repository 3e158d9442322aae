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
from paper_2411_18424_b200 import synthetic as orc  # noqa: E402  (plan generator)
from paper_2411_18424_b200.dataplane import HostKVPool, PagedKVCache, SwapDataPlane  # noqa: E402
from paper_2411_18424_b200.geometry import LLAMA3_8B  # noqa: E402
from paper_2411_18424_b200.live import DecodeEmulator  # noqa: E402

STEP_US = 2000.0
POOL = 4096
# DECODE_LAYERS=L: a step is L weight-stream kernels of STEP_US / L each (a
# model's per-layer kernels) instead of one STEP_US kernel.
LAYERS = int(os.environ.get("DECODE_LAYERS", "1"))


def decode_steps(dec, stream, n):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    evs[0].record(stream)
    for i in range(n):
        for _ in range(LAYERS):
            dec.launch_us(stream, STEP_US / LAYERS)
        evs[i + 1].record(stream)
    return evs


def main():
    geo = LLAMA3_8B
    cache = PagedKVCache(geo, POOL, device="cuda:0")
    host = HostKVPool(POOL, geo.block_bytes)
    dp = SwapDataPlane(cache, host)
    cache.planes.view(torch.int32).random_()
    dec = DecodeEmulator("cuda:0", weight_bytes=16 << 30,
                         ctas=int(os.environ.get("DECODE_CTAS", "0")))
    green = int(os.environ.get("GREEN", "0"))
    if green:
        # swap kernels on their own SM group (green contexts), decode on the rest
        from paper_2411_18424_b200.dataplane import sm_partition
        (s_out, s_in), comp, sms = sm_partition("cuda:0", swap_sms=green, swap_streams=2)
    else:
        comp = torch.cuda.Stream(priority=-1)
        s_out, s_in = torch.cuda.Stream(), torch.cuda.Stream()
        sms = None
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
    results = {"decode_step_solo_ms": round(solo, 4), "decode_ctas": dec.ctas,
               "decode_layers": LAYERS,
               "sm_partition": sms, "runs": []}
    print(json.dumps(results), flush=True)

    # (label, path, {dir: (ctas, threads)}, {dir: pace GB/s}, impl, dirs)
    # impl: kernel | ce_staged | ce_per_run
    sweep = os.environ.get("SWEEP", "in")
    configs = []
    if sweep == "probe":
        for ct, pace in (((148, 32), 20.0), ((148, 32), 40.0), ((148, 32), 50.0),
                         ((16, 512), 50.0), ((4, 512), 50.0), ((4, 512), 0.0)):
            configs.append((f"lsu{ct[0]}x{ct[1]}", "lsu", {"out": (8, 512), "in": ct},
                            {"out": 0.0, "in": pace}, "kernel", ("in",)))
        configs.append(("ce_per_run", "lsu", {"out": (8, 512), "in": (16, 512)},
                        {"out": 0.0, "in": 0.0}, "ce_per_run", ("in",)))
        configs.append(("lsu8x512", "lsu", {"out": (8, 512), "in": (148, 32)},
                        {"out": 52.0, "in": 0.0}, "kernel", ("out",)))
        configs.append(("lsu_duplex", "lsu", {"out": (8, 512), "in": (148, 32)},
                        {"out": 25.0, "in": 25.0}, "kernel", ("out", "in")))
    elif sweep == "probe2":
        for ct in ((2, 512), (3, 512), (4, 512), (6, 512), (4, 256), (8, 256), (16, 128)):
            configs.append((f"lsu{ct[0]}x{ct[1]}", "lsu", {"out": (8, 512), "in": ct},
                            {"out": 0.0, "in": 0.0}, "kernel", ("in",)))
        for ct in ((1, 512), (2, 512), (2, 256), (4, 128)):
            configs.append((f"lsu{ct[0]}x{ct[1]}", "lsu", {"out": ct, "in": (4, 512)},
                            {"out": 0.0, "in": 0.0}, "kernel", ("out",)))
        for po in (0.0, 26.0, 30.0):
            configs.append(("duplex_in4x512", "lsu", {"out": (8, 512), "in": (4, 512)},
                            {"out": po, "in": 0.0}, "kernel", ("out", "in")))
    elif sweep == "probe3":
        for ct, pace in (((8, 256), 0.0), ((6, 256), 0.0), ((8, 256), 50.0), ((8, 256), 52.0),
                         ((148, 32), 50.0), ((148, 32), 50.5), ((148, 32), 51.0),
                         ((4, 512), 50.0)):
            configs.append((f"lsu{ct[0]}x{ct[1]}", "lsu", {"out": (8, 512), "in": ct},
                            {"out": 0.0, "in": pace}, "kernel", ("in",)))
    elif sweep == "probe4":
        for ct, pace in (((8, 256), 0.0), ((148, 32), 50.0), ((32, 512), 0.0), ((8, 512), 0.0)):
            configs.append((f"lsu{ct[0]}x{ct[1]}", "lsu", {"out": (8, 512), "in": ct},
                            {"out": 0.0, "in": pace}, "kernel", ("in",)))
        for ct, pace in (((8, 512), 52.0), ((8, 512), 0.0), ((32, 512), 0.0)):
            configs.append((f"lsu{ct[0]}x{ct[1]}", "lsu", {"out": ct, "in": (8, 256)},
                            {"out": pace, "in": 0.0}, "kernel", ("out",)))
        configs.append(("duplex", "lsu", {"out": (8, 512), "in": (8, 256)},
                        {"out": 0.0, "in": 0.0}, "kernel", ("out", "in")))
        configs.append(("duplex_paced", "lsu", {"out": (8, 512), "in": (8, 256)},
                        {"out": 52.0, "in": 0.0}, "kernel", ("out", "in")))
    elif sweep == "policy":
        configs.append(("in8x256", "lsu", {"out": (8, 512), "in": (8, 256)},
                        {"out": 0.0, "in": 0.0}, "kernel", ("in",)))
        configs.append(("out8x512p52", "lsu", {"out": (8, 512), "in": (8, 256)},
                        {"out": 52.0, "in": 0.0}, "kernel", ("out",)))
        configs.append(("duplex", "lsu", {"out": (8, 512), "in": (8, 256)},
                        {"out": 52.0, "in": 0.0}, "kernel", ("out", "in")))
    elif sweep == "layers":
        # the serving policy's shapes, and swap-in paced lower
        for pace in (0.0, 40.0, 30.0, 20.0):
            configs.append((f"in8x256p{pace:g}", "lsu", {"out": (8, 512), "in": (8, 256)},
                            {"out": 0.0, "in": pace}, "kernel", ("in",)))
        configs.append(("out8x512p52", "lsu", {"out": (8, 512), "in": (8, 256)},
                        {"out": 52.0, "in": 0.0}, "kernel", ("out",)))
        configs.append(("out8x512p30", "lsu", {"out": (8, 512), "in": (8, 256)},
                        {"out": 30.0, "in": 0.0}, "kernel", ("out",)))
        configs.append(("bulk_in8", "bulk", {"out": (8, 32), "in": (8, 32)},
                        {"out": 0.0, "in": 0.0}, "kernel", ("in",)))
        configs.append(("ce_staged_in", "lsu", {"out": (8, 512), "in": (8, 256)},
                        {"out": 0.0, "in": 0.0}, "ce_staged", ("in",)))
        configs.append(("ce_staged_out", "lsu", {"out": (8, 512), "in": (8, 256)},
                        {"out": 0.0, "in": 0.0}, "ce_staged", ("out",)))
    elif sweep == "burst":
        # same mean swap-in rate, released steadily or in bursts (kvs_set_pace_burst)
        for pace in (10.0, 20.0, 40.0):
            for burst in (0, 1 << 20, 8 << 20, 32 << 20):
                configs.append((f"in8x256p{pace:g}b{burst >> 20}M", "lsu",
                                {"out": (8, 512), "in": (8, 256)},
                                {"out": 0.0, "in": pace}, "kernel", ("in",), burst))
    elif sweep == "knee":
        # swap-in pace just below the link rate: where does the cost jump?
        for pace in (30.0, 36.0, 40.0, 44.0, 46.0, 48.0, 50.0, 0.0):
            configs.append((f"in8x256p{pace:g}", "lsu", {"out": (8, 512), "in": (8, 256)},
                            {"out": 0.0, "in": pace}, "kernel", ("in",)))
        for pace in (20.0, 30.0, 40.0, 48.0, 52.0):
            configs.append((f"out8x512p{pace:g}", "lsu", {"out": (8, 512), "in": (8, 256)},
                            {"out": pace, "in": 0.0}, "kernel", ("out",)))
    elif sweep == "floor":
        # is there a cost of a running swap kernel that does not scale with its rate?
        for pace in (0.01, 0.1, 2.0, 5.0, 10.0, 20.0):
            configs.append((f"in8x256p{pace:g}", "lsu", {"out": (8, 512), "in": (8, 256)},
                            {"out": 0.0, "in": pace}, "kernel", ("in",)))
            configs.append((f"in1x32p{pace:g}", "lsu", {"out": (8, 512), "in": (1, 32)},
                            {"out": 0.0, "in": pace}, "kernel", ("in",)))
        for pace in (5.0, 20.0):
            configs.append((f"out8x512p{pace:g}", "lsu", {"out": (8, 512), "in": (8, 256)},
                            {"out": pace, "in": 0.0}, "kernel", ("out",)))
    elif sweep == "in":
        for ct in ((16, 512), (32, 128), (64, 64), (148, 32)):
            for pace in (0.0, 48.0, 40.0):
                configs.append((f"lsu{ct[0]}x{ct[1]}", "lsu", {"out": (8, 512), "in": ct},
                                {"out": 0.0, "in": pace}, "kernel", ("in",)))
        for ctas in (16, 148):
            for pace in (0.0, 48.0, 40.0):
                configs.append((f"bulk{ctas}", "bulk", {"out": (ctas, 32), "in": (ctas, 32)},
                                {"out": 0.0, "in": pace}, "kernel", ("in",)))
    else:
        for pace in (48.0, 52.0):
            configs.append(("lsu8x512", "lsu", {"out": (8, 512), "in": (148, 32)},
                            {"out": pace, "in": 0.0}, "kernel", ("out",)))
        configs.append(("bulk16", "bulk", {"out": (16, 32), "in": (16, 32)},
                        {"out": 48.0, "in": 0.0}, "kernel", ("out",)))
        for po, pi in ((20.0, 30.0), (25.0, 25.0), (30.0, 30.0), (15.0, 40.0)):
            configs.append(("lsu_duplex", "lsu", {"out": (8, 512), "in": (148, 32)},
                            {"out": po, "in": pi}, "kernel", ("out", "in")))
    for cfg in configs:
        label, path, ctas, pace, impl, dirs = cfg[:6]
        burst = cfg[6] if len(cfg) > 6 else 0
        for d in ("out", "in"):
            dp.set_path(d, path, 16384 if path == "bulk" else 0, 4 if path == "bulk" else 0)
            dp.set_launch(d, ctas[d][0], ctas[d][1] if path == "lsu" else 0)
            dp.set_pace(d, pace[d])
            dp.set_pace_burst(d, burst)
        torch.cuda.synchronize()
        t = {}
        moved = {}
        for d in dirs:
            st = s_out if d == "out" else s_in
            ops = ops_out if d == "out" else ops_in
            if 0.0 < pace[d] < 10.0:
                # slow paces: only ~0.5 s worth of bytes (decode is sampled for ~0.2 s)
                keep = max(1, int(pace[d] * 1e9 * 0.5 / geo.block_bytes))
                ops = orc.random_runs(np.random.default_rng(1), keep, 1, half, half).astype(
                    np.int32)
                if d == "in":
                    ops[:, 1:] += half
            moved[d] = int(np.asarray(ops)[:, 0].sum()) * geo.block_bytes
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            if impl == "kernel":
                dp.swap(d, ops, stream=st)
            else:
                dp.baseline(d, 2 if impl == "ce_staged" else 1, ops, stream=st)
            e1.record(st)
            t[d] = (e0, e1)
        # decode steps while the swaps run (steps that start before the swaps end count)
        evs = decode_steps(dec, comp, 80)
        torch.cuda.synchronize()
        swap_end = max(t[d][0].elapsed_time(t[d][1]) for d in dirs)
        steps = []
        for i in range(80):
            if t[dirs[0]][0].elapsed_time(evs[i]) > swap_end:
                break
            steps.append(evs[i].elapsed_time(evs[i + 1]))
        row = {"config": label, "impl": impl, "pace_gbs": pace, "ctas": ctas,
               "dirs": "+".join(dirs), "decode_steps_overlapped": len(steps),
               "decode_slowdown": round(statistics.median(steps) / solo - 1, 4) if steps else None,
               "decode_slowdown_mean": round(statistics.mean(steps) / solo - 1, 4) if steps else None,
               "swap_gbs": {d: round(moved[d] / (t[d][0].elapsed_time(t[d][1]) * 1e-3) / 1e9, 2)
                            for d in dirs}}
        results["runs"].append(row)
        print(json.dumps(row), flush=True)
    for d in ("out", "in"):
        dp.set_path(d, "lsu")
        dp.set_pace(d, 0.0)
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.environ.get("OUT", "gpurun_out/interference.json"), "w") as f:
        json.dump(results, f, indent=1)
    host.close()


if __name__ == "__main__":
    main()
