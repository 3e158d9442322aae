"""Where does a per-layer decode step lose time to a concurrent swap?

DESIGN §3.3: a decode step of 32 per-layer kernels pays ~20% under a
full-rate swap-in, one 2 ms kernel only ~7%, so the extra cost sits at kernel
boundaries.  This probe separates the boundary from the work:

* ``chain``: back-to-back near-empty kernels on the compute stream: µs per
  kernel boundary, idle vs. under each swap;
* ``decode``: the 32-layer decode step launched (a) one kernel after another
  on the stream, (b) as a CUDA graph, (c) with programmatic dependent launch
  (PDL: the next layer's kernel is scheduled while the previous one runs and
  waits on griddepcontrol.wait for its completion — a real layer-to-layer
  dependency), (d) PDL inside a CUDA graph;
  each idle and under swap-in / swap-out at full rate and at serving paces.

python tools/boundary_probe.py   -> gpurun_out/boundary_probe.json
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
from paper_2411_18424_b200.dataplane import (HostKVPool, PagedKVCache, SwapDataPlane,  # noqa: E402
                                             sm_partition)
from paper_2411_18424_b200.geometry import LLAMA3_8B  # noqa: E402
from paper_2411_18424_b200.live import DecodeEmulator  # noqa: E402

STEP_US = 2000.0
LAYERS = int(os.environ.get("DECODE_LAYERS", "32"))
POOL = 4096
PDL, WAIT = 1, 2


def main():
    geo = LLAMA3_8B
    cache = PagedKVCache(geo, POOL, device="cuda:0")
    host = HostKVPool(POOL, geo.block_bytes)
    dp = SwapDataPlane(cache, host)
    cache.planes.view(torch.int32).random_()
    green = int(os.environ.get("GREEN", "8"))
    if green:
        (s_out, s_in), comp, sms = sm_partition("cuda:0", swap_sms=green, swap_streams=2)
    else:
        comp = torch.cuda.Stream(priority=-1)
        s_out, s_in = torch.cuda.Stream(), torch.cuda.Stream()
        sms = None
    dec = DecodeEmulator("cuda:0", weight_bytes=16 << 30,
                         ctas=int(os.environ.get("DECODE_CTAS", "280")), stream=comp)
    layer_bytes = max(16, int(STEP_US / LAYERS * dec.bytes_per_us) // 16 * 16)

    def layer(stream, flags):
        rc = dec.lib.kvs_stream_read_ex(dec.index, int(stream.cuda_stream),
                                        dec.weights.data_ptr(), dec.weights.numel(),
                                        layer_bytes, dec.ctas, dec.sink.data_ptr(), flags)
        assert rc == 0, rc

    def tiny(stream):
        rc = dec.lib.kvs_stream_read_ex(dec.index, int(stream.cuda_stream),
                                        dec.weights.data_ptr(), dec.weights.numel(),
                                        16, 1, dec.sink.data_ptr(), 0)
        assert rc == 0, rc

    graphs = {}
    for name, flags in (("graph", 0), ("graph_pdl", PDL | WAIT)):
        try:
            cap = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                for _ in range(LAYERS):
                    layer(cap, flags)
            graphs[name] = g
        except Exception as exc:  # noqa: BLE001 - report and continue
            print(json.dumps({"graph_capture_failed": name, "error": str(exc)}), flush=True)

    def step(kind, stream):
        if kind == "stream":
            for _ in range(LAYERS):
                layer(stream, 0)
        elif kind == "pdl":
            for _ in range(LAYERS):
                layer(stream, PDL | WAIT)
        elif kind == "pdl_nowait":
            for _ in range(LAYERS):
                layer(stream, PDL)
        else:
            with torch.cuda.stream(stream):
                graphs[kind].replay()

    def run_steps(kind, n):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
        evs[0].record(comp)
        for i in range(n):
            step(kind, comp)
            evs[i + 1].record(comp)
        return evs

    # a chain of 500 near-empty kernels, as a graph so the CPU cannot be the bound
    cap = torch.cuda.Stream()
    chain_graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(chain_graph, stream=cap):
        for _ in range(500):
            tiny(cap)

    def run_chain(n):
        assert n % 500 == 0
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        evs[0].record(comp)
        with torch.cuda.stream(comp):
            for _ in range(n // 500):
                chain_graph.replay()
        evs[1].record(comp)
        return evs

    kinds = os.environ.get("KINDS", "stream,graph,pdl,graph_pdl,pdl_nowait").split(",")
    solo = {}
    for k in list(kinds):
        try:
            run_steps(k, 5)
            torch.cuda.synchronize()
        except Exception as exc:  # noqa: BLE001
            print(json.dumps({"kind_failed": k, "error": str(exc)}), flush=True)
            kinds.remove(k)
            continue
        evs = run_steps(k, 40)
        torch.cuda.synchronize()
        solo[k] = statistics.median(evs[i].elapsed_time(evs[i + 1]) for i in range(40))
    run_chain(500)
    torch.cuda.synchronize()
    ch = run_chain(2000)
    torch.cuda.synchronize()
    chain_solo = ch[0].elapsed_time(ch[1]) * 1e3 / 2000
    res = {"decode_layers": LAYERS, "decode_ctas": dec.ctas, "sm_partition": sms,
           "layer_bytes": layer_bytes, "solo_step_ms": {k: round(v, 4) for k, v in solo.items()},
           "chain_us_per_kernel_solo": round(chain_solo, 3), "runs": []}
    print(json.dumps(res), flush=True)

    rng = np.random.default_rng(0)
    half = POOL // 2
    ops_out = orc.random_runs(rng, half, 16, half, half).astype(np.int32)
    ops_in = orc.random_runs(rng, half, 16, half, half).astype(np.int32)
    ops_in[:, 1:] += half
    # (label, dir, (ctas, threads), pace GB/s, impl)
    swaps = [("in8x256", "in", (8, 256), 0.0, "kernel"),
             ("in8x256p40", "in", (8, 256), 40.0, "kernel"),
             ("in4x256", "in", (4, 256), 0.0, "kernel"),
             ("in2x256", "in", (2, 256), 0.0, "kernel"),
             ("out8x512p52", "out", (8, 512), 52.0, "kernel"),
             ("out8x512p20", "out", (8, 512), 20.0, "kernel"),
             ("ce_staged_in", "in", (8, 256), 0.0, "ce_staged")]
    sel = os.environ.get("SWAPS")
    if sel:
        swaps = [s for s in swaps if s[0] in sel.split(",")]
    for label, d, ct, pace, impl in swaps:
        for what in ["chain"] + kinds:
            dp.set_path(d, "lsu")
            dp.set_launch(d, ct[0], ct[1])
            dp.set_pace(d, pace)
            torch.cuda.synchronize()
            st = s_out if d == "out" else s_in
            ops = ops_out if d == "out" else ops_in
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            if impl == "kernel":
                dp.swap(d, ops, stream=st)
            else:
                dp.baseline(d, 2, ops, stream=st)
            e1.record(st)
            if what == "chain":
                # start the chain once the swap is at speed
                run_steps("stream", 2)
                chs = [run_chain(500) for _ in range(8)]
                torch.cuda.synchronize()
                swap_ms = e0.elapsed_time(e1)
                per = [c[0].elapsed_time(c[1]) * 1e3 / 500 for c in chs
                       if e0.elapsed_time(c[1]) < swap_ms]
                row = {"swap": label, "what": "chain", "pace": pace, "ctas": ct,
                       "chain_us_per_kernel": round(statistics.median(per), 3) if per else None,
                       "chains_overlapped": len(per)}
            else:
                evs = run_steps(what, 80)
                torch.cuda.synchronize()
                swap_ms = e0.elapsed_time(e1)
                steps = [evs[i].elapsed_time(evs[i + 1]) for i in range(80)
                         if e0.elapsed_time(evs[i + 1]) <= swap_ms]
                row = {"swap": label, "what": what, "pace": pace, "ctas": ct,
                       "steps_overlapped": len(steps),
                       "step_ms": round(statistics.median(steps), 4) if steps else None,
                       "slowdown": round(statistics.median(steps) / solo[what] - 1, 4)
                       if steps else None}
            nbytes = int(ops[:, 0].sum()) * geo.block_bytes
            row["swap_gbs"] = round(nbytes / (swap_ms * 1e-3) / 1e9, 2)
            res["runs"].append(row)
            print(json.dumps(row), flush=True)
    for d in ("out", "in"):
        dp.set_pace(d, 0.0)
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.environ.get("OUT", "gpurun_out/boundary_probe.json"), "w") as f:
        json.dump(res, f, indent=1)
    host.close()


if __name__ == "__main__":
    main()
