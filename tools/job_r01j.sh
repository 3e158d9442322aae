#!/bin/bash
# GPU tests, default bench (64-conv trace, warmed-up live engine, kernel KV writes).
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 1200 python bench.py > gpurun_out/bench_j.json 2> gpurun_out/bench_j.err; tail -3 gpurun_out/bench_j.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_j.json').read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ('value','e2e','per_direction_gbs','serving','trace')}))"
timeout 900 python tools/live_trace.py --convs 64 --rate 4 --think 2 --cpu-blocks 4096 --out gpurun_out/lt_j64.json 2>&1 | tail -2 | cut -c1-1500
