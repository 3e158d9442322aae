#!/bin/bash
# Re-entry check: GPU tests, default bench, repeated bench-shaped live traces.
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 900 python bench.py > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err; tail -3 gpurun_out/bench_h.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_h.json').read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ('value','e2e','per_direction_gbs','serving','trace')}))"
for i in 1 2 3; do
timeout 600 python tools/live_trace.py --convs 24 --rate 4 --think 2 --cpu-blocks 4096 --modes full:kernel,baseline:ce_per_block --out gpurun_out/lt_h$i.json 2>&1 | tail -1 | cut -c1-600
done
