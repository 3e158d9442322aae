#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python bench.py --no-sweep --no-trace --steps 2 > gpurun_out/bench_bf.json 2> gpurun_out/bench_bf.err; tail -2 gpurun_out/bench_bf.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_bf.json').read().strip().splitlines()[-1])
print(d['value'], d['per_direction_gbs'], d['e2e']['value'], d['cpu_baseline']['value'])"
timeout 300 python tools/latency_probe.py --blocks 1,16 2>&1 | tail -2
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 | tail -1 | cut -c1-200
