#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_dataplane_gpu.py -q -x --tb=short -k "partition or tp_shard" 2>&1 | grep -E "^E |passed|failed" | head
timeout 900 python tools/live_trace.py --convs 64 --rate 4 --think 2 --cpu-blocks 4096 --sm-partition 8 --out gpurun_out/lt_q64_green.json 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); lat=d['latency']; print(d['mode'], {k: lat[k] for k in ('ttft_p50_ms','ttft_p99_ms','tbt_p99_ms','tbt_p999_ms','swap_induced_decode_stall')}, d['swap'])"
timeout 900 python tools/live_trace.py --convs 64 --rate 4 --think 2 --cpu-blocks 4096 --modes full:kernel --out gpurun_out/lt_q64_full.json 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); lat=d['latency']; print(d['mode'], {k: lat[k] for k in ('ttft_p50_ms','ttft_p99_ms','tbt_p99_ms','tbt_p999_ms','swap_induced_decode_stall')}, d['swap'])"
timeout 900 python bench.py --no-sweep --no-trace --no-cpu-baseline --sm-partition 8 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; tail -2 gpurun_out/bench_q.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1])
print(json.dumps(d.get('serving')))"
