#!/bin/bash
# Reference-default workload size (200 conversations, think 10 s) at 2 req/s: ~1100 turns.
cd "$GRAFT_REPO_ROOT"
timeout 1500 python tools/live_trace.py --convs 200 --rate 2 --think 10 --cpu-blocks 8192 --sm-partition 8 --layered --out gpurun_out/lt_ae200.json 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); lat=d['latency']; print(d['mode'], {k: lat.get(k) for k in ('ttft_p50_ms','ttft_p95_ms','ttft_p99_ms','tbt_p50_ms','tbt_p99_ms','tbt_p999_ms','swap_induced_decode_stall','layered_joins','kv_read_gib','wall_s')}, d['ttft_anatomy'].get('turns'), d['ttft_anatomy'].get('all_mean_ms'), d['ttft_anatomy'].get('tail_mean_ms'), d['swap'])"
