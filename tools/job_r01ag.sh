#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -q -x --tb=short -m gpu -k "layered or signaled or op_flags or live or lockstep" 2>&1 | grep -E "^E |passed|failed|Error" | head
timeout 900 python tools/live_trace.py --convs 64 --rate 4 --think 2 --cpu-blocks 4096 --sm-partition 8 --layered --modes full:kernel --out gpurun_out/lt_ag64.json 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); lat=d['latency']; print(d['mode'], {k: lat.get(k) for k in ('ttft_p50_ms','ttft_p95_ms','ttft_p99_ms','tbt_p99_ms','tbt_p999_ms','swap_induced_decode_stall','layered_joins')}, d['ttft_anatomy'].get('all_mean_ms'), d['swap'])"
