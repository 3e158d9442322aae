#!/bin/bash
# Probe (removed afterwards): an unbudgeted "latency_partitioned" policy. Result: the 60 GB/s
# budget is not binding on the 8-SM partition (duplex 50.8 + 27.8 GB/s at +8.7% either way).
cd "$GRAFT_REPO_ROOT"
KVS_SERVING_POLICY=latency_partitioned timeout 900 python bench.py --no-sweep --no-trace --no-cpu-baseline > gpurun_out/bench_aw.json 2> gpurun_out/bench_aw.err; tail -2 gpurun_out/bench_aw.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_aw.json').read().strip().splitlines()[-1])
print(json.dumps(d['serving']))"
for P in latency latency_partitioned; do
timeout 900 python tools/live_trace.py --convs 64 --rate 4 --think 2 --cpu-blocks 4096 --sm-partition 8 --layered --modes full:kernel --policy $P --out gpurun_out/lt_aw_$P.json 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); lat=d['latency']; print('$P', {k: lat.get(k) for k in ('ttft_p50_ms','ttft_p95_ms','ttft_p99_ms','tbt_p99_ms','tbt_p999_ms','swap_induced_decode_stall')}, d['ttft_anatomy'].get('all_mean_ms'), d['swap'])"
done
