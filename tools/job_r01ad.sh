#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_dataplane_gpu.py -q -x --tb=short -k "split_kv or throughput_policy or executor" 2>&1 | grep -E "^E |passed|failed|Error" | head
t0=$(date +%s); timeout 1500 python bench.py > gpurun_out/bench_ad.json 2> gpurun_out/bench_ad.err; echo "bench wall $(( $(date +%s) - t0 )) s"; tail -2 gpurun_out/bench_ad.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_ad.json').read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ('value','e2e','per_direction_gbs','serving','trace','clocks')}))"
