#!/bin/bash
# Default bench line (the driver's N=1 run), timed.
cd "$GRAFT_REPO_ROOT"
t0=$(date +%s); timeout 1500 python bench.py > gpurun_out/bench_u.json 2> gpurun_out/bench_u.err; echo "bench wall $(( $(date +%s) - t0 )) s"; tail -3 gpurun_out/bench_u.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_u.json').read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ('value','e2e','per_direction_gbs','roofline','serving','trace','clocks','cpu_baseline','gpu_launches')}))"
