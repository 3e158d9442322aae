#!/bin/bash
# Round-1 final evidence: bench line, ncu launch list, ncu --set full of the swap kernels.
cd "$GRAFT_REPO_ROOT"
timeout 1200 python bench.py > gpurun_out/bench_o.json 2> gpurun_out/bench_o.err; tail -3 gpurun_out/bench_o.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_o.json').read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ('value','e2e','per_direction_gbs','serving','trace','clocks')}))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_o.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu-baseline --no-trace > /dev/null 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:kvs_swap_kernel -c 2 -o gpurun_out/prof_o python bench.py --steps 1 --warmup 0 --no-sweep --no-cpu-baseline --no-trace > gpurun_out/ncu_o.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_o.log
