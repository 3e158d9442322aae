#!/bin/bash
# Final round-1 evidence on the final kernel code: GPU suite, smoke, bench line, ncu.
cd "$GRAFT_REPO_ROOT"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
t0=$(date +%s); timeout 2400 python -m pytest tests -m gpu -q --tb=short 2>&1 | grep -E "^E |passed|failed|Error" | head -20; echo "suite wall $(( $(date +%s) - t0 )) s"
t0=$(date +%s); timeout 1500 python bench.py > gpurun_out/bench_bg.json 2> gpurun_out/bench_bg.err; echo "bench wall $(( $(date +%s) - t0 )) s"; tail -2 gpurun_out/bench_bg.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_bg.json').read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ('value','e2e','per_direction_gbs','serving','trace','clocks','cpu_baseline','gpu_launches')}))"
timeout 600 python bench.py --impl reference > gpurun_out/bench_bg_ref.json 2>&1; tail -1 gpurun_out/bench_bg_ref.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bg.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu-baseline --no-trace --sm-partition 0 > /dev/null 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:kvs_swap_kernel -c 2 -o gpurun_out/prof_bg python bench.py --steps 1 --warmup 0 --no-sweep --no-cpu-baseline --no-trace --sm-partition 0 > gpurun_out/ncu_bg.log 2>&1; echo "ncu rc=$?"
