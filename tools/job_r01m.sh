#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests -m gpu -q -x --tb=short 2>&1 | grep -E "^E |passed|failed|Error" | head -20
timeout 1200 python bench.py > gpurun_out/bench_m.json 2> gpurun_out/bench_m.err; tail -3 gpurun_out/bench_m.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_m.json').read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ('value','e2e','per_direction_gbs','serving','trace','config')}))"
KVS_BENCH_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --no-sweep --trace-convs 24 > gpurun_out/bench_m2.json 2> gpurun_out/bench_m2.err; tail -5 gpurun_out/bench_m2.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_m2.json').read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ('value','n_gpus','e2e','trace')}))"
