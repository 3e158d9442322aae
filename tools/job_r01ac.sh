#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for P in lsu bulk lsu bulk; do
KVS_E2E_PATH=$P timeout 600 python bench.py --no-sweep --no-trace --no-cpu-baseline --steps 5 > gpurun_out/bench_ac_$P.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench_ac_$P.json').read().strip().splitlines()[-1])
print('$P', d['value'], json.dumps(d['e2e']))"
done
