#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for i in 1 2; do
SWEEP=probe3 DECODE_CTAS=0 OUT=gpurun_out/intf_probe3_static_$i.json timeout 600 python tools/interference_bench.py 2>&1 | tail -8 | cut -c1-330
done
