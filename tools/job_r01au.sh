#!/bin/bash
# L2 evict-first variants vs decode stall (8-SM partition, static decode), twice each.
cd "$GRAFT_REPO_ROOT"
for rep in 1 2; do
for pol in 0 1 2; do
KVS_L2_POLICY=$pol SWEEP=policy GREEN=8 DECODE_CTAS=280 OUT=gpurun_out/intf_l2_${pol}_$rep.json timeout 600 python tools/interference_bench.py 2>&1 | grep config | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print('pol $pol', d['config'], d['swap_gbs'], d['decode_slowdown'])"
done; done
