#!/bin/bash
# Failing pacing test detail, host-access hint experiment, live TTFT anatomy.
cd "$GRAFT_REPO_ROOT"
timeout 300 python -m pytest tests/test_dataplane_gpu.py -q -x -k "pacing" 2>&1 | grep -E "assert|Error|passed|failed" | head -20
for h in 0 1 2 3; do KVS_HINT_OUT=$h KVS_HINT_IN=$h timeout 300 python tools/hint_bench.py --blocks 2048; done
timeout 600 python tools/live_trace.py --convs 24 --rate 4 --think 2 --cpu-blocks 4096 --out gpurun_out/lt_i24.json 2>&1 | tail -2 | cut -c1-2500
timeout 900 python tools/live_trace.py --convs 64 --rate 4 --think 2 --cpu-blocks 4096 --out gpurun_out/lt_i64.json 2>&1 | tail -2 | cut -c1-2500
