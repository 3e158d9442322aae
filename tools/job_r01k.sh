#!/bin/bash
# Pacing test detail; decode-stall mechanism probe (static vs tiled decode emulator).
cd "$GRAFT_REPO_ROOT"
timeout 300 python -m pytest tests/test_dataplane_gpu.py -q -x --tb=short 2>&1 | grep -E "^E |assert|passed|failed" | head -20
SWEEP=probe DECODE_CTAS=0 OUT=gpurun_out/intf_probe_static.json timeout 600 python tools/interference_bench.py 2>&1 | tail -12
SWEEP=probe DECODE_CTAS=-256 OUT=gpurun_out/intf_probe_tiled.json timeout 600 python tools/interference_bench.py 2>&1 | tail -12
