#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 300 python -m pytest tests/test_dataplane_gpu.py -q -x --tb=short 2>&1 | grep -E "^E |passed|failed" | head -20
SWEEP=probe2 DECODE_CTAS=0 OUT=gpurun_out/intf_probe2_static.json timeout 600 python tools/interference_bench.py 2>&1 | tail -16 | cut -c1-330
SWEEP=probe2 DECODE_CTAS=-256 OUT=gpurun_out/intf_probe2_tiled.json timeout 600 python tools/interference_bench.py 2>&1 | tail -16 | cut -c1-330
