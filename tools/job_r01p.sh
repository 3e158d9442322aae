#!/bin/bash
# Green-context SM partition: swap kernels on 8 SMs, decode on the other 140.
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,driver_version --format=csv,noheader
SWEEP=probe4 DECODE_CTAS=0 OUT=gpurun_out/intf_probe4_full.json timeout 600 python tools/interference_bench.py 2>&1 | tail -12 | cut -c1-300
SWEEP=probe4 GREEN=8 DECODE_CTAS=280 OUT=gpurun_out/intf_probe4_green8.json timeout 600 python tools/interference_bench.py 2>&1 | tail -12 | cut -c1-300
SWEEP=probe4 GREEN=8 DECODE_CTAS=-256 OUT=gpurun_out/intf_probe4_green8_tiled.json timeout 600 python tools/interference_bench.py 2>&1 | tail -12 | cut -c1-300
