#!/bin/bash
# ncu --set full of the TMA bulk kernels (bench e2e leg: throughput policy).
cd "$GRAFT_REPO_ROOT"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:kvs_swap_bulk_kernel -s 200 -c 2 -o gpurun_out/prof_bulk python bench.py --steps 1 --warmup 1 --no-sweep --no-cpu-baseline --no-trace --sm-partition 0 > gpurun_out/ncu_bulk.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_bulk.log
