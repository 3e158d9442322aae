#!/bin/bash
# ncu evidence for the current kernels: launch list + full capture of the two swap kernels.
cd "$GRAFT_REPO_ROOT"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_w.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu-baseline --no-trace --sm-partition 0 > /dev/null 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:kvs_swap_kernel -c 2 -o gpurun_out/prof_w python bench.py --steps 1 --warmup 0 --no-sweep --no-cpu-baseline --no-trace --sm-partition 0 > gpurun_out/ncu_w.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_w.log
