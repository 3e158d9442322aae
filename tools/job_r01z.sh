#!/bin/bash
# compute-sanitizer over the kernels' parity tests (memcheck, racecheck, synccheck).
cd "$GRAFT_REPO_ROOT"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --target-processes all --error-exitcode 99 --print-limit 20 \
    python -m pytest tests/test_dataplane_gpu.py -q -x \
    -k "bitexact_vs_oracle_small and (1028-3 or 4-1) or signaled or layered_swap_flags or op_flags or kv_token or empty_and_bad" \
    > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitizer_$tool.log | tail -3
done
