#!/bin/bash
# Soak: the executor hazard fuzz over 25 seeds x 4 modes.
cd "$GRAFT_REPO_ROOT"
KVS_FUZZ_SEEDS=25 timeout 1500 python -m pytest tests/test_executor_fuzz_gpu.py -q --tb=line 2>&1 | grep -E "passed|failed|Error" | tail -5
