#!/bin/bash
cd "$GRAFT_REPO_ROOT"
KVS_FUZZ_CASES=120 timeout 1500 python -m pytest tests/test_kernel_fuzz_gpu.py -q -x --tb=short 2>&1 | grep -E "^E |passed|failed|Error|case" | head -20
