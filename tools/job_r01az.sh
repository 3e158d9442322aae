#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_executor_fuzz_gpu.py -q -x --tb=short 2>&1 | grep -E "^E |passed|failed|Error|assert" | head -20
