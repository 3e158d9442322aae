#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests/test_live_tp_gpu.py -q -x --tb=short --durations=3 2>&1 | grep -E "^E |passed|failed|Error|s call" | head
