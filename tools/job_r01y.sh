#!/bin/bash
cd "$GRAFT_REPO_ROOT"
t0=$(date +%s); timeout 2400 python -m pytest tests -m gpu -q --tb=short --durations=8 2>&1 | grep -E "^E |passed|failed|Error|s call" | head -30; echo "suite wall $(( $(date +%s) - t0 )) s"
