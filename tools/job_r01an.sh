#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
t0=$(date +%s); timeout 2400 python -m pytest tests -m gpu -q --tb=short 2>&1 | grep -E "^E |passed|failed|Error" | head -20; echo "suite wall $(( $(date +%s) - t0 )) s"
