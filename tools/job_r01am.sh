#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -q -x --tb=short -m gpu -k "kv_token or live_attention or live_engine" 2>&1 | grep -E "^E |passed|failed|Error" | head
timeout 2400 python tools/config_runs.py c5 2>&1 | grep -E "^c5|Error" | cut -c1-400
