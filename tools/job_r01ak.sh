#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 2400 python tools/config_runs.py c3 c5 2>&1 | grep -E "^c[345]|Error|error" | cut -c1-700
