#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_engine_runtime_gpu.py -q -x --tb=short -k "flag_ring or layered_admission" 2>&1 | grep -E "^E |passed|failed|Error" | head
