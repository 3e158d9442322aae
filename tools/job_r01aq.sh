#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_dataplane_gpu.py -q -x --tb=short -k "kv_image" 2>&1 | grep -E "^E |passed|failed|Error" | head
