#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_dataplane_gpu.py -q -x --tb=short -k "layered or signaled" 2>&1 | grep -E "^E |passed|failed|Error" | head
timeout 600 python tools/layer_group_probe.py llama3-8b 2>&1 | tail -1
timeout 600 python tools/layer_group_probe.py llama3-70b 2>&1 | tail -1
