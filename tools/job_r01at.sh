#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -q -x --tb=short -m gpu -k "layered or signaled or op_flags or executor or done_flag or live_engine" 2>&1 | grep -E "^E |passed|failed|Error" | head
for i in 1 2; do timeout 600 python tools/latency_probe.py --model llama3-70b --tp 8 --blocks 1,4,16 2>&1 | tail -3; done
