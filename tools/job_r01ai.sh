#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests -q -x --tb=short -m gpu -k "layered or signaled or op_flags or executor or live or lockstep or done_flag or config1 or bench_two" 2>&1 | grep -E "^E |passed|failed|Error" | head
timeout 600 python tools/latency_probe.py --model llama3-70b --tp 8 --blocks 1,4,16 2>&1 | tail -3
