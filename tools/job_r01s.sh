#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python tools/latency_probe.py --model llama3-70b --tp 8 2>&1 | tail -6
timeout 600 python tools/latency_probe.py --model llama3-8b --tp 1 --blocks 1,4,16,64 2>&1 | tail -5
