#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python tools/host_mem_probe.py --blocks 2048 2>&1 | tail -4
