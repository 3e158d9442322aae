#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python tools/hybrid_probe.py 2>&1 | tail -14
