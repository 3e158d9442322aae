#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for v in 0 1 2; do KVS_ST_VARIANT=$v timeout 600 python tools/floor_probe.py 2>&1 | grep '"in"' | sed "s/^/v$v /"; done
