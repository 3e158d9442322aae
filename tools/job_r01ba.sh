#!/bin/bash
# Power check of the fuzz test: with swap-ins NOT waiting for queued compute
# (the pre-fix executor), does it catch the WAW race?  (patched in the box copy only)
cd "$GRAFT_REPO_ROOT"
python - <<'PY'
p='paper_2411_18424_b200/swap.py'
s=open(p).read()
s=s.replace("        stream.wait_stream(self.compute)\n        deps = 0","        if direction == 'out':\n            stream.wait_stream(self.compute)\n        deps = 0",1)
open(p,'w').write(s)
PY
grep -n "wait_stream(self.compute)" -B1 paper_2411_18424_b200/swap.py | head -4
for i in 1 2 3; do timeout 900 python -m pytest tests/test_executor_fuzz_gpu.py -q --tb=line 2>&1 | grep -E "passed|failed" | tail -1; done
