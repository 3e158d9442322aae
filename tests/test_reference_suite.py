"""Run the reference's OWN unit tests (pkg/tests, unmodified, read-only)
against this package by aliasing `kvswitch` -> paper_2411_18424_b200.

Covers every hot-path file of the reference suite (alloc, cpu_store, swap,
costmodel, scheduler, engine, core, workload): 123 tests incl. the golden
engine counts (test_engine.py:97-107) and the scheduler golden permutation
(test_scheduler.py:17-25).  test_cli.py is out of scope (CLI front end).
Skipped where /root/reference is absent (the GPU box) — tests/test_golden.py
carries the same parity there.
"""

import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_TESTS = Path("/root/reference/pkg/tests")
FILES = ["alloc", "core", "costmodel", "cpu_store", "engine", "scheduler", "swap", "workload"]

SHIM = '''
import importlib, sys
sys.path.insert(0, {root!r})
import paper_2411_18424_b200 as pkg
sys.modules["kvswitch"] = pkg
for m in {mods!r}:
    sys.modules["kvswitch." + m] = importlib.import_module("paper_2411_18424_b200." + m)
'''


@pytest.mark.skipif(not REF_TESTS.is_dir(), reason="reference not mounted")
def test_reference_suite_passes_on_this_package(tmp_path):
    (tmp_path / "conftest.py").write_text(SHIM.format(root=str(ROOT), mods=FILES))
    for f in FILES:
        src = REF_TESTS / f"test_{f}.py"
        (tmp_path / src.name).write_text(src.read_text())
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                          str(tmp_path)], capture_output=True, text=True, cwd=tmp_path,
                         timeout=900)
    tail = res.stdout[-3000:]
    assert res.returncode == 0, tail
    assert "123 passed" in tail, tail
