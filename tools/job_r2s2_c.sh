# round-2 session-2 c: GPU suite after the runtime fix; swap-in signal-variant probe
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2i_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r2i_pytest.log
timeout 600 python tools/swapin_path_probe.py > gpurun_out/r2i_swapin_probe.log 2>&1; echo probe=$?
