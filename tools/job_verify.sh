set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2s2_pytest.log 2>&1; echo pytest=$?
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s2_smoke.log 2>&1; echo smoke=$?
tail -3 gpurun_out/r2s2_pytest.log
