# round-2 session-3: staged copy-engine path (replaces the closed batched-memcpy API): parity, e2e policies, bench legs, suite
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,pci.bus_id --format=csv
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_dataplane_gpu.py -q -x -k "staged or copy_engine" > gpurun_out/r2s3_staged_pytest.log 2>&1; echo staged_pytest=$?
tail -3 gpurun_out/r2s3_staged_pytest.log
GROUPS=16,64 timeout 900 python tools/e2e_policy_probe.py > gpurun_out/r2s3_e2e_probe.log 2>&1; echo probe=$?
s=$(date +%s); timeout 1200 python bench.py --steps 5 --warmup 3 --no-trace --no-cpu-baseline > gpurun_out/r2s3_bench_short.json 2> gpurun_out/r2s3_bench_short.err; echo bench=$? secs=$(( $(date +%s)-s ))
s=$(date +%s); timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2s3_pytest.log 2>&1; echo pytest=$? secs=$(( $(date +%s)-s ))
tail -3 gpurun_out/r2s3_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3_smoke.log 2>&1; echo smoke=$?
