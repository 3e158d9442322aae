# round-2 session-3: HEAD verification on a fresh box (suite, smoke, both bench arms), timed
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,pci.bus_id --format=csv
python -c "import __graft_entry__ as g; g.build()"
s=$(date +%s); timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2s3_pytest.log 2>&1; echo pytest=$? secs=$(( $(date +%s)-s ))
tail -3 gpurun_out/r2s3_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3_smoke.log 2>&1; echo smoke=$?
s=$(date +%s); timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2s3_ref.json 2> gpurun_out/r2s3_ref.err; echo ref=$? secs=$(( $(date +%s)-s ))
s=$(date +%s); timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r2s3_bench.json 2> gpurun_out/r2s3_bench.err; echo bench=$? secs=$(( $(date +%s)-s ))
