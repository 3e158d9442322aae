# round-2 session-3: 128 MiB staging slots: staged tests, suite, both bench arms
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,pci.bus_id --format=csv
python -c "import __graft_entry__ as g; g.build()"
s=$(date +%s); timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2s3j_pytest.log 2>&1; echo pytest=$? secs=$(( $(date +%s)-s ))
tail -3 gpurun_out/r2s3j_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3j_smoke.log 2>&1; echo smoke=$?
s=$(date +%s); timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2s3j_ref.json 2> gpurun_out/r2s3j_ref.err; echo ref=$? secs=$(( $(date +%s)-s ))
s=$(date +%s); timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r2s3j_bench.json 2> gpurun_out/r2s3j_bench.err; echo bench=$? secs=$(( $(date +%s)-s ))
