# round-2 session-3: final-code evidence: suite, smoke, both bench arms, ncu launch list + full capture, duplex first-use probe
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,pci.bus_id --format=csv
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python tools/duplex_group_probe.py > gpurun_out/r2s3f_duplex_group.log 2>&1; echo duplex=$?
s=$(date +%s); timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2s3f_pytest.log 2>&1; echo pytest=$? secs=$(( $(date +%s)-s ))
tail -3 gpurun_out/r2s3f_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3f_smoke.log 2>&1; echo smoke=$?
s=$(date +%s); timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2s3f_ref.json 2> gpurun_out/r2s3f_ref.err; echo ref=$? secs=$(( $(date +%s)-s ))
s=$(date +%s); timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r2s3f_bench.json 2> gpurun_out/r2s3f_bench.err; echo bench=$? secs=$(( $(date +%s)-s ))
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_r2s3.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu-baseline --no-trace --sm-partition 0 > /dev/null 2> gpurun_out/r2s3f_ncu1.err; echo ncu1=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:kvs_swap_kernel -c 2 -o gpurun_out/prof_r2s3 python bench.py --steps 1 --warmup 0 --no-sweep --no-cpu-baseline --no-trace --sm-partition 0 > /dev/null 2> gpurun_out/r2s3f_ncu2.err; echo ncu2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kvs_stage_kernel -c 4 -o gpurun_out/prof_r2s3_stage python bench.py --steps 1 --warmup 0 --no-sweep --no-cpu-baseline --no-trace --sm-partition 0 > /dev/null 2> gpurun_out/r2s3f_ncu3.err; echo ncu3=$?
ls -la gpurun_out/
