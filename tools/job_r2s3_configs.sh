# round-2 session-3: BASELINE configs 3-5 on the final code (decode timed from the graph launch, serving paced 48)
set -x
python -c "import __graft_entry__ as g; g.build()"
s=$(date +%s); timeout 2400 python tools/config_runs.py c3 c4 c5 > gpurun_out/r2s3_configs.log 2>&1; echo configs=$? secs=$(( $(date +%s)-s ))
cp gpurun_out/config_runs.json gpurun_out/r2s3_config_runs.json
tail -5 gpurun_out/r2s3_configs.log
