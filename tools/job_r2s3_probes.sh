# round-2 session-3: duplex bulk group anomaly; swap-in rate per completion-signal variant
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python tools/duplex_group_probe.py > gpurun_out/r2s3_duplex_group.log 2>&1; echo duplex=$?
timeout 900 python tools/swapin_path_probe.py > gpurun_out/r2s3_swapin_path.log 2>&1; echo swapin=$?
