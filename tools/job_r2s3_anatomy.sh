# round-2 session-3: live-loop iteration anatomy (stress VTC trace)
set -x
python -c "import __graft_entry__ as g; g.build()"
A="--convs 64 --rate 4 --think 2 --cpu-blocks 4096 --pattern vtc --sm-partition 8"
timeout 900 python tools/live_trace.py $A --layered --modes full:kernel,baseline:ce_per_block --policy serving --out gpurun_out/r2s3_anatomy.json > gpurun_out/r2s3_anatomy.log 2>&1; echo live=$?
tail -5 gpurun_out/r2s3_anatomy.log
