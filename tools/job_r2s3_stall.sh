# round-2 session-3: live stall (decode start timed after the graph capture) vs swap-in pace / reads in flight / attention
set -x
python -c "import __graft_entry__ as g; g.build()"
A="--convs 64 --rate 4 --think 2 --cpu-blocks 4096 --pattern vtc --sm-partition 8 --layered --modes full:kernel --control-plane native"
run() { name=$1; shift; timeout 600 python tools/live_trace.py $A "$@" --out gpurun_out/r2s3_stall_$name.json > gpurun_out/r2s3_stall_$name.log 2>&1; echo $name=$?; }
run serving --policy serving
run noattend --policy serving --no-attend
run in45 --policy p_in45 --policy-json '{"out": [8, 512, 52], "in": [8, 256, 45], "budget": 60, "share": {"in": 42}}'
run in40 --policy p_in40 --policy-json '{"out": [8, 512, 52], "in": [8, 256, 40], "budget": 60, "share": {"in": 38}}'
run in8x128 --policy p_in8x128 --policy-json '{"out": [8, 512, 52], "in": [8, 128, 0], "budget": 60, "share": {"in": 42}}'
run paced --policy serving_paced
