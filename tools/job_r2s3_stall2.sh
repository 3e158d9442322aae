# round-2 session-3: one-call native step capture; live stall vs swap-in pace with it
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_decode_graph_gpu.py tests/test_engine_runtime_gpu.py tests/test_live_tp_gpu.py -q -x > gpurun_out/r2s3_s2_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r2s3_s2_pytest.log
A="--convs 64 --rate 4 --think 2 --cpu-blocks 4096 --pattern vtc --sm-partition 8 --layered --modes full:kernel --control-plane native"
run() { name=$1; shift; timeout 600 python tools/live_trace.py $A "$@" --out gpurun_out/r2s3_stall2_$name.json > gpurun_out/r2s3_stall2_$name.log 2>&1; echo $name=$?; }
run serving --policy serving
run in48 --policy p_in48 --policy-json '{"out": [8, 512, 52], "in": [8, 256, 48], "budget": 60, "share": {"in": 42}}'
run in45 --policy p_in45 --policy-json '{"out": [8, 512, 52], "in": [8, 256, 45], "budget": 60, "share": {"in": 42}}'
run serving_b --policy serving
