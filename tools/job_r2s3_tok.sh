# round-2 session-3: kv_tokens size classes; live stall and anatomy with them
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_decode_graph_gpu.py tests/test_engine_runtime_gpu.py tests/test_kernel_fuzz_gpu.py -q -x > gpurun_out/r2s3_tok_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r2s3_tok_pytest.log
A="--convs 64 --rate 4 --think 2 --cpu-blocks 4096 --pattern vtc --sm-partition 8 --layered --modes full:kernel --control-plane native"
for r in a b; do timeout 600 python tools/live_trace.py $A --policy serving --out gpurun_out/r2s3_tok_serving_$r.json > gpurun_out/r2s3_tok_serving_$r.log 2>&1; echo serving_$r=$?; done
timeout 600 python tools/live_trace.py $A --policy serving_link --out gpurun_out/r2s3_tok_link.json > gpurun_out/r2s3_tok_link.log 2>&1; echo link=$?
