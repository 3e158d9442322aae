# round-2 session-3: one fence per batch of completion words: flag tests, fuzz, probe
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
KVS_FUZZ_CASES=120 KVS_FUZZ_SEEDS=4 timeout 1500 python -m pytest tests/test_kernel_fuzz_gpu.py tests/test_executor_fuzz_gpu.py tests/test_dataplane_gpu.py tests/test_decode_graph_gpu.py tests/test_engine_runtime_gpu.py -q -x > gpurun_out/r2s3_fence_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r2s3_fence_pytest.log
timeout 600 python tools/layer_group_size_probe.py > gpurun_out/r2s3_fence_probe.log 2>&1; echo probe=$?
cat gpurun_out/r2s3_fence_probe.log
timeout 600 python tools/swapin_path_probe.py > gpurun_out/r2s3_fence_swapin.log 2>&1; echo swapin=$?
grep '"budget": 0.0' gpurun_out/r2s3_fence_swapin.log
