# round-2 session-3: staged path under the executor hazard fuzz and the kernel fuzz; decode interference of the staged path
set -x
python -c "import __graft_entry__ as g; g.build()"
KVS_FUZZ_SEEDS=3 timeout 900 python -m pytest tests/test_executor_fuzz_gpu.py -q -x -k "staged or mix" > gpurun_out/r2s3_fuzz_exec.log 2>&1; echo fuzz_exec=$?
tail -3 gpurun_out/r2s3_fuzz_exec.log
KVS_FUZZ_CASES=120 timeout 900 python -m pytest tests/test_kernel_fuzz_gpu.py -q -x > gpurun_out/r2s3_fuzz_kernel.log 2>&1; echo fuzz_kernel=$?
tail -3 gpurun_out/r2s3_fuzz_kernel.log
for L in 1 32; do
  SWEEP=layers GREEN=8 DECODE_LAYERS=$L DECODE_CTAS=280 timeout 900 python tools/interference_bench.py > gpurun_out/r2s3_intf_L$L.log 2>&1; echo intf_$L=$?
  cp gpurun_out/interference.json gpurun_out/r2s3_intf_L$L.json
done
