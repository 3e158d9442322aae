# round-2 session-3: compute-sanitizer on the staged path (stage kernel, ring reuse, release)
set -x
python -c "import __graft_entry__ as g; g.build()"
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all python -m pytest tests/test_dataplane_gpu.py -q -x -k "staged or copy_engine" > gpurun_out/r2s3_san_$tool.log 2>&1; echo $tool=$?
  tail -4 gpurun_out/r2s3_san_$tool.log
done
timeout 900 compute-sanitizer --tool memcheck --target-processes all python -m pytest tests/test_executor_fuzz_gpu.py -q -x -k "staged or mix" > gpurun_out/r2s3_san_fuzz.log 2>&1; echo fuzz_memcheck=$?
tail -4 gpurun_out/r2s3_san_fuzz.log
