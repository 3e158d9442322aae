# round-2 session-2: decode as a CUDA graph; native control plane; GPU suite
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2g_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r2g_pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep --no-trace --no-cpu-baseline > gpurun_out/r2g_bench_serving.json 2> gpurun_out/r2g_bench_serving.err; echo bench=$?
A="--convs 64 --rate 4 --think 2 --cpu-blocks 4096 --pattern vtc --sm-partition 8"
for pol in latency serving; do
  timeout 900 python tools/live_trace.py $A --layered --modes full:kernel --policy $pol --out gpurun_out/r2g_live_$pol.json > gpurun_out/r2g_live_$pol.log 2>&1; echo live_$pol=$?
done
timeout 900 python tools/live_trace.py $A --layered --modes full:kernel --policy latency --stream-decode --out gpurun_out/r2g_live_latency_stream.json > gpurun_out/r2g_live_latency_stream.log 2>&1; echo live_stream=$?
