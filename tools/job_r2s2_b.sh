# round-2 session-2 b: GPU suite (graph decode, native control plane), host cost of graph launch, full bench
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2h_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r2h_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; echo smoke=$?
timeout 300 python tools/graph_cost.py > gpurun_out/r2h_graph_cost.log 2>&1; echo graph_cost=$?
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2h_ref.json 2> gpurun_out/r2h_ref.err; echo ref=$?
timeout 2400 python bench.py --steps 20 --warmup 5 > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; echo bench=$?
tail -c 400 gpurun_out/r2h_bench.json
