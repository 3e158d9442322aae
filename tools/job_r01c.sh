timeout 600 python -m pytest tests/test_dataplane_gpu.py -q -x -k "layered or bitexact" 2>&1 | tail -4
timeout 600 python tools/layered_bench.py 2>&1 | tail -5
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 5000 gpurun_out/bench_full.json; tail -3 gpurun_out/bench_full.err
timeout 1500 python tools/live_trace.py --convs 100 --rate 2 --modes full:kernel,baseline:ce_per_block,blockgroup:kernel --out gpurun_out/live_trace_100.json 2>&1 | tail -5
