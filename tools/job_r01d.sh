timeout 1500 python tools/live_trace.py --convs 100 --rate 2 --modes full:kernel,baseline:ce_per_block --out gpurun_out/live_trace_100b.json 2>&1 | tail -5
