timeout 900 python -m pytest tests/test_engine_runtime_gpu.py -q -x 2>&1 | tail -15
timeout 1200 python tools/live_trace.py --convs 40 --rate 2 --modes full:kernel,full:ce_batch,baseline:ce_per_block,baseline:kernel 2>&1 | tail -20
