timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 900 python bench.py > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_g.json').read().strip().splitlines()[-1])
print(json.dumps({k: d[k] for k in ('value','e2e','per_direction_gbs','serving','trace')}))"; tail -3 gpurun_out/bench_g.err
timeout 1500 python tools/live_trace.py --convs 100 --rate 2 --modes full:kernel --out gpurun_out/live_trace_paced.json 2>&1 | tail -2 | cut -c1-1500
