timeout 300 python -m pytest tests/test_dataplane_gpu.py -q -x -k "pacing" 2>&1 | grep -E "assert|Error|passed|failed" | head -12
for pol in latency latency unpaced; do
timeout 600 python tools/live_trace.py --convs 24 --rate 4 --think 2 --cpu-blocks 4096 --modes full:kernel --policy $pol --out gpurun_out/dbg_$pol.json 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['wall_s'], {k:d['latency'][k] for k in ('ttft_p99_ms','tbt_p999_ms','swap_induced_decode_stall')}, d['slowest_transfers_ms'][:4], d['slowest_iterations'][:3], d['ttft_top'][:4])"
done
