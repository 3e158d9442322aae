timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 600 python tools/layered_bench.py 2>&1 | tail -4
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 6000 gpurun_out/bench_final.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu-baseline --no-trace > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kvs_swap_kernel -c 2 -o gpurun_out/prof_final python bench.py --steps 1 --warmup 0 --no-sweep --no-cpu-baseline --no-trace > gpurun_out/ncu_final.log 2>&1; tail -2 gpurun_out/ncu_final.log
timeout 1200 python tools/config_runs.py c5 2>&1 | grep -E "^c5" | cut -c1-600
