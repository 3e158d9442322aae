set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout 600 python bench.py > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; tail -c 3000 gpurun_out/bench_ours.json; tail -5 gpurun_out/bench_ours.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2>&1; cat gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; tail -3 gpurun_out/ncu_launch_bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kvs_swap_kernel -c 2 -o gpurun_out/prof python bench.py --steps 1 --warmup 0 --no-sweep --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; tail -5 gpurun_out/ncu_full.log
ls -la gpurun_out
