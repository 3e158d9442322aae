timeout 600 python tools/duplex_bw.py 2>&1 | tail -30
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_dataplane_gpu.py -q -x -k "bitexact and (1028 or 4-1)" 2>&1 | tail -6
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_dataplane_gpu.py -q -x -k "bitexact and 1028" 2>&1 | tail -6
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-sweep --no-cpu-baseline --trace-convs 8 2>&1 | tail -3
/usr/bin/time -v timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 4000 gpurun_out/bench_full.json; grep -E "Elapsed|Maximum resident" gpurun_out/bench_full.err
